// Exact-kernel sampled validation on the device:
// validate_sampled (include/h2kit/validate.hpp:26-62).
//   x = random_vector(n, seed)               (validate.hpp:13-20, mt19937_64 U[0,1))
//   y = hmv(A, x)                            (the B200 mat-vec)
//   rows = first ceil(f n) of a partial Fisher-Yates shuffle with
//          mt19937_64(seed ^ 0x9E3779B97F4A7C15) (validate.hpp:41-46)
//   exact_i = sum_j exp(-|p_i - p_j| / ell) x_j   (one CTA per sampled row, FP64)
//   err = sqrt(sum (y_i - exact_i)^2 / sum exact_i^2)
// The host RNG calls are the reference's own libstdc++ ones, so the sample
// and x are identical; exact_i differs from the host only through exp() ulps.
#include <cuda_runtime.h>

#include <cmath>
#include <random>
#include <vector>

#include "h2b_internal.hpp"

namespace h2b {

void hmv_for_validation(Matrix& A, const double* x_dev, double* y_dev, cudaStream_t s);

namespace {

constexpr int kT = 256;

__global__ void __launch_bounds__(kT) k_exact_rows(const double* __restrict__ pts, int dim, double ell,
                                                   const double* __restrict__ x, int64_t n,
                                                   const int32_t* __restrict__ rows,
                                                   double* __restrict__ exact) {
  __shared__ double red[kT / 32];
  const int64_t i = rows[blockIdx.x];
  double pi[3] = {0, 0, 0};
  for (int a = 0; a < dim; ++a) pi[a] = pts[i * dim + a];
  double acc = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += kT) {
    double d2 = 0.0;
    for (int a = 0; a < dim; ++a) {
      const double d = pi[a] - pts[j * dim + a];
      d2 += d * d;
    }
    acc += exp(-sqrt(d2) / ell) * x[j];
  }
  for (int s = 16; s >= 1; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kT / 32; ++w) t += red[w];
    exact[blockIdx.x] = t;
  }
}

}  // namespace

double validate_sampled_device(Matrix& A, const double* points_host, int dim, double ell,
                               double fraction, uint64_t seed) {
  require(fraction > 0 && fraction <= 1, "validate_sampled: fraction in (0,1]");
  require(dim == 2 || dim == 3, "validate_sampled: dim must be 2 or 3");
  require(ell > 0, "validate_sampled: correlation length must be positive");
  cudaStream_t s = A.stream;
  const int64_t n = A.n;
  // points (original order) on the device
  DevBuf<double> dp;
  const double* pts = A.pts_orig.p;
  if (points_host) {
    dp.alloc(size_t(n) * dim);
    H2B_CUDA(cudaMemcpyAsync(dp.p, points_host, size_t(n) * dim * sizeof(double), cudaMemcpyHostToDevice, s));
    pts = dp.p;
  } else {
    require(pts != nullptr && A.pts_dim == dim,
            "validate_sampled: no points stored with this matrix (pass them explicitly)");
  }
  // x = random_vector(n, seed)
  std::vector<double> x(n);
  {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(0.0, 1.0);
    for (int64_t i = 0; i < n; ++i) x[i] = dist(rng);
  }
  // sample rows (validate.hpp:41-46)
  const int64_t samples = int64_t(std::ceil(fraction * double(n)));
  std::vector<int32_t> rows(n);
  for (int64_t i = 0; i < n; ++i) rows[i] = int32_t(i);
  {
    std::mt19937_64 rng(seed ^ 0x9E3779B97F4A7C15ull);
    for (int64_t k = 0; k < samples; ++k) {
      std::uniform_int_distribution<int32_t> pick(int32_t(k), int32_t(n - 1));
      std::swap(rows[k], rows[pick(rng)]);
    }
  }
  DevBuf<double> dx, dy, dex;
  DevBuf<int32_t> drows;
  dx.alloc(n);
  dy.alloc(n);
  dex.alloc(samples);
  drows.alloc(samples);
  H2B_CUDA(cudaMemcpyAsync(dx.p, x.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
  H2B_CUDA(cudaMemcpyAsync(drows.p, rows.data(), samples * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  hmv_for_validation(A, dx.p, dy.p, s);
  k_exact_rows<<<unsigned(samples), kT, 0, s>>>(pts, dim, ell, dx.p, n, drows.p, dex.p);
  H2B_CUDA(cudaGetLastError());
  std::vector<double> y(n), ex(samples);
  H2B_CUDA(cudaMemcpyAsync(y.data(), dy.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  H2B_CUDA(cudaMemcpyAsync(ex.data(), dex.p, samples * sizeof(double), cudaMemcpyDeviceToHost, s));
  H2B_CUDA(cudaStreamSynchronize(s));
  double num = 0, den = 0;
  for (int64_t k = 0; k < samples; ++k) {
    const double d = y[rows[k]] - ex[k];
    num += d * d;
    den += ex[k] * ex[k];
  }
  return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

}  // namespace h2b
