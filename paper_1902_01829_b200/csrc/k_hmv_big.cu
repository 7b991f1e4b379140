// Single-vector HMV kernels for blocks of up to 128 rows / columns (ranks and
// leaf sizes 65..128: 2D grid_order 9..11, 3D grid_order 5, leaf_size up to
// 128; the reference allows any, construction.hpp:14-24).  Same phases and
// arithmetic as k_hmv.cu; a lane owns the rows (2L, 2L+1) and (64+2L, 65+2L)
// of a block, a transposed product runs over two 64-column blocks.  The
// dataflow-fused sweeps of k_hmv.cu are replaced by one launch per level.
// Blocks of at most 64 x 64 keep the k_hmv.cu kernels (launchers dispatch).
#include "h2b_internal.hpp"
#include "warp_gemv.cuh"

#include <algorithm>

namespace h2b {
namespace {

using namespace wg;
constexpr int kThreads = 256;

// Column 2L + g + 64 cb of A^T v for an (up to) 128-row column-major block A
// (leading dim ld, `cols` <= 128 columns); the lane holds v at the rows
// (2L, 2L+1) in (v0, v1) and (64+2L, 65+2L) in (v2, v3).
__device__ __forceinline__ double gemvT128(const double* __restrict__ A, int ld, int cols, int g, int cb,
                                           double v0, double v1, double v2, double v3) {
  const int r = 2 * lane_id();
  const int c0 = 64 * cb;
  if (c0 >= cols) return 0.0;  // warp-uniform
  const double* Ac = A + int64_t(c0) * ld;
  return gemvT_group<true>(Ac, Ac + 64, ld, cols - c0, g, v0, v1, v2, v3, r < ld, r + 64 < ld);
}

// Rows (2L, 2L+1, 64+2L, 65+2L) of A v for an (up to) 128 x 128 block; v is
// pair-distributed: lane L holds v[2L], v[2L+1] (a0, a1), v[64+2L], v[65+2L] (a2, a3).
__device__ __forceinline__ void gemvN128(const double* __restrict__ A, int ld, int cols, double a0, double a1,
                                         double a2, double a3, double acc[4]) {
  const int r = 2 * lane_id();
  const bool ok0 = r < ld, ok1 = r + 64 < ld;
  acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
  for (int c0 = 0; c0 < cols; c0 += 8) {
    double2 lo[8], hi[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = c0 + u;
      const double* col = A + int64_t(c) * ld + r;
      lo[u] = (c < cols && ok0) ? ld_stream(col) : make_double2(0.0, 0.0);
      hi[u] = (c < cols && ok1) ? ld_stream(col + 64) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = c0 + u;  // warp-uniform
      if (c < cols) {
        const double src = c < 64 ? ((c & 1) ? a1 : a0) : ((c & 1) ? a3 : a2);
        const double sv = __shfl_sync(kFull, src, (c >> 1) & 31);
        acc[0] += lo[u].x * sv;
        acc[1] += lo[u].y * sv;
        acc[2] += hi[u].x * sv;
        acc[3] += hi[u].y * sv;
      }
    }
  }
}

__device__ __forceinline__ int row4(int h) { return 2 * lane_id() + (h & 1) + 64 * (h >> 1); }

__global__ void __launch_bounds__(kThreads) k_up_leaf_big(const double* __restrict__ x,
                                                          const int32_t* __restrict__ perm,
                                                          const double* __restrict__ leaf, int m, int ldm, int k,
                                                          int64_t nleaves, int64_t leaf0, double* __restrict__ xc,
                                                          double* __restrict__ xh) {
  const int64_t stride = int64_t(ldm) * k;
  for (int64_t il = warp_global(); il < nleaves; il += warp_count()) {
    const int64_t i = leaf0 + il;
    const int64_t base = i * m;
    double v[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int rr = row4(h);
      v[h] = 0.0;
      if (rr < m) {
        v[h] = __ldg(x + (perm ? __ldg(perm + base + rr) : base + rr));
        xc[base + rr] = v[h];
      }
    }
    if (k == 0) continue;
    const double* V = leaf + il * stride;
#pragma unroll
    for (int cb = 0; cb < 2; ++cb)
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const double o = gemvT128(V, ldm, k, g, cb, v[0], v[1], v[2], v[3]);
        const int c = 64 * cb + 2 * lane_id() + g;
        if (c < k) xh[i * k + c] = o;
      }
  }
}

// parents [p0, p1) of level l-1: x^_p = F_2p^T x^_2p + F_2p+1^T x^_2p+1
__global__ void __launch_bounds__(kThreads) k_up_level_big(const double* __restrict__ F, int ldc, int kc, int kp,
                                                           int64_t p0, int64_t p1, int64_t cbegin,
                                                           const double* __restrict__ xl,
                                                           double* __restrict__ xp) {
  const int64_t stride = int64_t(ldc) * kp;
  for (int64_t p = p0 + warp_global(); p < p1; p += warp_count()) {
    double v[2][4];
#pragma unroll
    for (int ch = 0; ch < 2; ++ch)
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int rr = row4(h);
        v[ch][h] = rr < kc ? xl[(2 * p + ch) * kc + rr] : 0.0;
      }
    const double* A0 = F + (2 * p - cbegin) * stride;
    const double* A1 = A0 + stride;
#pragma unroll
    for (int cb = 0; cb < 2; ++cb)
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const double o = gemvT128(A0, ldc, kp, g, cb, v[0][0], v[0][1], v[0][2], v[0][3]) +
                         gemvT128(A1, ldc, kp, g, cb, v[1][0], v[1][1], v[1][2], v[1][3]);
        const int c = 64 * cb + 2 * lane_id() + g;
        if (c < kp) xp[p * kp + c] = o;
      }
  }
}

// children [c0, c1) of level l: y^_c += E_c y^_{c/2}
__global__ void __launch_bounds__(kThreads) k_down_level_big(const double* __restrict__ E, int ldc, int kc, int kp,
                                                             int64_t c0, int64_t c1, int64_t cbegin,
                                                             const double* __restrict__ yp_all,
                                                             double* __restrict__ yl) {
  const int r = 2 * lane_id();
  const int64_t stride = int64_t(ldc) * kp;
  for (int64_t c = c0 + warp_global(); c < c1; c += warp_count()) {
    const double* yp = yp_all + (c >> 1) * kp;
    const double a0 = r < kp ? yp[r] : 0.0, a1 = r + 1 < kp ? yp[r + 1] : 0.0;
    const double a2 = r + 64 < kp ? yp[r + 64] : 0.0, a3 = r + 65 < kp ? yp[r + 65] : 0.0;
    double acc[4];
    gemvN128(E + (c - cbegin) * stride, ldc, kp, a0, a1, a2, a3, acc);
    double* y = yl + c * kc;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int rr = row4(h);
      if (rr < kc) y[rr] = acc[h] + y[rr];
    }
  }
}

// yc += U y^ for the leaves, then the alpha / beta scatter (to_user) or the
// cluster-order slice
__global__ void __launch_bounds__(kThreads) k_down_leaf_big(const double* __restrict__ U, int ldm, int m, int k,
                                                            int64_t nleaves, int64_t leaf0,
                                                            const double* __restrict__ yh,
                                                            const double* __restrict__ yc,
                                                            const int32_t* __restrict__ perm, double* __restrict__ y,
                                                            double alpha, double beta, int to_user) {
  const int r = 2 * lane_id();
  const int64_t stride = int64_t(ldm) * k;
  for (int64_t il = warp_global(); il < nleaves; il += warp_count()) {
    const int64_t i = leaf0 + il;
    const double* yq = yh + i * k;
    const double a0 = r < k ? yq[r] : 0.0, a1 = r + 1 < k ? yq[r + 1] : 0.0;
    const double a2 = r + 64 < k ? yq[r + 64] : 0.0, a3 = r + 65 < k ? yq[r + 65] : 0.0;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (k > 0) gemvN128(U + il * stride, ldm, k, a0, a1, a2, a3, acc);
    const int64_t base = i * m;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int rr = row4(h);
      if (rr >= m) continue;
      const double v = acc[h] + yc[base + rr];
      if (to_user) {
        const int64_t o = perm[base + rr];
        y[o] = alpha * v + (beta == 0.0 ? 0.0 : beta * y[o]);
      } else {
        y[il * m + rr] = v;
      }
    }
  }
}

struct BigLayer {
  const double* val;
  const int32_t* rp;
  const int32_t* ci;
  const double* x;
  double* y;
  int64_t stride;
  int br, bc, ld, pad;
};
struct BigTable {
  BigLayer L[kMaxLevels + 2];
};

// y_r = sum_b B_b x_{col(b)} (bsr.hpp:50-73, beta = 0) for blocks up to 128 x 128;
// x segment in four registers per lane (x[L + 32 q]).
__global__ void __launch_bounds__(kThreads) k_bsr_big(const __grid_constant__ BigTable T,
                                                      const uint32_t* __restrict__ work, int64_t nwork) {
  const int lane = lane_id();
  const int r = 2 * lane;
  for (int64_t it = warp_global(); it < nwork; it += warp_count()) {
    const uint32_t u = __ldg(work + it);
    const BigLayer& D = T.L[u >> kLayerShift];
    const int row = int(u & ((1u << kLayerShift) - 1));
    const bool ok0 = r < D.ld, ok1 = r + 64 < D.ld;
    double y[4] = {0.0, 0.0, 0.0, 0.0};
    for (int b = __ldg(D.rp + row), b1 = __ldg(D.rp + row + 1); b < b1; ++b) {
      const double* xs = D.x + int64_t(__ldg(D.ci + b)) * D.bc;
      double xr[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) xr[q] = lane + 32 * q < D.bc ? __ldg(xs + lane + 32 * q) : 0.0;
      const double* blk = D.val + int64_t(b) * D.stride + r;
      for (int j0 = 0; j0 < D.bc; j0 += 8) {
        double2 lo[8], hi[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int j = j0 + q;
          lo[q] = (j < D.bc && ok0) ? ld_stream(blk + int64_t(j) * D.ld) : make_double2(0.0, 0.0);
          hi[q] = (j < D.bc && ok1) ? ld_stream(blk + int64_t(j) * D.ld + 64) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int j = j0 + q;  // warp-uniform
          if (j < D.bc) {
            const double src = (j >> 5) == 0 ? xr[0] : (j >> 5) == 1 ? xr[1] : (j >> 5) == 2 ? xr[2] : xr[3];
            const double xj = __shfl_sync(kFull, src, j & 31);
            y[0] += lo[q].x * xj;
            y[1] += lo[q].y * xj;
            y[2] += hi[q].x * xj;
            y[3] += hi[q].y * xj;
          }
        }
      }
    }
    double* yr = D.y + int64_t(row) * D.br;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int rr = row4(h);
      if (rr < D.br) yr[rr] = y[h];
    }
  }
}

unsigned grid_big(int64_t items) {
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return unsigned(std::max<int64_t>(1, std::min<int64_t>((items + 7) / 8, int64_t(sms) * 8)));
}

}  // namespace

bool big_basis(const Matrix& B) {
  if (B.m > kMaxDim) return true;
  for (int k : B.rank)
    if (k > kMaxDim) return true;
  return false;
}

bool big_matrix(const Matrix& A) { return big_basis(A) || (!A.symmetric && big_basis(*A.colb)); }

void launch_up_leaf_big(const Matrix& B, const double* x, double* xc, double* xhat, cudaStream_t s,
                        bool cluster_order) {
  const int64_t nl = B.own_count(B.q);
  k_up_leaf_big<<<grid_big(nl), kThreads, 0, s>>>(x, cluster_order ? nullptr : B.perm.p, B.leaf.p, B.m, B.ldm,
                                                  B.rank[B.q], nl, B.own_begin(B.q), xc, xhat + B.vec_off[B.q]);
  H2B_CUDA(cudaGetLastError());
}

void launch_up_level_big(const Matrix& B, int l, double* xhat, cudaStream_t s, int64_t p0, int64_t p1) {
  k_up_level_big<<<grid_big(p1 - p0), kThreads, 0, s>>>(B.transfer.p + B.tr_off[l], B.ld(l), B.rank[l],
                                                        B.rank[l - 1], p0, p1, B.tr_begin(l),
                                                        xhat + B.vec_off[l], xhat + B.vec_off[l - 1]);
  H2B_CUDA(cudaGetLastError());
}

void launch_down_level_big(const Matrix& A, int l, double* yhat, cudaStream_t s, int64_t c0, int64_t c1) {
  k_down_level_big<<<grid_big(c1 - c0), kThreads, 0, s>>>(A.transfer.p + A.tr_off[l], A.ld(l), A.rank[l],
                                                          A.rank[l - 1], c0, c1, A.tr_begin(l),
                                                          yhat + A.vec_off[l - 1], yhat + A.vec_off[l]);
  H2B_CUDA(cudaGetLastError());
}

void launch_down_leaf_big(const Matrix& A, const double* yhat, const double* yc, double* y, double alpha,
                          double beta, bool to_user, cudaStream_t s) {
  const int64_t nl = A.own_count(A.q);
  k_down_leaf_big<<<grid_big(nl), kThreads, 0, s>>>(A.leaf.p, A.ldm, A.m, A.rank[A.q], nl, A.own_begin(A.q),
                                                    yhat + A.vec_off[A.q], yc, A.perm.p, y, alpha, beta,
                                                    to_user ? 1 : 0);
  H2B_CUDA(cudaGetLastError());
}

void launch_bsr_big(const Matrix& A, const uint32_t* work, int64_t nwork, const double* xdense, double* ydense,
                    const double* xh, double* yh, cudaStream_t s, const Matrix* xb) {
  if (nwork == 0) return;
  const std::vector<int64_t>& xoff = xb ? xb->vec_off : A.vec_off;
  BigTable T{};
  for (int l = 0; l <= A.q; ++l) {
    const Layer& L = A.cpl[l];
    BigLayer& d = T.L[l];
    d.val = L.val;
    d.rp = L.rp;
    d.ci = L.ci;
    d.x = xh + xoff[l];
    d.y = yh + A.vec_off[l];
    d.stride = L.block_stride();
    d.br = L.br;
    d.bc = L.bc;
    d.ld = std::max(2, L.ld);
  }
  BigLayer& d = T.L[A.q + 1];
  d.val = A.dense.val;
  d.rp = A.dense.rp;
  d.ci = A.dense.ci;
  d.x = xdense;
  d.y = ydense;
  d.stride = A.dense.block_stride();
  d.br = A.dense.br;
  d.bc = A.dense.bc;
  d.ld = std::max(2, A.dense.ld);
  k_bsr_big<<<grid_big(nwork), kThreads, 0, s>>>(T, work, nwork);
  H2B_CUDA(cudaGetLastError());
}

}  // namespace h2b
