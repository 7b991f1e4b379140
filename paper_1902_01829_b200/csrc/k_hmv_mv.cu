// Multi-vector H^2 mat-vec on the FP64 tensor cores (BASELINE.json configs[3]:
// n = 2^22, 16 vectors, "FP64 MMA path").  Same phase structure as k_hmv.cu
// (hmv.hpp:175-188 applied column by column), but every matrix block is read
// ONCE for up to 16 right-hand sides and multiplied with mma.sync m8n8k4 f64
// (SASS DMMA.8x8x4): a 64 x 64 block times a 64 x 16 panel is 8 x 2 output
// tiles x 16 k-steps = 256 DMMA per warp.
//
// Node vectors and cluster-order vectors are stored "vector-minor":
// element (row t, vector v) at t * 16 + v, so an 8 x 4 / 4 x 8 fragment of a
// panel is four 64-byte segments.  Matrix operands are streamed from HBM
// straight into the A fragments with evict-first loads.
#include "h2b_internal.hpp"

#include <algorithm>

namespace h2b {
namespace {

constexpr int kThreads = 256;
constexpr int NV = 16;  // vectors per pass (2 DMMA column tiles)

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int64_t warp_global() {
  return (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
}
__device__ __forceinline__ int64_t warp_count() { return (int64_t(gridDim.x) * blockDim.x) >> 5; }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct Acc {
  double c[8][2][2];  // 8 row tiles (M <= 64) x 2 column tiles (16 vectors)
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int x = 0; x < 8; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) c[x][y][0] = c[x][y][1] = 0.0;
  }
};

// acc (M x 16) += op(A) (M x K) * B (K x 16), B vector-minor (B[p * 16 + v]).
// op(A)(i, p) = TA ? A[p + i * lda] : A[i + p * lda]; A streamed (evict-first).
template <bool TA, int UNROLL = 2>
__device__ __forceinline__ void mma_panel(Acc& acc, const double* __restrict__ A, int lda, int M,
                                          int K, const double* __restrict__ B) {
  const int lane = lane_id();
  const int fr = lane >> 2, fk = lane & 3;
#pragma unroll UNROLL
  for (int p0 = 0; p0 < K; p0 += 4) {
    const int p = p0 + fk;
    const bool pk = p < K;
    double b[2];
#pragma unroll
    for (int y = 0; y < 2; ++y) b[y] = pk ? __ldg(B + p * NV + 8 * y + fr) : 0.0;
    double a[8];
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const int i = 8 * x + fr;
      a[x] = (pk && i < M) ? __ldcs(TA ? A + p + int64_t(i) * lda : A + i + int64_t(p) * lda) : 0.0;
    }
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      if (8 * x < M) {  // warp-uniform
        dmma(acc.c[x][0][0], acc.c[x][0][1], a[x], b[0]);
        dmma(acc.c[x][1][0], acc.c[x][1][1], a[x], b[1]);
      }
    }
  }
}

// out (M x 16, vector-minor) = acc (+ out when add).
__device__ __forceinline__ void store_panel(const Acc& acc, double* __restrict__ out, int M, bool add) {
  const int lane = lane_id();
  const int fr = lane >> 2, fc = 2 * (lane & 3);
#pragma unroll
  for (int x = 0; x < 8; ++x) {
    const int i = 8 * x + fr;
    if (i >= M) continue;
#pragma unroll
    for (int y = 0; y < 2; ++y) {
      double2* o = reinterpret_cast<double2*>(out + i * NV + 8 * y + fc);
      double2 v = make_double2(acc.c[x][y][0], acc.c[x][y][1]);
      if (add) {
        const double2 old = *o;
        v.x += old.x;
        v.y += old.y;
      }
      *o = v;
    }
  }
}

// xc16[t][v] = X[perm[t] + v * ldx] (v < nv; zero padding above).
__global__ void k_gather_mv(const int32_t* __restrict__ perm, const double* __restrict__ X,
                            int64_t ldx, int nv, int64_t n, double* __restrict__ xc) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n * NV;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = e / NV;
    const int v = int(e - t * NV);
    xc[e] = v < nv ? X[perm[t] + v * ldx] : 0.0;
  }
}

__global__ void __launch_bounds__(kThreads) k_up_leaf_mv(const double* __restrict__ leaf, int ldm,
                                                         int m, int k, int64_t nleaves,
                                                         const double* __restrict__ xc,
                                                         double* __restrict__ xh) {
  const int64_t stride = int64_t(ldm) * k;
  for (int64_t i = warp_global(); i < nleaves; i += warp_count()) {
    Acc acc;
    acc.zero();
    mma_panel<true>(acc, leaf + i * stride, ldm, k, m, xc + i * m * NV);  // V^T (k x m) X (m x 16)
    store_panel(acc, xh + i * k * NV, k, false);
  }
}

__global__ void __launch_bounds__(kThreads) k_up_level_mv(const double* __restrict__ F, int ldc,
                                                          int kc, int kp, int64_t np,
                                                          const double* __restrict__ xl,
                                                          double* __restrict__ xp) {
  const int64_t stride = int64_t(ldc) * kp;
  for (int64_t p = warp_global(); p < np; p += warp_count()) {
    Acc acc;
    acc.zero();
    mma_panel<true>(acc, F + (2 * p) * stride, ldc, kp, kc, xl + (2 * p) * kc * NV);
    mma_panel<true>(acc, F + (2 * p + 1) * stride, ldc, kp, kc, xl + (2 * p + 1) * kc * NV);
    store_panel(acc, xp + p * kp * NV, kp, false);
  }
}

struct LayerDescMV {
  const double* val;
  const int32_t* rp;
  const int32_t* ci;
  const double* x;  // vector-minor panel base
  double* y;
  int64_t stride;
  int br, bc, ld, pad;
};
struct LayerTableMV {
  LayerDescMV L[kMaxLevels + 2];
};

// Y_r = sum_b B_b X_{col(b)} for every work item (row of one layer).
__global__ void __launch_bounds__(kThreads, 1) k_bsr_mv(const __grid_constant__ LayerTableMV T,
                                                     const uint32_t* __restrict__ work,
                                                     int64_t nwork) {
  for (int64_t it = warp_global(); it < nwork; it += warp_count()) {
    const uint32_t u = __ldg(work + it);
    const LayerDescMV& D = T.L[u >> kLayerShift];
    const int row = int(u & ((1u << kLayerShift) - 1));
    const int b0 = __ldg(D.rp + row), b1 = __ldg(D.rp + row + 1);
    Acc acc;
    acc.zero();
    for (int b = b0; b < b1; ++b) {
      const int col = __ldg(D.ci + b);
      // the whole 64-deep block unrolled: its 128 fragment loads per lane are
      // in flight together (measured at n = 2^22: 8 k-steps 19.35 ms per
      // 16 vectors, 16 k-steps 18.39 ms, 4 k-steps at 2 CTAs/SM 19.78 ms)
      mma_panel<false, 16>(acc, D.val + int64_t(b) * D.stride, D.ld, D.br, D.bc,
                          D.x + int64_t(col) * D.bc * NV);
    }
    store_panel(acc, D.y + int64_t(row) * D.br * NV, D.br, false);
  }
}

__global__ void __launch_bounds__(kThreads) k_down_level_mv(const double* __restrict__ E, int ldc,
                                                            int kc, int kp, int64_t nc,
                                                            const double* __restrict__ yp,
                                                            double* __restrict__ yl) {
  const int64_t stride = int64_t(ldc) * kp;
  for (int64_t c = warp_global(); c < nc; c += warp_count()) {
    Acc acc;
    acc.zero();
    mma_panel<false>(acc, E + c * stride, ldc, kc, kp, yp + (c >> 1) * kp * NV);
    store_panel(acc, yl + c * kc * NV, kc, true);
  }
}

// Y[perm[t] + v ldy] = alpha (U y^ + yc)[t][v] + beta Y[...].
__global__ void __launch_bounds__(kThreads) k_down_leaf_mv(
    const double* __restrict__ U, int ldm, int m, int k, int64_t nleaves,
    const double* __restrict__ yh, const double* __restrict__ yc, const int32_t* __restrict__ perm,
    double* __restrict__ Y, int64_t ldy, int nv, double alpha, double beta) {
  const int lane = lane_id();
  const int fr = lane >> 2, fc = 2 * (lane & 3);
  const int64_t stride = int64_t(ldm) * k;
  for (int64_t i = warp_global(); i < nleaves; i += warp_count()) {
    Acc acc;
    acc.zero();
    if (k > 0) mma_panel<false>(acc, U + i * stride, ldm, m, k, yh + i * k * NV);
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const int r = 8 * x + fr;
      if (r >= m) continue;
      const int64_t t = i * m + r;
      const int64_t o = perm[t];
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int v = 8 * y + fc + h;
          if (v >= nv) continue;
          const double val = acc.c[x][y][h] + yc[t * NV + v];
          double* dst = Y + o + v * ldy;
          *dst = alpha * val + (beta == 0.0 ? 0.0 : beta * *dst);
        }
    }
  }
}

int sms() {
  static int v = [] {
    int dev = 0, s = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    return s;
  }();
  return v;
}

unsigned wgrid(int64_t items) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>((items + 7) / 8, int64_t(sms()) * 8)));
}

}  // namespace

// Y (n x nv, ld ldy) <- alpha A X + beta Y for nv <= 16 vectors, device pointers.
void hmv_multi_device(Matrix& A, Work& w, const double* X, int64_t ldx, double* Y, int64_t ldy, int nv,
                      double alpha, double beta, cudaStream_t s) {
  require(nv >= 1 && nv <= NV, "hmv_multi: 1..16 vectors per pass");
  const int q = A.q;
  const Matrix& C = A.col_basis();  // upsweep on the column basis (hmv.hpp:182)
  const int64_t nvec_pool = std::max<int64_t>({1, A.vec_off[q + 1], C.vec_off[q + 1]}) * NV;
  if (w.xc16.n < size_t(A.n) * NV) {
    w.xc16.alloc(size_t(A.n) * NV);
    w.yc16.alloc(size_t(A.n) * NV);
  }
  if (w.xh16.n < size_t(nvec_pool)) {
    w.xh16.alloc(nvec_pool);
    w.yh16.alloc(nvec_pool);
  }
  const int64_t n = A.n;
  k_gather_mv<<<unsigned(std::min<int64_t>((n * NV + 255) / 256, int64_t(sms()) * 16)), 256, 0, s>>>(
      A.perm.p, X, ldx, nv, n, w.xc16.p);
  H2B_CUDA(cudaGetLastError());
  const int64_t nl = A.nodes(q);
  double* xh = w.xh16.p;
  double* yh = w.yh16.p;
  if (C.rank[q] > 0) {
    k_up_leaf_mv<<<wgrid(nl), kThreads, 0, s>>>(C.leaf.p, C.ldm, C.m, C.rank[q], nl, w.xc16.p,
                                               xh + C.vec_off[q] * NV);
    H2B_CUDA(cudaGetLastError());
  }
  for (int l = q; l >= 1; --l) {
    const int kc = C.rank[l], kp = C.rank[l - 1];
    const int64_t np = A.nodes(l - 1);
    if (kp == 0) continue;
    if (kc == 0) {
      H2B_CUDA(cudaMemsetAsync(xh + C.vec_off[l - 1] * NV, 0, size_t(np) * kp * NV * sizeof(double), s));
      continue;
    }
    k_up_level_mv<<<wgrid(np), kThreads, 0, s>>>(C.transfer.p + C.tr_off[l], C.ld(l), kc, kp, np,
                                                 xh + C.vec_off[l] * NV, xh + C.vec_off[l - 1] * NV);
    H2B_CUDA(cudaGetLastError());
  }
  LayerTableMV T{};
  for (int l = 0; l <= q; ++l) {
    const Layer& L = A.cpl[l];
    LayerDescMV& d = T.L[l];
    d.val = L.val;
    d.rp = L.rp;
    d.ci = L.ci;
    d.x = xh + C.vec_off[l] * NV;
    d.y = yh + A.vec_off[l] * NV;
    d.stride = L.block_stride();
    d.br = L.br;
    d.bc = L.bc;
    d.ld = std::max(2, L.ld);
  }
  LayerDescMV& d = T.L[q + 1];
  d.val = A.dense.val;
  d.rp = A.dense.rp;
  d.ci = A.dense.ci;
  d.x = w.xc16.p;
  d.y = w.yc16.p;
  d.stride = A.dense.block_stride();
  d.br = A.dense.br;
  d.bc = A.dense.bc;
  d.ld = std::max(2, A.dense.ld);
  if (A.nwork) {
    k_bsr_mv<<<wgrid(A.nwork), kThreads, 0, s>>>(T, A.work.p, A.nwork);
    H2B_CUDA(cudaGetLastError());
  }
  for (int l = 1; l <= q; ++l) {
    const int kc = A.rank[l], kp = A.rank[l - 1];
    if (kc == 0 || kp == 0) continue;
    const int64_t nc = A.nodes(l);
    k_down_level_mv<<<wgrid(nc), kThreads, 0, s>>>(A.transfer.p + A.tr_off[l], A.ld(l), kc, kp, nc,
                                                   yh + A.vec_off[l - 1] * NV, yh + A.vec_off[l] * NV);
    H2B_CUDA(cudaGetLastError());
  }
  k_down_leaf_mv<<<wgrid(nl), kThreads, 0, s>>>(A.leaf.p, A.ldm, A.m, A.rank[q], nl,
                                                yh + A.vec_off[q] * NV, w.yc16.p, A.perm.p, Y, ldy, nv,
                                                alpha, beta);
  H2B_CUDA(cudaGetLastError());
}

}  // namespace h2b
