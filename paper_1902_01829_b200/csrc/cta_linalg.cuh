// CTA-cooperative FP64 small dense linear algebra in shared memory (the
// per-entry bodies of the reference's batched engine, include/h2kit/linalg.hpp
// and batch.hpp, re-designed for one CTA per batch entry).
//
// Conventions follow the reference exactly where results are defined by them:
//  * Householder QR with beta = -sign(alpha)||x||, tau = (beta-alpha)/beta,
//    zero columns get tau = 0 (linalg.hpp:48-75); R is returned with a
//    non-negative diagonal and the matching Q columns negated (:100-131).
//  * One-sided Jacobi SVD with the skip rule |a_pq| <= 16 eps sqrt(a_pp a_qq)
//    or a_pq == 0 and at most 60 sweeps (:142-176); sigma are the column norms,
//    stable-sorted descending; zero columns give zero vectors (:178-232).
//    (The Jacobi kernel itself is k_jacobi64 in compress.cu.)
// All matrices are column-major with explicit leading dimensions.
#pragma once

#include <cuda_runtime.h>

namespace h2b {
namespace cta {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int lane() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp() { return threadIdx.x >> 5; }
__device__ __forceinline__ int nthreads() { return blockDim.x; }
__device__ __forceinline__ int nwarps() { return blockDim.x >> 5; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) v += __shfl_xor_sync(kFull, v, s);
  return v;
}

// Deterministic CTA-wide sum; `red` is >= nwarps() + 1 doubles of scratch smem.
__device__ __forceinline__ double cta_sum(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if (lane() == 0) red[warp()] = v;
  __syncthreads();
  if (warp() == 0) {
    double t = lane() < nwarps() ? red[lane()] : 0.0;
    t = warp_sum(t);
    if (lane() == 0) red[nwarps()] = t;
  }
  __syncthreads();
  return red[nwarps()];
}

// Copy a rows x cols block between column-major buffers (global or smem).
__device__ __forceinline__ void copy_block(double* dst, int ldd, const double* src, int lds,
                                          int rows, int cols) {
  for (int e = threadIdx.x; e < rows * cols; e += nthreads()) {
    const int j = e / rows, i = e - j * rows;
    dst[i + j * ldd] = src[i + j * lds];
  }
}

// Smallest leading dimension >= rows that is == 4 (mod 16) doubles: makes the
// 8x4 / 4x8 DMMA fragment loads below 2-way (optimal) bank-conflicted.
__host__ __device__ __forceinline__ int sld(int rows) { return ((rows + 11) / 16) * 16 + 4; }

// FP64 tensor-core MMA (SASS DMMA.8x8x4): D(8x8) += A(8x4) B(4x8).
// Fragments: A[lane>>2][lane&3], B[lane&3][lane>>2], C[lane>>2][2(lane&3)+{0,1}].
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// C (m x n) = op(A) (m x k) * op(B) (k x n) on the FP64 tensor cores.  Each
// warp owns 32 x 16 output tiles (4 x 2 DMMA tiles, 16 accumulators); any
// m, n, k (edges predicated to zero).  Operands may live in smem or global.
// TRI = 1: op(A)(i, p) == 0 for p < i (upper triangular A, e.g. an R factor);
// TRI = 2: op(B)(p, j) == 0 for p < j (B = R^T with R upper triangular).  The
// DMMAs whose fragments are structurally zero are skipped; skipped terms are
// exact zeros, so the result is bitwise that of the full product.
// VM bit 1 (2): A's (B's) storage holds Householder vectors below its
// diagonal (V with an implicit unit diagonal, zero above; the storage on and
// above the diagonal is NOT read).  EPI = 1: C <- (i < epi_rows ? C : 0) - op(A) op(B).
template <bool TA, bool TB, int TRI = 0, int VM = 0, int EPI = 0>
__device__ void gemm_tc(double* C, int ldc, const double* A, int lda, const double* B, int ldb,
                        int m, int n, int k, int epi_rows = 0) {
  const int t = lane();
  const int fr = t >> 2, fk = t & 3;  // fragment row (A) / col (B), k index
  const int mt = (m + 31) >> 5, nt = (n + 15) >> 4;
  for (int wt = warp(); wt < mt * nt; wt += nwarps()) {
    const int i0 = (wt % mt) * 32, j0 = (wt / mt) * 16;
    double acc[4][2][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    const int p_begin = TRI == 1 ? (i0 & ~3) : TRI == 2 ? (j0 & ~3) : 0;
    for (int p0 = p_begin; p0 < k; p0 += 4) {
      const int p = p0 + fk;
      const bool pk = p < k;
      double a[4], b[2];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int i = i0 + 8 * x + fr;
        if (VM & 1) {
          const int r = TA ? p : i, c = TA ? i : p;  // storage coordinates
          a[x] = (pk && i < m) ? (r > c ? A[r + c * lda] : (r == c ? 1.0 : 0.0)) : 0.0;
        } else {
          a[x] = (pk && i < m && (TRI != 1 || p >= i)) ? (TA ? A[p + i * lda] : A[i + p * lda]) : 0.0;
        }
      }
#pragma unroll
      for (int y = 0; y < 2; ++y) {
        const int j = j0 + 8 * y + fr;
        if (VM & 2) {
          const int r = TB ? j : p, c = TB ? p : j;  // storage coordinates
          b[y] = (pk && j < n) ? (r > c ? B[r + c * ldb] : (r == c ? 1.0 : 0.0)) : 0.0;
        } else {
          b[y] = (pk && j < n && (TRI != 2 || p >= j)) ? (TB ? B[j + p * ldb] : B[p + j * ldb]) : 0.0;
        }
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) {
          // structurally zero fragments (warp-uniform test)
          if (TRI == 1 && p0 + 3 < i0 + 8 * x) continue;
          if (TRI == 2 && p0 + 3 < j0 + 8 * y) continue;
          dmma(acc[x][y][0], acc[x][y][1], a[x], b[y]);
        }
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int i = i0 + 8 * x + fr, j = j0 + 8 * y + 2 * fk + v;
          if (i < m && j < n) {
            if (EPI == 1)
              C[i + j * ldc] = (i < epi_rows ? C[i + j * ldc] : 0.0) - acc[x][y][v];
            else
              C[i + j * ldc] = acc[x][y][v];
          }
        }
  }
}

// In-place Householder factorisation (linalg.hpp:48-75): reflectors below the
// diagonal, R on and above it; tau[cols] in smem.  Register-resident: thread
// (c = tid / G, group = tid % G) of the 64 G-thread CTA holds rows
// [group RQ, (group + 1) RQ) of column c (cols <= 64, rows <= G RQ).  For
// reflector j the owner column publishes its RAW entries below the diagonal
// (and alpha = A[j,j], the squared norm partials) to shared memory; every
// column then forms the Householder scalars itself -- sqrt and one division,
// in parallel with its dot product (log2 G shuffles) -- and updates its own
// registers.  One barrier per reflector (double-buffered publish slot).
// Group g's rows sit at x[g XQ + i]: XQ is padded so that the G groups of a
// warp (same i) read disjoint banks with 128-bit loads (a stride of RQ
// doubles puts them all in one bank).
// Same arithmetic as the reference: beta = -sign(alpha) ||x||,
// tau = (beta - alpha) / beta, v = x / (alpha - beta), zero column -> tau = 0.
// xb: smem scratch, >= kHhScratch doubles (aligned to 16 bytes here).
constexpr int kHhScratch = 2 * (144 + 16) + 2;
template <int RQ, int G = 4>
__device__ void householder_regs(double* A, int lda, int rows, int cols, double* tau, double* xb) {
  static_assert((G == 4 && (RQ == 16 || RQ == 32)) || (G == 8 && (RQ == 8 || RQ == 16)), "householder_regs");
  constexpr int XQ = G == 8 ? RQ + 2 : RQ + 4;
  constexpr int XS = G * XQ + 16;
  static_assert(2 * XS + 2 <= kHhScratch, "householder_regs: scratch");
  xb = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(xb) + 15) & ~uintptr_t(15));
  const int c = threadIdx.x / G, qd = threadIdx.x % G;
  const int r0 = qd * RQ;
  const unsigned qmask = ((1u << G) - 1u) << (lane() & ~(G - 1));
  const bool live = c < cols;
  double col[RQ];
#pragma unroll
  for (int i = 0; i < RQ; ++i) col[i] = (live && r0 + i < rows) ? A[r0 + i + c * lda] : 0.0;
  const int steps = rows < cols ? rows : cols;
  const int nb = (steps + RQ - 1) / RQ;
  for (int jb = 0; jb < nb; ++jb) {
#pragma unroll
    for (int jj = 0; jj < RQ; ++jj) {
      const int j = jb * RQ + jj;
      if (j >= steps) break;  // uniform
      double* x = xb + (j & 1) * XS;
      const double* xq = x + qd * XQ;  // this group's rows
      if (c == j) {  // owner: publish raw x (rows > j), alpha, norm^2 partial
        double q2 = 0.0;
#pragma unroll
        for (int i = 0; i < RQ; i += 2) {
          const double v0 = (r0 + i > j) ? col[i] : 0.0;
          const double v1 = (r0 + i + 1 > j) ? col[i + 1] : 0.0;
          *reinterpret_cast<double2*>(x + qd * XQ + i) = make_double2(v0, v1);
          q2 = fma(v0, v0, q2);
          q2 = fma(v1, v1, q2);
        }
        x[G * XQ + qd] = q2;
        if (qd == jb) x[G * XQ + 8] = col[jj];
      }
      __syncthreads();
      const double al = x[G * XQ + 8];
      double qs;
      {
        const double* qp = x + G * XQ;
        if (G == 8)
          qs = ((qp[0] + qp[1]) + (qp[2] + qp[3])) + ((qp[4] + qp[5]) + (qp[6] + qp[7]));
        else
          qs = (qp[0] + qp[1]) + (qp[2] + qp[3]);
      }
      const double nx = sqrt(fma(al, al, qs));
      if (nx != 0.0) {
        const double be = al >= 0.0 ? -nx : nx;
        const double am = al - be;
        const double rr = 1.0 / (be * am);  // sc = 1/(al-be) = be rr, tau = (be-al)/be = -am^2 rr
        const double sc = be * rr;
        if (c == j) {
#pragma unroll
          for (int i = 0; i < RQ; ++i)
            if (r0 + i > j) col[i] *= sc;
          if (qd == jb) col[jj] = be;
          if (threadIdx.x == G * j) tau[j] = -(am * am) * rr;
        } else if (c > j && live) {
          double w0 = 0.0, w1 = 0.0;
#pragma unroll
          for (int i = 0; i < RQ; i += 2) {
            const double2 xx = *reinterpret_cast<const double2*>(xq + i);
            w0 = fma(xx.x, col[i], w0);
            w1 = fma(xx.y, col[i + 1], w1);
          }
          double w = w0 + w1;
#pragma unroll
          for (int o = 1; o < G; o <<= 1) w += __shfl_xor_sync(qmask, w, o);
          // column c's entry in row j lives in group jb
          const double cj = __shfl_sync(qmask, col[jj], (lane() & ~(G - 1)) | jb);
          const double d = fma(sc, w, cj) * (-(am * am) * rr);
          const double f = sc * d;
          asm volatile("" ::: "memory");  // re-read x: RQ registers saved
#pragma unroll
          for (int i = 0; i < RQ; i += 2) {
            const double2 xx = *reinterpret_cast<const double2*>(xq + i);
            col[i] = fma(-xx.x, f, col[i]);
            col[i + 1] = fma(-xx.y, f, col[i + 1]);
          }
          if (qd == jb) col[jj] -= d;
        }
      } else if (threadIdx.x == G * j) {
        tau[j] = 0.0;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < RQ; ++i)
    if (live && r0 + i < rows) A[r0 + i + c * lda] = col[i];
  __syncthreads();
}

// Y <- H_0 H_1 ... H_{k-1} [Y0; 0] for the k reflectors below the diagonal
// of A (rows x k, unit leading entries, tau[j]; tau = 0 marks an identity),
// Y0 = the top k x ncols of Y (global or smem, ld ldy; rows k.. of Y are
// written).  Compact WY on the FP64 tensor cores:
//   Q = I - V T V^T,  T^{-1} = diag(1/tau) + triu(V^T V, 1)   (so no T build)
//   Z = V^T [Y0; 0] = V(0:k,:)^T Y0,  solve T^{-1} W = Z,  Y = [Y0; 0] - V W.
// A's strict upper triangle (the R factor, dead by now) is overwritten with
// triu(V^T V, 1); Zw (smem, k x ncols, ld k) holds Z then W.
__device__ void apply_q_wy(double* A, int lda, int rows, int k, const double* tau, double* Y, int ldy,
                           int ncols, double* Zw, bool y0_identity = false) {
  // G = V^T V, strict upper triangle into A's upper triangle: computed into Zw
  // first (A's upper triangle is still being read as structural zeros)
  gemm_tc<true, false, 0, 3>(Zw, k, A, lda, A, lda, k, k, rows);
  __syncthreads();
  for (int e = threadIdx.x; e < k * k; e += nthreads()) {
    const int j = e / k, i = e - j * k;
    if (i < j) A[i + j * lda] = Zw[i + j * k];
  }
  __syncthreads();
  // Z = V(0:k, :)^T Y0  (Y0 = I: Z = V(0:k, :)^T, unit upper triangular)
  if (y0_identity) {
    for (int e = threadIdx.x; e < k * ncols; e += nthreads()) {
      const int j = e / k, i = e - j * k;
      Zw[i + j * k] = j > i ? A[j + i * lda] : (i == j ? 1.0 : 0.0);
    }
  } else {
    gemm_tc<true, false, 0, 1>(Zw, k, A, lda, Y, ldy, k, ncols, k);
  }
  __syncthreads();
  // solve T^{-1} W = Z column by column: 4 lanes per column, lane t owns rows
  // i = t (mod 4) and keeps their running sums s_i = sum_{j > i} G_ij W_j
  {
    const int q4 = threadIdx.x & 3;
    for (int col = threadIdx.x >> 2; col < ncols; col += nthreads() / 4) {
      double* z = Zw + col * k;
      double sacc[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) sacc[r] = 0.0;
      const unsigned gm = 0xfu << (threadIdx.x & 28);
      for (int j = k - 1; j >= 0; --j) {
        double wj = 0.0;
        if ((j & 3) == q4) {
          const double tj = tau[j];
          double sj = 0.0;
#pragma unroll
          for (int r = 0; r < 16; ++r)
            if (4 * r + q4 == j) sj = sacc[r];
          wj = tj == 0.0 ? 0.0 : tj * (z[j] - sj);
          z[j] = wj;
        }
        wj = __shfl_sync(gm, wj, j & 3, 4);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const int i = 4 * r + q4;
          if (i < j) sacc[r] = fma(A[i + j * lda], wj, sacc[r]);
        }
      }
    }
  }
  __syncthreads();
  // Y = [Y0; 0] - V W
  gemm_tc<false, false, 0, 1, 1>(Y, ldy, A, lda, Zw, k, rows, ncols, k, k);
  __syncthreads();
}

// R (cols x cols, non-negative diagonal) to R_out; flip[j] (smem ints) marks
// negated rows (linalg.hpp:100-113).
__device__ void extract_r(const double* A, int lda, int cols, double* R, int ldr, int* flip) {
  for (int j = threadIdx.x; j < cols; j += nthreads()) flip[j] = A[j + j * lda] < 0.0;
  __syncthreads();
  for (int e = threadIdx.x; e < cols * cols; e += nthreads()) {
    const int j = e / cols, i = e - j * cols;
    const double v = i <= j ? A[i + j * lda] : 0.0;
    R[i + j * ldr] = flip[i] ? -v : v;
  }
}

// Sweep histogram of the truncation Jacobi (compile with -DH2B_SWEEP_HIST).
#ifdef H2B_SWEEP_HIST
__device__ int g_sweep_hist[64];
#endif

}  // namespace cta
}  // namespace h2b
