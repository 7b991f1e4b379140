// Algebraic recompression on the device (include/h2kit/compression.hpp:466-551).
//
//   orthogonalize (QR upsweep)   k_orth_leaf, k_orth_level          compression.hpp:69-126
//   project S <- T S T^T         k_project (one CTA per block row)  :130-169
//   ||A||_F^2                    k_sumsq                            :453-460
//   weight tree (R-only QR)      k_weights (streaming TSQR, unpadded stacks)  :184-256
//   truncate (SVD upsweep)       k_trunc_{leaf,level}_pre, k_jacobi64, k_svd_apply, k_trunc_*_apply  :267-420
//   project with rectangular T   k_project                          :542
//
// One 256-thread CTA owns one batch entry; its matrices live in shared memory
// (cta_linalg.cuh).  The per-level rank max (compression.hpp:301,375) is a
// device atomicMax; the host reads one int per level.  Pools change shape
// after truncation, so the matrix is re-laid out (new leaf/transfer/coupling
// pools, x^/y^ workspace, BSR work list) at the end.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <functional>
#include <map>
#include <mutex>
#include <vector>

#include "cta_linalg.cuh"
#include "tma.cuh"
#include "h2b_internal.hpp"

namespace h2b {

void upload_structure(Matrix& A);
void rebuild_work_list(Matrix& A);

namespace {

using cta::kThreads;

constexpr int kXb = cta::kHhScratch;  // cta::householder scratch (doubles)

// ------------------------------------------------------------------ kernels
// L2 prefetch of the QR kernels' inputs for the CTA one wave ahead (C3:
// orthogonalization 26.5 -> 25.9 ms, compress 242.7 -> 241.2 ms)
#ifndef H2B_LEVEL_PREFETCH
#define H2B_LEVEL_PREFETCH 1
#endif
constexpr bool kLevelPrefetch = H2B_LEVEL_PREFETCH;
__device__ __forceinline__ int nsm() {  // SMs on this device
  int v;
  asm("mov.u32 %0, %%nsmid;" : "=r"(v));
  return v;
}
__global__ void __launch_bounds__(kThreads) k_orth_leaf(double* __restrict__ leaf, int ldm, int m,
                                                        int k, double* __restrict__ T) {
  extern __shared__ double sm[];
  double* A = sm;                 // m x k, ld m
  double* Q = A + m * k;          // m x k, ld m
  double* Zw = Q + m * k;         // k x k
  double* tau = Zw + k * k;       // 64
  double* xb = tau + 64;          // householder publish slots
  int* flip = reinterpret_cast<int*>(xb + kXb);
  const int64_t i = blockIdx.x;
  double* U = leaf + i * int64_t(ldm) * k;
  if (kLevelPrefetch && threadIdx.x == 0 && i + 2 * nsm() < gridDim.x)  // one wave ahead (2 CTAs/SM)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(U + 2 * nsm() * int64_t(ldm) * k),
                 "r"(uint32_t(ldm * k * 8)) : "memory");
  cta::copy_block(A, m, U, ldm, m, k);
  __syncthreads();
  cta::householder_regs<16>(A, m, m, k, tau, xb);  // m <= 64
  cta::extract_r(A, m, k, T + i * int64_t(k) * k, k, flip);
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int j = e / k, r = e - j * k;
    Q[r + j * m] = r == j ? 1.0 : 0.0;
  }
  __syncthreads();
  cta::apply_q_wy(A, m, m, k, tau, Q, m, k, Zw, /*y0_identity=*/true);  // Q = H_0..H_{k-1} [I; 0]
  for (int e = threadIdx.x; e < m * k; e += blockDim.x) {
    const int j = e / m, r = e - j * m;
    U[r + int64_t(j) * ldm] = flip[j] ? -Q[r + j * m] : Q[r + j * m];
  }
}

// Parent p at level l-1: Z = [T_2p F_2p; T_2p+1 F_2p+1] (2kc x kp) -> QR.
constexpr int kLevelThreads = 512;  // level QR kernels: 16 warps (one 164 KB CTA per SM)

__global__ void __launch_bounds__(kLevelThreads) k_orth_level(double* __restrict__ F, int ldf, int kc,
                                                         int kp, const double* __restrict__ Tl,
                                                         double* __restrict__ Tp) {
  extern __shared__ double sm[];
  const int zr = 2 * kc;
  double* Z = sm;                    // zr x kp
  double* Q = Z + zr * kp;           // zr x kp
  double* Zw = Q + zr * kp;          // kp x kp
  double* tau = Zw + kp * kp;
  double* xb = tau + 64;             // householder publish slots
  int* flip = reinterpret_cast<int*>(xb + kXb);
  const int64_t p = blockIdx.x;
  const int64_t fs = int64_t(ldf) * kp;
  // L2 prefetch for the CTA that runs one wave later (one CTA per SM): its
  // two children's T and F blocks arrive while this parent's chain runs
  if (kLevelPrefetch && threadIdx.x == 0) {
    const int64_t pn = p + nsm();
    if (pn < gridDim.x) {
      const double* t0 = Tl + 2 * pn * int64_t(kc) * kc;
      const double* f0 = F + 2 * pn * fs;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(t0), "r"(uint32_t(2 * kc * kc * 8)) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(f0), "r"(uint32_t(2 * fs * 8)) : "memory");
    }
  }
  for (int ci = 0; ci < 2; ++ci) {
    const int64_t c = 2 * p + ci;
    cta::gemm_tc<false, false, 1>(Z + ci * kc, zr, Tl + c * int64_t(kc) * kc, kc, F + c * fs, ldf, kc, kp, kc);
  }
  __syncthreads();
  if (zr <= 64)
    cta::householder_regs<8, 8>(Z, zr, zr, kp, tau, xb);
  else
    cta::householder_regs<16, 8>(Z, zr, zr, kp, tau, xb);  // zr <= 128
  cta::extract_r(Z, zr, kp, Tp + p * int64_t(kp) * kp, kp, flip);
  for (int e = threadIdx.x; e < kp * kp; e += blockDim.x) {
    const int j = e / kp, r = e - j * kp;
    Q[r + j * zr] = r == j ? 1.0 : 0.0;
  }
  __syncthreads();
  cta::apply_q_wy(Z, zr, zr, kp, tau, Q, zr, kp, Zw, /*y0_identity=*/true);
  for (int ci = 0; ci < 2; ++ci) {
    double* dst = F + (2 * p + ci) * fs;
    for (int e = threadIdx.x; e < kc * kp; e += blockDim.x) {
      const int j = e / kc, r = e - j * kc;
      const double v = Q[ci * kc + r + j * zr];
      dst[r + int64_t(j) * ldf] = flip[j] ? -v : v;
    }
  }
}

struct ProjRow {
  int32_t level;
  int32_t row;
};

struct ProjLevel {
  const double* S;    // old blocks (ld_old x co)
  double* out;        // new blocks (ld_new x cn), block b at out + b * ostride
  const int32_t* rp;
  const int32_t* ci;
  const int32_t* mirror;  // symmetric levels: block index of (col, row), or null
  const double* T;    // row projections: rn x ro per node, ld rn
  const double* Tc;   // column projections: cn x co per node, ld cn (== T when symmetric)
  int ro, rn, co, cn, ld_old, ld_new;
  int64_t istride;    // block stride of S
  int64_t ostride;    // block stride of out (compress(): the old slots, == istride)
};
struct ProjTable {
  ProjLevel L[kMaxLevels + 1];
  // TMA staging of the launched level (tma != 0): 3D views {ld, cols, blocks}
  // of S, T_row and T_col, box {kPLd, 64, 1} -- one load lands a zero-padded
  // 64 x kPLd tile exactly like stage64 (out-of-range rows / columns filled
  // with zeros by the TMA unit)
  CUtensorMap mS, mT, mTc;
  int tma;
  int tri;          // T upper triangular (orthogonalization's R factors)
  double* rowsum;   // per block row: sum of squares of the projected blocks (or null)
  int max_row;      // longest block row over the levels (smem work list)
};

// S_b <- T_row S_b T_col^T for every block of one block row (compression.hpp:160-168),
// ranks <= 64.  T_row stays in smem for the row; per block, S_b and T_col are
// staged in smem (cp.async) and warp w computes the 8-row strip [8w, 8w+8) of
//   TS  = T_row S_b    (DMMA, the strip's accumulators stay in registers) and
//   out = TS T_col^T   (DMMA; TS's A fragments come from the accumulators by
//                       two quad shuffles per k-step -- TS never touches smem).
// With TRI (orthogonalization: T are upper-triangular R factors) the
// structurally zero fragments of both products are skipped.
constexpr int kPLd = 68;  // smem leading dimension (== 4 mod 16: conflict-free fragments)
// TS strip = Tr[i0:i0+8, :] S (8 x co) of warp w, i0 = 8w (false: idle warp).
template <bool TRI>
__device__ __forceinline__ bool ts_strip(const double* Tr, const double* Sb, int ro, int co, int rn,
                                         double (&acc)[8][2]) {
  const int w = cta::warp(), t = cta::lane();
  const int fr = t >> 2, fk = t & 3;
  const int i0 = 8 * w;
#pragma unroll
  for (int y = 0; y < 8; ++y) acc[y][0] = acc[y][1] = 0.0;
  if (i0 >= rn) return false;
  const int kc_end = (ro + 3) >> 2;
#pragma unroll
  for (int kc = 0; kc < 16; ++kc) {
    if (kc < kc_end && (!TRI || 4 * kc + 3 >= i0)) {
      const int p = 4 * kc + fk;
      const double a = Tr[i0 + fr + p * kPLd];
#pragma unroll
      for (int y = 0; y < 8; ++y) {
        if (8 * y < co) {
          const double b = Sb[p + (8 * y + fr) * kPLd];
          cta::dmma(acc[y][0], acc[y][1], a, b);
        }
      }
    }
  }
  return true;
}

// out strip = TS strip (8 x co) T_col^T (co x cn); TS's A fragments come from
// the accumulators by two quad shuffles per k-step (TS never touches smem).
template <bool TRI>
__device__ __forceinline__ void out_strip(const double (&acc)[8][2], const double* Tc, double* out, double* outT,
                                          int ld_new, int co, int rn, int cn, double& sumsq) {
  const int w = cta::warp(), t = cta::lane();
  const int fr = t >> 2, fk = t & 3;
  const int i0 = 8 * w;
  const int kc_end = (co + 3) >> 2;
  double o[8][2];
#pragma unroll
  for (int y = 0; y < 8; ++y) o[y][0] = o[y][1] = 0.0;
  const int src = fr * 4 + (fk >> 1);
#pragma unroll
  for (int kc = 0; kc < 16; ++kc) {
    if (kc < kc_end) {
      // A fragment TS[i0 + fr, 4 kc + fk] lives in acc[kc / 2][(fk & 1)] of
      // lane fr * 4 + 2 (kc & 1) + fk / 2
      const int sl = src + 2 * (kc & 1);
      const double s0 = __shfl_sync(0xffffffffu, acc[kc >> 1][0], sl);
      const double s1 = __shfl_sync(0xffffffffu, acc[kc >> 1][1], sl);
      const double a = (fk & 1) ? s1 : s0;
      const int p = 4 * kc + fk;
#pragma unroll
      for (int y = 0; y < 8; ++y) {
        if (8 * y < cn && (!TRI || 4 * kc + 3 >= 8 * y)) {
          const double b = Tc[8 * y + fr + p * kPLd];  // T_col[j, p]
          cta::dmma(o[y][0], o[y][1], a, b);
        }
      }
    }
  }
  const int i = i0 + fr;
  if (i < rn) {
#pragma unroll
    for (int y = 0; y < 8; ++y)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int j = 8 * y + 2 * fk + v;
        if (j < cn) {
          out[i + int64_t(j) * ld_new] = o[y][v];
          if (outT) outT[j + int64_t(i) * ld_new] = o[y][v];  // mirror block (col, row)
          sumsq = fma(o[y][v], o[y][v], sumsq);
        }
      }
  }
  if (ld_new > rn && w == 0)
    for (int j = t; j < cn; j += 32) {
      out[rn + int64_t(j) * ld_new] = 0.0;
      if (outT) outT[rn + int64_t(j) * ld_new] = 0.0;
    }
}

// Column-strip form of TS = Tr S for warp w: columns [8w, 8w+8) of TS, all
// row tiles below rn (acc[x] = row tile x).  With a triangular Tr every warp
// skips the same fragments (row tile x needs k >= 8x), so the 8 warps carry
// equal work -- the row-strip form gives warp w 16 - 2w k-steps.  Returns
// false for an idle warp (8w >= co).
template <bool TRI>
__device__ __forceinline__ bool ts_cols(const double* Tr, const double* Sb, int ro, int co, int rn,
                                        double (&acc)[8][2]) {
  const int w = cta::warp(), t = cta::lane();
  const int fr = t >> 2, fk = t & 3;
  const int j0 = 8 * w;
#pragma unroll
  for (int x = 0; x < 8; ++x) acc[x][0] = acc[x][1] = 0.0;
  if (j0 >= co) return false;
  const int kc_end = (ro + 3) >> 2;
#pragma unroll
  for (int kc = 0; kc < 16; ++kc) {
    if (kc < kc_end) {
      const int p = 4 * kc + fk;
      const double b = Sb[p + (j0 + fr) * kPLd];  // S[p, j0 + fr]
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        if (8 * x < rn && (!TRI || 4 * kc + 3 >= 8 * x)) {
          const double a = Tr[8 * x + fr + p * kPLd];
          cta::dmma(acc[x][0], acc[x][1], a, b);
        }
      }
    }
  }
  return true;
}

// TS column strip of warp w into smem (ld kPLd): acc[x][v] = TS[8x + fr, 8w + 2fk + v].
__device__ __forceinline__ void ts_store(const double (&acc)[8][2], double* TSb, int rn) {
  const int w = cta::warp(), t = cta::lane();
  const int fr = t >> 2, fk = t & 3;
#pragma unroll
  for (int x = 0; x < 8; ++x)
    if (8 * x < rn) {
      TSb[8 * x + fr + (8 * w + 2 * fk) * kPLd] = acc[x][0];
      TSb[8 * x + fr + (8 * w + 2 * fk + 1) * kPLd] = acc[x][1];
    }
}

// out strip of warp w = TS[8w:8w+8, :] T_col^T with TS's A fragments from smem.
template <bool TRI>
__device__ __forceinline__ void out_rows(const double* TSb, const double* Tc, double* out, double* outT,
                                         int ld_new, int co, int rn, int cn, double& sumsq) {
  const int w = cta::warp(), t = cta::lane();
  const int fr = t >> 2, fk = t & 3;
  const int i0 = 8 * w;
  if (i0 >= rn) return;
  const int kc_end = (co + 3) >> 2;
  double o[8][2];
#pragma unroll
  for (int y = 0; y < 8; ++y) o[y][0] = o[y][1] = 0.0;
#pragma unroll
  for (int kc = 0; kc < 16; ++kc) {
    if (kc < kc_end) {
      const int p = 4 * kc + fk;
      const double a = TSb[i0 + fr + p * kPLd];
#pragma unroll
      for (int y = 0; y < 8; ++y) {
        if (8 * y < cn && (!TRI || 4 * kc + 3 >= 8 * y)) {
          const double b = Tc[8 * y + fr + p * kPLd];  // T_col[j, p]
          cta::dmma(o[y][0], o[y][1], a, b);
        }
      }
    }
  }
  const int i = i0 + fr;
  if (i < rn) {
#pragma unroll
    for (int y = 0; y < 8; ++y)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int j = 8 * y + 2 * fk + v;
        if (j < cn) {
          out[i + int64_t(j) * ld_new] = o[y][v];
          if (outT) outT[j + int64_t(i) * ld_new] = o[y][v];  // mirror block (col, row)
          sumsq = fma(o[y][v], o[y][v], sumsq);
        }
      }
  }
  if (ld_new > rn && w == 0)
    for (int j = t; j < cn; j += 32) {
      out[rn + int64_t(j) * ld_new] = 0.0;
      if (outT) outT[rn + int64_t(j) * ld_new] = 0.0;
    }
}

// 8-byte asynchronous global -> shared copies (cp.async.ca), grouped.
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

// rows x cols block (ld lds, global) into a zero-padded 64 x 64 smem tile (ld kPLd)
__device__ __forceinline__ void stage64(double* dst, const double* src, int lds, int rows, int cols) {
  if (((rows | lds) & 1) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    // 16-byte copies (even rows and ld, aligned base): half the instructions
    for (int e = threadIdx.x; e < 64 * 32; e += blockDim.x) {
      const int j = e >> 5, i = 2 * (e & 31);
      if (i < rows && j < cols)
        cp_async16(dst + i + j * kPLd, src + i + int64_t(j) * lds);
      else
        *reinterpret_cast<double2*>(dst + i + j * kPLd) = make_double2(0.0, 0.0);
    }
    return;
  }
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
    const int j = e >> 6, i = e & 63;
    if (i < rows && j < cols)
      cp_async8(dst + i + j * kPLd, src + i + int64_t(j) * lds);
    else
      dst[i + j * kPLd] = 0.0;
  }
}

// S_b <- T_row S_b T_col^T for every block of one block row (compression.hpp:
// 160-168), ranks <= 64.  T_row stays in smem for the row; per block, S_b and
// T_col are staged in smem by cp.async and warp w computes the 8-row strip
// [8w, 8w+8) of TS = T_row S_b (DMMA, accumulators in registers) and then of
// out = TS T_col^T.  Software pipeline over the row's blocks with single
// buffers: S_{b+1} is loaded while out_b is computed (S_b is dead by then) and
// T_col,{b+1} while TS_{b+1} is computed.  With TRI (orthogonalization: T are
// upper-triangular R factors) the structurally zero fragments are skipped.
// The row's work list (symmetric levels: upper blocks only, each also writing
// its mirror) is compacted into smem first: no dependent global index loads
// between blocks.
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(tma::smem_u32(dst)),
      "l"(map), "r"(0), "r"(0), "r"(c2), "r"(tma::smem_u32(bar))
      : "memory");
}
constexpr uint32_t kTileBytes = 64 * kPLd * sizeof(double);
#ifndef H2B_PROJ_TMA
#define H2B_PROJ_TMA 1
#endif
constexpr bool kProjTma = H2B_PROJ_TMA;

__global__ void __launch_bounds__(kThreads, 2) k_project(const __grid_constant__ ProjTable P,
                                                         const ProjRow* __restrict__ rows) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[3];  // TMA staging: T_row, S, T_col
  const ProjRow pr = rows[blockIdx.x];
  const ProjLevel& L = P.L[pr.level];
  const int ro = L.ro, rn = L.rn, co = L.co, cn = L.cn;
  double* Tr = sm;                // rn x ro
  double* Sb = Tr + 64 * kPLd;    // ro x co
  double* Tc = Sb + 64 * kPLd;    // cn x co
  int* wcnt = reinterpret_cast<int*>(Tc + 64 * kPLd);  // kWarps
  int* blist = wcnt + 32;  // blocks to project
  int* clist = blist + P.max_row;  // their block columns
  int* mlist = clist + P.max_row;  // their mirror block (or -1)
  const bool tma = P.tma != 0;
  uint32_t ph_s = 0, ph_t = 0;
  // staging: TMA (one elected thread, mbarrier per buffer) or cp.async groups
  auto issue = [&](int which, double* dst, int node) {
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic accesses of dst before
      tma::mbar_expect_tx(&bar[which], kTileBytes);
      tma_3d(dst, which == 0 ? &P.mT : which == 1 ? &P.mS : &P.mTc, node, &bar[which]);
    }
  };
  auto stage_S = [&](int k) {
    if (tma) issue(1, Sb, blist[k]);
    else stage64(Sb, L.S + int64_t(blist[k]) * L.istride, L.ld_old, ro, co);
  };
  auto stage_Tc = [&](int k) {
    if (tma) issue(2, Tc, clist[k]);
    else stage64(Tc, L.Tc + int64_t(clist[k]) * cn * co, cn, cn, co);
  };
  if (tma) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < 3; ++i) tma::mbar_init(&bar[i], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    issue(0, Tr, pr.row);
  } else {
    stage64(Tr, L.T + int64_t(pr.row) * rn * ro, rn, rn, ro);
  }
  const int b0 = L.rp[pr.row], b1 = L.rp[pr.row + 1];
  // ---- ordered compaction of the row's work list ----
  int nk = 0;
  for (int base = b0; base < b1; base += kThreads) {
    const int b = base + threadIdx.x;
    bool keep = false;
    int c = 0, mb = -1;
    if (b < b1) {
      c = L.ci[b];
      mb = L.mirror ? L.mirror[b] : -1;
      // symmetric level: (col, row) is the transpose of (row, col); the upper
      // block computes both (S_ji' = T_j S_ij^T T_i^T = (T_i S_ij T_j^T)^T)
      keep = !(L.mirror && c < pr.row && mb >= 0);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (cta::lane() == 0) wcnt[cta::warp()] = __popc(bal);
    __syncthreads();
    int off = nk;
    for (int w = 0; w < cta::warp(); ++w) off += wcnt[w];
    int tot = nk;
    for (int w = 0; w < kThreads / 32; ++w) tot += wcnt[w];
    if (keep) {
      const int pos = off + __popc(bal & ((1u << cta::lane()) - 1u));
      blist[pos] = b;
      clist[pos] = c;
      mlist[pos] = (mb >= 0 && c > pr.row) ? mb : -1;
    }
    nk = tot;
    __syncthreads();
  }
  double ss = 0.0;
  if (nk > 0) {
    stage_S(0);
    cp_async_commit();  // {T_row, S_0}
    stage_Tc(0);
    cp_async_commit();  // {T_col,0}
  }
  if (tma) tma::mbar_wait(&bar[0], 0);  // T_row
  auto wait_S = [&](bool two_in_flight) {
    if (tma) {
      tma::mbar_wait(&bar[1], ph_s);
      ph_s ^= 1u;
    } else if (two_in_flight) {
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
  };
  auto wait_Tc = [&](bool two_in_flight) {
    if (tma) {
      tma::mbar_wait(&bar[2], ph_t);
      ph_t ^= 1u;
    } else if (two_in_flight) {
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
  };
  for (int k = 0; k < nk; ++k) {
    wait_S(true);  // S_k (T_col,k may still be in flight)
    __syncthreads();
    const int b = blist[k], mb = mlist[k];
    double* out = L.out + int64_t(b) * L.ostride;
    double* outT = mb >= 0 ? L.out + int64_t(mb) * L.ostride : nullptr;
    double s1 = 0.0;
    double acc[8][2];
    if (P.tri) {
      // triangular T_row: TS by column strips (balanced over the warps; the
      // row strips give warp w 16 - 2w k-steps), through smem over S_k, into
      // the row strips of out.  S_{k+1} then loads after out_k.
      const bool live = ts_cols<true>(Tr, Sb, ro, co, rn, acc);
      __syncthreads();  // S_k consumed
      if (live) ts_store(acc, Sb, rn);
      wait_Tc(false);  // T_col,k
      __syncthreads();
      out_rows<true>(Sb, Tc, out, outT, L.ld_new, co, rn, cn, s1);
      __syncthreads();  // TS, T_col,k consumed
      if (k + 1 < nk) {
        stage_S(k + 1);
        cp_async_commit();
        stage_Tc(k + 1);
        cp_async_commit();
      }
    } else {
      // row strips, TS in registers: S_{k+1} loads under out_k and T_col,{k+1}
      // under TS_{k+1}
      const bool live = ts_strip<false>(Tr, Sb, ro, co, rn, acc);
      __syncthreads();  // S_k consumed
      if (k + 1 < nk) stage_S(k + 1);
      cp_async_commit();
      wait_Tc(true);  // T_col,k
      __syncthreads();
      if (live) out_strip<false>(acc, Tc, out, outT, L.ld_new, co, rn, cn, s1);
      __syncthreads();  // T_col,k consumed
      if (k + 1 < nk) stage_Tc(k + 1);
      cp_async_commit();
    }
    ss += outT ? 2.0 * s1 : s1;
  }
  cp_async_wait<0>();
  // ||S||_F^2 of the projected row, fused (compression.hpp:487, frob_norm_sq)
  if (P.rowsum) {
    double* red = sm;  // Tr is dead
    __syncthreads();
    ss = cta::cta_sum(ss, red);
    if (threadIdx.x == 0) P.rowsum[blockIdx.x] = ss;
  }
}

// nb blocks of bs_new doubles from stride bs_old to stride bs_new (the
// compaction of the coupling pool after the truncation; cudaMemcpy2D moves
// these ~10 KB rows at a fraction of the copy bandwidth).  Ranges of one
// launch never overlap (the host chunks the pool so).  All sizes even.
__global__ void __launch_bounds__(kThreads) k_compact(double* __restrict__ dst, const double* __restrict__ src,
                                                      int64_t bs_new, int64_t bs_old, int64_t nb) {
  const int64_t h = bs_new >> 1;
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const double2* s = reinterpret_cast<const double2*>(src + b * bs_old);
    double2* d = reinterpret_cast<double2*>(dst + b * bs_new);
    for (int64_t e = threadIdx.x; e < h; e += kThreads) __stcs(d + e, __ldcs(s + e));
  }
}

__global__ void k_sumsq(const double* __restrict__ v, int64_t n, double* __restrict__ part) {
  __shared__ double red[16];
  double s = 0.0;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x)
    s += v[e] * v[e];
  s = cta::cta_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// Parent contributions P_r = R^{l-1}_{r/2} E_r^T (kp x kc) for every node of
// level l (the first rows of the weight stack, compression.hpp:228-235).
__global__ void __launch_bounds__(kThreads) k_weights_parent(const double* __restrict__ E, int lde,
                                                             int kc, int kp,
                                                             const double* __restrict__ Rpar,
                                                             double* __restrict__ P) {
  const int64_t r = blockIdx.x;
  cta::gemm_tc<false, true, 1>(P + r * int64_t(kp) * kc, kp, Rpar + (r >> 1) * int64_t(kp) * kp, kp,
                            E + r * int64_t(lde) * kp, lde, kp, kc, kp);
}

// R^l_r = R-factor of [P_r ; S_rb^T ...] (compression.hpp:213-256) by
// streaming TSQR over the UNPADDED stack, ONE WARP PER NODE (no block
// barriers).  Lane L owns stack columns c_t = L + 32 t (t < NCOL); the
// current chunk -- CR consecutive rows of the stack: the parent rows P_r,
// then each transposed coupling block S_rb^T in CR-row pieces (the warp walks
// rows c of S_rb, so every load instruction covers 32 consecutive doubles) --
// lives in registers, the running R (upper triangular, packed column-wise) in
// shared memory.  [R; chunk] is re-triangularised by a structured
// Householder pass whose reflector j touches row j of R plus the chunk.
//
// Per reflector the owner of column j publishes its RAW chunk column and
// alpha = R[j,j] to shared memory; every lane then forms the Householder
// scalars itself (||x||^2, one sqrt, one division) in parallel with its dot
// products and applies the reflector to its own columns.  Arithmetic as
// linalg.hpp:48-75: beta = -sign(alpha) ||x||, tau = (beta - alpha) / beta,
// v = x / (alpha - beta) below the unit entry.
// One reflector of k_weights (see below) on column slots [T0, NCOL).
template <int T0, int NCOL, int CR>
__device__ __forceinline__ void weights_step(double (&B)[NCOL][CR], const double* x, double* xn, double* Rp,
                                             const int (&coff)[NCOL], int lane, int j, int kc) {
  // ||x||^2 and the dot products with the raw column (branch-free: every
  // lane runs the same straight-line code, dead columns get f = 0)
  double w[NCOL][2];
#pragma unroll
  for (int t = T0; t < NCOL; ++t) w[t][0] = w[t][1] = 0.0;
#pragma unroll
  for (int i = 0; i < CR; i += 2) {
    const double2 xx = *reinterpret_cast<const double2*>(x + i);
#pragma unroll
    for (int t = T0; t < NCOL; ++t) {
      w[t][0] = fma(xx.x, B[t][i], w[t][0]);
      w[t][1] = fma(xx.y, B[t][i + 1], w[t][1]);
    }
  }
  // ||x||^2 by a butterfly over the warp (lane L squares rows L, L + 32, ...):
  // off the FP64 pipe, and shorter than the dot-product chains above; every
  // lane ends with the same value
  double q = 0.0;
#pragma unroll
  for (int i = lane; i < CR; i += 32) q = fma(x[i], x[i], q);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const double al = x[CR];
  const double nx = sqrt(fma(al, al, q));
  const double be = al >= 0.0 ? -nx : nx;
  const double am = al - be;
  const double r = 1.0 / (be * am);  // sc = 1/(al-be) = be r, tau = (be-al)/be = -am^2 r
  const double sc = be * r;
  const double tau = -(am * am) * r;
  double f[NCOL];
#pragma unroll
  for (int t = T0; t < NCOL; ++t) {
    const int c = lane + 32 * t;
    f[t] = 0.0;
    if (c > j && c < kc && nx != 0.0) {
      const double d = fma(sc, w[t][0] + w[t][1], Rp[coff[t] + j]) * tau;
      Rp[coff[t] + j] -= d;
      f[t] = sc * d;
    }
    if (c == j && nx != 0.0) {
      Rp[coff[t] + j] = be;
      f[t] = 1.0;  // x == this column: B - x = 0 exactly (it becomes the reflector)
    }
  }
  asm volatile("" ::: "memory");  // re-read x below instead of holding CR more registers
#pragma unroll
  for (int i = 0; i < CR; i += 2) {
    const double2 xx = *reinterpret_cast<const double2*>(x + i);
#pragma unroll
    for (int t = T0; t < NCOL; ++t) {
      B[t][i] = fma(-xx.x, f[t], B[t][i]);
      B[t][i + 1] = fma(-xx.y, f[t], B[t][i + 1]);
    }
  }
  // next owner hands over its updated column
  const int jn = j + 1;
  if (jn < kc && lane == (jn & 31)) {
    if (jn < 32) {
#pragma unroll
      for (int i = 0; i < CR; i += 2) *reinterpret_cast<double2*>(xn + i) = make_double2(B[0][i], B[0][i + 1]);
      xn[CR] = Rp[coff[0] + jn];
    } else {
#pragma unroll
      for (int i = 0; i < CR; i += 2)
        *reinterpret_cast<double2*>(xn + i) = make_double2(B[NCOL - 1][i], B[NCOL - 1][i + 1]);
      xn[CR] = Rp[coff[NCOL - 1] + jn];
    }
  }
}

// nodes (warps) per CTA.  One-warp CTAs, 12 per SM (the register and shared
// memory limit), measured at C3: weight tree 108.2 ms against 112.8 ms for
// 4-warp CTAs x 3 (2 x 6: 112.7, 6 x 2: 113.3).
constexpr int kWWarps = 1;
constexpr int kWCtas = 12;  // resident CTAs per SM (launch bound)
// A work item of k_weights: the stack rows [parent rows if par][blocks b0..b1)
// of node `node`, R written to slot `out` (transposed when the launch's out_t
// is set, so a merge launch can read the partial R's as "blocks").
struct WItem {
  int32_t node, b0, b1, out, par;
};
// Where the blocks of the stacks come from: row stacks hold S_b^T of the
// blocks of a block row (trans = 1); column stacks (non-symmetric matrices,
// the transposed layers of compression.hpp:493-522) hold S_b of the blocks of
// a block column (trans = 0), listed by bidx.  sb: stack rows per block.
struct WSrc {
  const double* S;
  int lds;
  int64_t stride;
  int sb;
  int trans;
  const int32_t* bidx;  // block of stack position p (null: p itself)
};

template <int NCOL, int CR, bool TRANS>
__global__ void __launch_bounds__(32 * kWWarps, kWCtas) k_weights(const double* __restrict__ P, int kc, int kp,
                                                          const __grid_constant__ WSrc src_blocks,
                                                          double* __restrict__ Rout, int out_t,
                                                          const WItem* __restrict__ items, int64_t nitems,
                                                          int* __restrict__ next) {
  constexpr int XS = CR + 2;  // publish slot: raw column, alpha
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int rsz = (((kc * (kc + 1)) / 2 + 1) & ~1);
  double* Rp = sm + wid * (rsz + 2 * XS);  // packed R: column c at c(c+1)/2
  double* xb = Rp + rsz;                   // 2 x XS
  // persistent warps: nodes are claimed in decreasing-work order (LPT)
  for (;;) {
  int idx = 0;
  if (lane == 0) idx = atomicAdd(next, 1);
  idx = __shfl_sync(0xffffffffu, idx, 0);
  if (idx >= nitems) break;
  const WItem it = items[idx];
  const int64_t node = it.node;
  for (int e = lane; e < rsz; e += 32) Rp[e] = 0.0;
  int coff[NCOL];
#pragma unroll
  for (int t = 0; t < NCOL; ++t) {
    const int c = lane + 32 * t;
    coff[t] = (c * (c + 1)) >> 1;
  }
  const int b1 = it.b1;
  int b = it.b0;
  int prow = it.par ? 0 : kp;  // next parent row
  int brow = 0;  // next row of block b's transpose
  double B[NCOL][CR];
  int jg = 0;    // reflector counter (selects the publish slot)
  __syncwarp();
  while (prow < kp || b < b1) {
    // ---- load the next CR-row chunk ----
    if (prow < kp) {
      const int nr = min(CR, kp - prow);
#pragma unroll
      for (int t = 0; t < NCOL; ++t) {
        const int c = lane + 32 * t;
        const double* src = P + node * int64_t(kp) * kc + int64_t(c) * kp + prow;
#pragma unroll
        for (int i = 0; i < CR; ++i) B[t][i] = (c < kc && i < nr) ? src[i] : 0.0;
      }
      prow += nr;
    } else {
      const WSrc& W = src_blocks;
      const int nr = min(CR, W.sb - brow);
      const int64_t bb = W.bidx ? W.bidx[b] : b;
      const int lds = W.lds;
      if (TRANS) {  // stack rows = columns of S_b: row c of the block, coalesced over lanes
#pragma unroll
        for (int t = 0; t < NCOL; ++t) {
          const int c = lane + 32 * t;
          const double* src = W.S + bb * W.stride + c + int64_t(brow) * lds;
#pragma unroll
          for (int i = 0; i < CR; ++i) {
            B[t][i] = (c < kc && i < nr) ? __ldcs(src) : 0.0;
            src += lds;
          }
        }
      } else {  // stack rows = rows of S_b: column c of the block
#pragma unroll
        for (int t = 0; t < NCOL; ++t) {
          const int c = lane + 32 * t;
          const double* src = W.S + bb * W.stride + int64_t(c) * lds + brow;
#pragma unroll
          for (int i = 0; i < CR; ++i) B[t][i] = (c < kc && i < nr) ? __ldcs(src + i) : 0.0;
        }
      }
      brow += nr;
      if (brow >= W.sb) {
        brow = 0;
        ++b;
      }
    }
    if (lane == 0) {  // column 0 opens the chunk
      double* x = xb + (jg & 1) * XS;
#pragma unroll
      for (int i = 0; i < CR; i += 2) *reinterpret_cast<double2*>(x + i) = make_double2(B[0][i], B[0][i + 1]);
      x[CR] = Rp[0];
    }
    __syncwarp();
#pragma unroll 1
    for (int j = 0; j < kc; ++j, ++jg) {
      const double* x = xb + (jg & 1) * XS;
      double* xn = xb + ((jg + 1) & 1) * XS;
      // column slot 0 holds only dead columns once j >= 32: skip it (uniform)
      if (NCOL == 2 && j >= 32)
        weights_step<1, NCOL, CR>(B, x, xn, Rp, coff, lane, j, kc);
      else
        weights_step<0, NCOL, CR>(B, x, xn, Rp, coff, lane, j, kc);
      __syncwarp();
    }
  }
  // R with non-negative diagonal (linalg.hpp:100-113); row i by lane, so the
  // stores of one column are coalesced
  double* Ro = Rout + int64_t(it.out) * kc * kc;
  for (int cc = 0; cc < kc; ++cc) {
    const int ccoff = (cc * (cc + 1)) >> 1;
    for (int i = lane; i < kc; i += 32) {
      const double v = i <= cc ? Rp[ccoff + i] : 0.0;
      const double o = Rp[((i * (i + 1)) >> 1) + i] < 0.0 ? -v : v;
      if (out_t)
        Ro[cc + int64_t(i) * kc] = o;
      else
        Ro[i + int64_t(cc) * kc] = o;
    }
  }
  __syncwarp();
  }
}

// Truncation SVDs (svd_truncated_batched, batch.hpp:107-140 / linalg.hpp:142-232):
// left singular vectors U (rows x s), singular values, and the count
// #{sigma_j >= eps sigma_1} of W (rows x cols), s = min(rows, cols), in three
// stages over the whole batch:
//   A  (256 threads)  precondition (Drmac-Veselic):
//        tall  W = Q1 R1 (Householder), R1^T = Q2 R2  ->  J = R2^T,  U = Q1 [U_J; 0]
//        wide  W^T = Q1 R1                            ->  J = R1^T,  U = U_J
//      J (s x s) and Q1's reflectors go to global scratch;
//   B  (64 threads, k_jacobi64)  one-sided Jacobi on J with lane c owning
//      column c in registers (no reductions: dot products are lane-local, the
//      partner column is read from shared memory), sigma = column norms,
//      stable descending sort, U_J normalised -> the top rows of U;
//   C  (256 threads, tall only)  U = Q1 [U_J; 0] by compact WY on the FP64
//      tensor cores (apply_q_wy).
// Same singular values and subspaces as the reference's Jacobi on W (which
// takes 10-26 sweeps on these graded spectra; J converges in ~6); columns of U
// may differ in sign.  The Jacobi rule (|a_pq| <= 16 eps sqrt(a_pp a_qq) or
// a_pq == 0), 60-sweep cap, sigma = column norms and stable descending sort
// are the reference's; the pair order is the parallel round-robin ordering.
struct SvdScratch {
  double tau[64];
  double tau2[64];
  double xb[cta::kHhScratch];  // householder publish slots
};
constexpr int kSvdScratch = int((sizeof(SvdScratch) + 15) / 16) * 2;  // in doubles, 16 B aligned

// Stage A on W (rows x cols, smem, ld rows; destroyed).  X: smem >= s*s and
// >= cols*rows.  Writes J (s x s, ld s) and, when tall, the factored Q1 (V:
// rows x cols, ld rows; tau: cols) to global.
template <int RQW, int G>  // W's QR: G threads per column, RQW rows each (rows <= G RQW)
__device__ void svd_precondition(double* W, int rows, int cols, double* X, double* J, double* V,
                                 double* tau, SvdScratch& sc) {
  const int s = rows < cols ? rows : cols;
  if (s == 0) return;
  if (rows >= cols) {
    const int c = cols;
    cta::householder_regs<RQW, G>(W, rows, rows, c, sc.tau, sc.xb);
    for (int e = threadIdx.x; e < rows * c; e += blockDim.x) V[e] = W[e];
    for (int j = threadIdx.x; j < c; j += blockDim.x) tau[j] = sc.tau[j];
    // X = R1^T (c x c, lower), then QR of it: R2 in the upper triangle
    for (int e = threadIdx.x; e < c * c; e += blockDim.x) {
      const int j = e / c, i = e - j * c;
      X[i + j * c] = i >= j ? W[j + i * rows] : 0.0;
    }
    __syncthreads();
    cta::householder_regs<64 / G, G>(X, c, c, c, sc.tau2, sc.xb);
    for (int e = threadIdx.x; e < c * c; e += blockDim.x) {  // J = R2^T
      const int j = e / c, i = e - j * c;
      J[i + j * c] = i >= j ? X[j + i * c] : 0.0;
    }
  } else {
    const int r = rows;
    double* Gt = X;  // W^T (cols x r)
    for (int e = threadIdx.x; e < cols * r; e += blockDim.x) {
      const int j = e / cols, i = e - j * cols;
      Gt[i + j * cols] = W[j + i * rows];
    }
    __syncthreads();
    cta::householder_regs<64 / G, G>(Gt, cols, cols, r, sc.tau, sc.xb);  // cols <= 64 rows
    for (int e = threadIdx.x; e < r * r; e += blockDim.x) {  // J = R1^T
      const int j = e / r, i = e - j * r;
      J[i + j * r] = i >= j ? Gt[j + i * cols] : 0.0;
    }
  }
  __syncthreads();
}

__device__ void check_finite(const double* W, int n, int* bad) {
  for (int e = threadIdx.x; e < n; e += blockDim.x)
    if (!isfinite(W[e])) *bad = 1;
}

// Stage A, leaves: W = U R^T (m x k) (compression.hpp:285-300).
__global__ void __launch_bounds__(kThreads) k_trunc_leaf_pre(const double* __restrict__ leaf, int ldm, int m,
                                                             int k, const double* __restrict__ R,
                                                             double* __restrict__ Jout, double* __restrict__ Vout,
                                                             double* __restrict__ tauout, int* __restrict__ bad) {
  extern __shared__ double sm[];
  const int s = m < k ? m : k;
  SvdScratch& sc = *reinterpret_cast<SvdScratch*>(sm);
  double* W = sm + kSvdScratch;  // m x k
  double* X = W + m * k;         // >= s s, >= k m
  const int64_t i = blockIdx.x;
  if (kLevelPrefetch && threadIdx.x == 0 && i + 2 * nsm() < gridDim.x) {  // one wave ahead (2 CTAs/SM)
    const int64_t in = i + 2 * nsm();
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(leaf + in * int64_t(ldm) * k),
                 "r"(uint32_t(ldm * k * 8)) : "memory");
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(R + in * int64_t(k) * k), "r"(uint32_t(k * k * 8))
                 : "memory");
  }
  cta::gemm_tc<false, true, 2>(W, m, leaf + i * int64_t(ldm) * k, ldm, R + i * int64_t(k) * k, k, m, k, k);
  __syncthreads();
  check_finite(W, m * k, bad);
  svd_precondition<16, 4>(W, m, k, X, Jout + i * int64_t(s) * s, Vout + i * int64_t(m) * k, tauout + i * 64, sc);
}

// Stage A, parent p: Z = [Tt_c E_c] (2kt_c x kp), W = Z R^{l-1,T} (:327-376).
__global__ void __launch_bounds__(kLevelThreads) k_trunc_level_pre(
    const double* __restrict__ E, int lde, int kc, int kp, int ktc, const double* __restrict__ Tt,
    const double* __restrict__ Rp, double* __restrict__ Zout, double* __restrict__ Jout,
    double* __restrict__ Vout, double* __restrict__ tauout, int* __restrict__ bad) {
  extern __shared__ double sm[];
  const int zr = 2 * ktc;
  const int s = zr < kp ? zr : kp;
  SvdScratch& sc = *reinterpret_cast<SvdScratch*>(sm);
  double* W = sm + kSvdScratch;  // zr x kp
  double* X = W + zr * kp;       // >= s s, >= kp zr
  const int64_t p = blockIdx.x;
  const int64_t es = int64_t(lde) * kp;
  double* Z = Zout + p * int64_t(zr) * kp;  // Z lives in global memory (L2)
  if (kLevelPrefetch && threadIdx.x == 0) {  // one wave ahead, as in k_orth_level
    const int64_t pn = p + nsm();
    if (pn < gridDim.x) {
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Tt + 2 * pn * int64_t(ktc) * kc),
                   "r"(uint32_t(2 * ktc * kc * 8)) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(E + 2 * pn * es), "r"(uint32_t(2 * es * 8))
                   : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Rp + pn * int64_t(kp) * kp),
                   "r"(uint32_t(kp * kp * 8)) : "memory");
    }
  }
  for (int ci = 0; ci < 2; ++ci) {
    const int64_t c = 2 * p + ci;
    cta::gemm_tc<false, false>(Z + ci * ktc, zr, Tt + c * int64_t(ktc) * kc, ktc, E + c * es, lde, ktc, kp, kc);
  }
  __syncthreads();
  cta::gemm_tc<false, true, 2>(W, zr, Z, zr, Rp + p * int64_t(kp) * kp, kp, zr, kp, kp);
  __syncthreads();
  check_finite(W, zr * kp, bad);
  if (zr <= 64)
    svd_precondition<8, 8>(W, zr, kp, X, Jout + p * int64_t(s) * s, Vout + p * int64_t(zr) * kp, tauout + p * 64, sc);
  else
    svd_precondition<16, 8>(W, zr, kp, X, Jout + p * int64_t(s) * s, Vout + p * int64_t(zr) * kp, tauout + p * 64, sc);
}

// Stage B: one-sided Jacobi on J (r x r, r <= 64), one 64-thread CTA per
// matrix, lane c owns column c in registers.  Per round-robin round every lane
// publishes its column to shared memory, reads its partner's, forms the three
// dot products itself (both lanes of a pair get bitwise the same values) and
// rotates its own column.  Output: U_J (normalised, sorted) into the top r
// rows of U (ld ldu), sigma (s = r values), atomicMax of the truncation rank.
__global__ void __launch_bounds__(64) k_jacobi64(const double* __restrict__ Jall, int r,
                                                 double* __restrict__ Uall, int ldu, int64_t ustride,
                                                 double* __restrict__ sig_all, double eps,
                                                 int* __restrict__ kmax) {
  constexpr int LD = 66;  // even: 16-byte aligned columns (128-bit, conflict-free quarter-warps)
  __shared__ __align__(16) double cols[64 * LD];
  __shared__ double nrm2[64];
  __shared__ double nrm[64];
  __shared__ double dpart[64];  // half dot products of the round (rows of this lane's half)
  __shared__ int flag, big;
  const int c = threadIdx.x;
  const int n = r + (r & 1);  // zero pad column when odd
  const double* J = Jall + blockIdx.x * int64_t(r) * r;
  double g[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) g[i] = (c < r && i < r) ? J[i + c * r] : 0.0;
  // published copy of every column and its squared norm (the reference
  // recomputes the norms at every pair visit; so does this kernel, once per
  // rotated column, and both lanes of a pair read the same published values)
  auto norm2 = [&]() {
    double t0 = 0.0, t1 = 0.0;
#pragma unroll
    for (int i = 0; i < 64; i += 2) {
      t0 = fma(g[i], g[i], t0);
      t1 = fma(g[i + 1], g[i + 1], t1);
    }
    return t0 + t1;
  };
  auto publish = [&](double a) {
    double2* dst = reinterpret_cast<double2*>(cols + c * LD);
#pragma unroll
    for (int i = 0; i < 64; i += 2) dst[i / 2] = make_double2(g[i], g[i + 1]);
    nrm2[c] = a;
  };
  double a = norm2();
  if (c < n) publish(a);
  if (c == 0) flag = big = 0;
  const double tol = 2.220446049250313e-16 * 16.0;
  // A sweep whose rotations all had |a_pq| <= tol_q sqrt(a_pp a_qq) is the
  // last one that rotates: the next would find |a_pq| ~ (that)^2 <= tol/16 on
  // every pair (quadratic convergence) and only confirm it, so it is skipped.
  const double tol_q = 0.25 * sqrt(tol);
  const int m1 = n - 1;
  for (int sweep = 0; sweep < 60 && r > 1; ++sweep) {
    for (int rd = 0; rd < m1; ++rd) {
      __syncthreads();  // this round's columns are published
      bool rot = false;
      // round-robin (circle) partner of column c in round rd
      const int pt = c == m1 ? rd : (c == rd ? m1 : (2 * rd - c + 2 * m1) % m1);
      const bool is_p = c < pt;
      if (c < n) {
        // the pair's dot product in two halves: column p's lane reads rows
        // 0..31 of the partner, column q's lane rows 32..63 (half the shared
        // memory reads of the round's dot products; the kernel is bound by
        // them).  Keeping that half in registers for the rotation as well:
        // 243 registers, 4 CTAs/SM instead of 6, compress 252.7 -> 255.2 ms.
        const int h0 = is_p ? 0 : 32;
        const double2* pc = reinterpret_cast<const double2*>(cols + pt * LD + h0);
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const double2 x = pc[i / 2];
          d0 = fma(is_p ? g[i] : g[i + 32], x.x, d0);
          d1 = fma(is_p ? g[i + 1] : g[i + 33], x.y, d1);
        }
        dpart[c] = d0 + d1;
      }
      __syncthreads();  // both halves of every pair's dot product
      if (c < n) {
        const double d = is_p ? dpart[c] + dpart[pt] : dpart[pt] + dpart[c];  // (rows 0..31) + (rows 32..63)
        const double2* pc = reinterpret_cast<const double2*>(cols + pt * LD);
        const double b = nrm2[pt];
        const double ap = is_p ? a : b, aq = is_p ? b : a;
        // skip rule of linalg.hpp:155-160 (sqrt(a) sqrt(b): no underflow)
        const double sab = sqrt(ap) * sqrt(aq);
        if (!(fabs(d) <= tol * sab || d == 0.0)) {
          rot = true;
          flag = 1;
          if (fabs(d) > tol_q * sab) big = 1;
          const double z = (aq - ap) / (2.0 * d);
          const double t = (z >= 0.0 ? 1.0 : -1.0) / (fabs(z) + hypot(1.0, z));
          const double cs = 1.0 / sqrt(1.0 + t * t);
          const double sn = cs * t;
          // new_p = cs u - sn w, new_q = sn u + cs w  (u = column p, w = column q)
          const double fp = is_p ? -sn : sn;
#pragma unroll
          for (int i = 0; i < 64; i += 2) {
            const double2 x = pc[i / 2];
            g[i] = fma(cs, g[i], fp * x.x);
            g[i + 1] = fma(cs, g[i + 1], fp * x.y);
          }
          a = norm2();
        }
      }
      __syncthreads();  // everyone has read the partners
      if (rot) publish(a);
    }
    __syncthreads();
    const int f = flag, fb = big;
    __syncthreads();
    if (c == 0) flag = big = 0;
#ifdef H2B_SWEEP_HIST
    if (c == 0 && (!f || !fb || sweep == 59)) atomicAdd(&cta::g_sweep_hist[(f && fb) ? 60 : sweep], 1);
#endif
    if (!f || !fb) break;
  }
  // sigma = column norms, stable descending order
  const double sg = sqrt(norm2());
  nrm[c] = c < n ? sg : -1.0;
  __syncthreads();
  int pos = 0;
  double smax = 0.0;
  for (int i = 0; i < n; ++i) {
    const double v = nrm[i];
    pos += (v > sg) || (v == sg && i < c);
    smax = fmax(smax, v);
  }
  const bool keep = smax > 0.0 && c < n && sg >= eps * smax && pos < r;
  const int rank = __syncthreads_count(keep);
  if (c < n && pos < r) {
    sig_all[blockIdx.x * int64_t(r) + pos] = sg;
    double* U = Uall + blockIdx.x * ustride + int64_t(pos) * ldu;
    const double inv = sg > 0.0 ? 1.0 / sg : 0.0;
#pragma unroll
    for (int i = 0; i < 64; ++i)
      if (i < r) U[i] = sg > 0.0 ? g[i] * inv : 0.0;
  }
  if (c == 0) atomicMax(kmax, rank);
}

// Stage C (tall): U = Q1 [U_J; 0] (rows x s) in place in global memory.
__global__ void __launch_bounds__(kThreads) k_svd_apply(const double* __restrict__ Vall, const double* __restrict__ tauall,
                                                        int rows, int c, double* __restrict__ Uall) {
  extern __shared__ double sm[];
  double* V = sm;            // rows x c
  double* Zw = V + rows * c; // c x c
  double* tau = Zw + c * c;  // 64
  const int64_t i = blockIdx.x;
  const double* Vg = Vall + i * int64_t(rows) * c;
  for (int e = threadIdx.x; e < rows * c; e += blockDim.x) V[e] = Vg[e];
  for (int j = threadIdx.x; j < c; j += blockDim.x) tau[j] = tauall[i * 64 + j];
  __syncthreads();
  cta::apply_q_wy(V, rows, rows, c, tau, Uall + i * int64_t(rows) * c, rows, c, Zw);
}

// T^q = Q^T U_old (kt x k), new leaf = Q (m x kt), discarded energy (:309-324).
__global__ void __launch_bounds__(kThreads) k_trunc_leaf_apply(const double* __restrict__ leaf, int ldm,
                                                               int m, int k, int s, int kt,
                                                               const double* __restrict__ Uq,
                                                               const double* __restrict__ sig,
                                                               double* __restrict__ Tq,
                                                               double* __restrict__ newleaf, int ldn,
                                                               double* __restrict__ energy) {
  const int64_t i = blockIdx.x;
  const double* Q = Uq + i * int64_t(m) * s;
  if (kt > 0)
    cta::gemm_tc<true, false>(Tq + i * int64_t(kt) * k, kt, Q, m, leaf + i * int64_t(ldm) * k, ldm, kt, k, m);
  double* nl = newleaf + i * int64_t(ldn) * kt;
  for (int e = threadIdx.x; e < ldn * kt; e += blockDim.x) {
    const int j = e / ldn, r = e - j * ldn;
    nl[e] = r < m ? Q[r + int64_t(j) * m] : 0.0;
  }
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int j = kt; j < s; ++j) acc += sig[i * s + j] * sig[i * s + j];
    energy[i] = acc;
  }
}

// T^{l-1}_p = Q^T Z (kt_p x kp); new transfers = Q row blocks (:382-415).
__global__ void __launch_bounds__(kThreads) k_trunc_level_apply(
    int ktc, int kp, int s, int ktp, const double* __restrict__ Zin, const double* __restrict__ Uin,
    const double* __restrict__ sig, double* __restrict__ Tp, double* __restrict__ Enew, int ldn,
    double* __restrict__ energy) {
  const int zr = 2 * ktc;
  const int64_t p = blockIdx.x;
  const double* Q = Uin + p * int64_t(zr) * s;
  if (ktp > 0)
    cta::gemm_tc<true, false>(Tp + p * int64_t(ktp) * kp, ktp, Q, zr, Zin + p * int64_t(zr) * kp, zr, ktp,
                           kp, zr);
  for (int ci = 0; ci < 2; ++ci) {
    double* dst = Enew + (2 * p + ci) * int64_t(ldn) * ktp;
    for (int e = threadIdx.x; e < ldn * ktp; e += blockDim.x) {
      const int j = e / ldn, r = e - j * ldn;
      dst[e] = r < ktc ? Q[ci * ktc + r + int64_t(j) * zr] : 0.0;
    }
  }
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int j = ktp; j < s; ++j) acc += sig[p * s + j] * sig[p * s + j];
    energy[p] = acc;
  }
}

// ------------------------------------------------------------------ host helpers
template <class K>
void set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    H2B_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

constexpr size_t kSmemCap = 227 * 1024;

void check_smem(size_t bytes, const char* what) {
  if (bytes > kSmemCap) throw Error(H2B_UNSUPPORTED, std::string(what) + ": shared-memory footprint too large");
}

struct Flops {
  double gemm(double c, double m, double n, double k) { return 2.0 * m * n * k * c; }
  double qr(double c, double r, double k) { return 2.0 * k * k * (r - k / 3.0) * c; }
  double svd(double c, double r, double k) {
    const double s = std::min(r, k);
    return (2.0 * s * s * (std::max(r, k) - s / 3.0) + 60.0 * s * s * s) * c;
  }
};

struct Timer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  explicit Timer(cudaStream_t st) : s(st) {
    H2B_CUDA(cudaEventCreate(&a));
    H2B_CUDA(cudaEventCreate(&b));
    H2B_CUDA(cudaEventRecord(a, s));
  }
  double stop() {
    H2B_CUDA(cudaEventRecord(b, s));
    H2B_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    H2B_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
  }
};

// Level-concatenated pool of per-node (rows[l] x cols[l]) matrices, ld = rows,
// carved from the compression workspace.
struct TreePool {
  double* p = nullptr;
  std::vector<int64_t> off;
  std::vector<int> rows, cols;
  static size_t need(const Matrix& A, const std::vector<int>& r, const std::vector<int>& c) {
    size_t t = 0;
    for (int l = 0; l <= A.q; ++l) t += size_t(A.nodes(l)) * r[l] * c[l];
    return std::max<size_t>(1, t);
  }
  void alloc(const Matrix& A, const std::vector<int>& r, const std::vector<int>& c, double* base) {
    rows = r;
    cols = c;
    off.assign(A.q + 2, 0);
    for (int l = 0; l <= A.q; ++l) off[l + 1] = off[l] + A.nodes(l) * int64_t(r[l]) * c[l];
    p = base;
  }
  double* at(int l) { return p + off[l]; }
};

// Bump allocator over one workspace region: the phases size their scratch up
// front instead of allocating per level.
struct Arena {
  double* base = nullptr;
  size_t cap = 0, off = 0;
  void reserve(double* b, size_t doubles) {
    base = b;
    cap = doubles;
    off = 0;
  }
  template <class T>
  T* take(size_t n) {
    const size_t d = ((n * sizeof(T) + 255) / 256) * 32;  // 256-byte granules, in doubles
    if (off + d > cap) throw Error(H2B_CUDA_ERROR, "scratch arena overflow");
    T* p = reinterpret_cast<T*>(base + off);
    off += d;
    return p;
  }
  static size_t need(size_t n, size_t elem) { return ((n * elem + 255) / 256) * 32; }
};

// Per-device cache of compression workspaces: plain cudaMalloc, grow-only,
// reused by the next compress() (mapping tens of GB of fresh device memory,
// or re-mapping it through a stream-ordered pool, costs 0.1-5 s -- more than
// the compression itself); h2b_release_cached_memory frees it.  Concurrent
// compressions (one per partition handle) check out separate buffers.
struct WsCache {
  std::mutex mu;
  std::vector<std::vector<DevBuf<double>>> free;  // per device
};
WsCache& ws_cache() {
  static WsCache c;
  return c;
}
DevBuf<double> ws_checkout(int dev, size_t doubles) {
  DevBuf<double> b;
  {
    std::lock_guard<std::mutex> lk(ws_cache().mu);
    auto& fr = ws_cache().free;
    if (int(fr.size()) <= dev) fr.resize(dev + 1);
    auto& v = fr[dev];
    if (!v.empty()) {
      auto it = std::max_element(v.begin(), v.end(), [](const DevBuf<double>& x, const DevBuf<double>& y) {
        return x.n < y.n;
      });
      b = std::move(*it);
      v.erase(it);
    }
  }
  if (b.n < doubles) {
    b.release();
    b.alloc(doubles + doubles / 8);  // headroom for the next, slightly larger matrix
  }
  return b;
}
void ws_return(int dev, DevBuf<double>&& b) {
  std::lock_guard<std::mutex> lk(ws_cache().mu);
  auto& fr = ws_cache().free;
  if (int(fr.size()) <= dev) fr.resize(dev + 1);
  fr[dev].push_back(std::move(b));
}
struct Workspace {
  int dev;
  DevBuf<double> buf;
  double* trees;  // region A: To, later Tt
  double* rtree;  // region B: R
  double* arena;  // region C: per-phase scratch
  size_t arena_cap;
  ~Workspace() {
    if (buf.p) ws_return(dev, std::move(buf));
  }
};

// Subtree partition of the compression: 2^s ranks, this one
// owns the nodes [own_begin(l), own_end(l)) of every level l >= s (levels < s
// replicated, computed redundantly).  Trees indexed by global node (T, R, Tt)
// are allocated full-size; leaf / transfer pools are the handle's local ones.
struct Part {
  const h2b_comm* comm = nullptr;
  int s = 0, g = 0;
  bool dist() const { return comm != nullptr; }
  // slice of level l >= s owned by this rank: contiguous in a per-level pool
  void allgather(double* buf, int64_t count, cudaStream_t st) const {
    if (!comm || count == 0) return;
    H2B_CUDA(cudaStreamSynchronize(st));
    if (comm->allgather(comm->ctx, buf, count) != 0) throw Error(H2B_CUDA_ERROR, "communicator: allgather failed");
  }
  void max_i32(int32_t* v, int n) const {
    if (comm && comm->allreduce_max_i32(comm->ctx, v, n) != 0)
      throw Error(H2B_CUDA_ERROR, "communicator: allreduce(max) failed");
  }
  void sum_f64(double* v, int n) const {
    if (comm && comm->allreduce_sum_f64(comm->ctx, v, n) != 0)
      throw Error(H2B_CUDA_ERROR, "communicator: allreduce(sum) failed");
  }
  // replicated levels are counted by rank 0 only in global sums
  bool counts(int l) const { return !comm || l >= s || g == 0; }
};

// ---------------------------------------------------------------- phases
// on_t(l) (optional): called once T(l) is final in stream order on s.
using LevelHook = std::function<void(int)>;
void orthogonalize(Matrix& A, TreePool& T, cudaStream_t s, Flops& fl, double& flops, const Part& pt,
                   double* tree_mem, const LevelHook& on_t_user = nullptr) {
  const int q = A.q, m = A.m, kq = A.rank[q];
  // partitioned: T(l) of a level >= s is complete (remote column bases
  // included) only after the all-gather below, so its hook waits for it
  std::vector<int> deferred;
  bool gathered = !pt.dist();
  const LevelHook on_t = !on_t_user ? LevelHook() : LevelHook([&](int l) {
    if (!gathered && l >= pt.s)
      deferred.push_back(l);
    else
      on_t_user(l);
  });
  require(m >= kq, "orthogonalize_basis: leaf_dim must be >= leaf rank");
  T.alloc(A, A.rank, A.rank, tree_mem);
  const int64_t nl = A.nodes(q);
  if (kq > 0) {
    const size_t sm = (2 * size_t(m) * kq + size_t(kq) * kq + 64 + kXb) * sizeof(double) + 64 * sizeof(int);
    check_smem(sm, "orthogonalize");
    set_smem(k_orth_leaf, sm);
    if (A.own_count(q) > 0)
      k_orth_leaf<<<unsigned(A.own_count(q)), kThreads, sm, s>>>(A.leaf.p, A.ldm, m, kq,
                                                                 T.at(q) + A.own_begin(q) * int64_t(kq) * kq);
    H2B_CUDA(cudaGetLastError());
  }
  if (on_t) on_t(q);
  flops += fl.qr(double(nl), m, kq);
  auto level = [&](int l) {
    const int kc = A.rank[l], kp = A.rank[l - 1];
    const int64_t np = A.nodes(l - 1);
    flops += fl.gemm(double(A.nodes(l)), kc, kp, kc) + fl.qr(double(np), 2 * kc, kp);
    require(2 * kc >= kp, "qr_batched: requires rows >= cols");
    if (kp == 0) {
      if (on_t) on_t(l - 1);
      return;
    }
    const size_t sm = (2 * size_t(2 * kc) * kp + size_t(kp) * kp + 64 + kXb) * sizeof(double) + 64 * sizeof(int);
    check_smem(sm, "orthogonalize");
    set_smem(k_orth_level, sm);
    // parents [p0, p1) at level l-1; children 2p0.. in the (local) transfer pool
    const int64_t p0 = A.own_begin(l - 1), p1 = A.own_end(l - 1);
    k_orth_level<<<unsigned(p1 - p0), kLevelThreads, sm, s>>>(
        A.transfer.p + A.tr_off[l] + (2 * p0 - A.tr_begin(l)) * A.tr_stride(l), A.ld(l), kc, kp,
        T.at(l) + 2 * p0 * int64_t(kc) * kc, T.at(l - 1) + p0 * int64_t(kp) * kp);
    H2B_CUDA(cudaGetLastError());
    if (on_t) on_t(l - 1);
  };
  for (int l = q; l > pt.s; --l) level(l);
  // the projection tree of the partitioned levels: remote column bases for
  // the projection, the level-s roots for the replicated top
  for (int l = pt.s; l <= q; ++l)
    pt.allgather(T.at(l), (int64_t(1) << (l - pt.s)) * A.rank[l] * A.rank[l], s);
  gathered = true;
  for (int l : deferred) on_t_user(l);
  for (int l = pt.s; l >= 1; --l) level(l);
}

// Projection S <- T_row S T_col^T of every coupling level (project_coupling,
// compression.hpp:130-169), split so that it can run level by level on a
// side stream while the orthogonalization / truncation chains (which produce
// T level by level, bottom-up) continue on the main stream:
//   ProjRows        the block rows with work (structure only: on symmetric
//                   levels the rows holding an upper block), uploaded once;
//   project_level   one k_project launch for level l once T(l) is final;
//   project_finish  after every level: relabel the layers and, for the
//                   rectangular T of the truncation, compact the pool.
// Square T (orthogonalization) projects in place.  Rectangular T shrinks
// every block: each block is written at the start of its old slot (ld =
// pad2(new rank)), then the compaction moves the blocks down in block-order
// chunks -- chunk k's destination ends where chunk k+1's source starts or
// earlier (every block only shrinks), so nothing unread is clobbered and no
// second coupling pool is ever allocated.
struct ProjRows {
  std::vector<int64_t> off;  // level l's rows: [off[l], off[l + 1])
  ProjRow* d = nullptr;
  double* rsum = nullptr;    // per row: sum of squares of the projected blocks
  std::vector<ProjRow> h;
  int max_row = 1;
  static size_t need(const Matrix& A) {
    size_t r = 1;
    for (int l = 0; l <= A.q; ++l) r += size_t(A.cpl[l].rows);
    return Arena::need(r, sizeof(ProjRow)) + Arena::need(r, sizeof(double));
  }
};

const int32_t* mirror_of(const Matrix& A, int l) {
  return (A.mirror_sym[l] && l < int(A.value_sym.size()) && A.value_sym[l]) ? A.mirror.p + A.mirror_off[l]
                                                                           : nullptr;
}

// sym_T: the row and column projection trees are the same tree, so a
// symmetric level's lower blocks are the upper ones' transposes.
void project_rows(const Matrix& A, Arena& ar, ProjRows& R, cudaStream_t s, bool sym_T = true) {
  require(A.mirror_ready, "project_coupling: mirror map missing");
  const int q = A.q;
  R.off.assign(q + 2, 0);
  R.h.clear();
  R.max_row = 1;
  for (int l = 0; l <= q; ++l) {
    const Layer& L = A.cpl[l];
    R.off[l] = int64_t(R.h.size());
    R.max_row = std::max(R.max_row, L.max_row);
    const bool mir = sym_T && mirror_of(A, l) != nullptr;
    for (int64_t r = 0; r < L.rows && L.nb > 0; ++r) {
      bool any = false;
      for (int32_t b = L.h_rp[r]; b < L.h_rp[r + 1] && !any; ++b) any = !mir || L.h_ci[b] > r;
      if (any) R.h.push_back({l, int32_t(r)});
    }
  }
  R.off[q + 1] = int64_t(R.h.size());
  ar.off = 0;
  R.d = ar.take<ProjRow>(std::max<size_t>(1, R.h.size()));
  R.rsum = ar.take<double>(std::max<size_t>(1, R.h.size()));
  if (!R.h.empty())
    H2B_CUDA(cudaMemcpyAsync(R.d, R.h.data(), R.h.size() * sizeof(ProjRow), cudaMemcpyHostToDevice, s));
  H2B_CUDA(cudaStreamSynchronize(s));  // (pageable source)
}

// Level l with T(l) (T.rows[l] x T.cols[l] per node) on stream st.
// Level l with T(l) (row projections, T.rows[l] x T.cols[l] per node) and
// Tc(l) (column projections; the same tree when symmetric) on stream st.
// out / ostride: where the projected blocks go (default: the old slots).
void project_level(const Matrix& A, const TreePool& T, const TreePool& Tc, const ProjRows& R, int l, bool tri,
                   bool want_sum, Flops& fl, double& flops, const Part& pt, cudaStream_t st, bool sym_T = true,
                   double* out = nullptr, int64_t ostride = 0) {
  const Layer& L = A.cpl[l];
  const int rn = T.rows[l], ro = T.cols[l], cn = Tc.rows[l], co = Tc.cols[l];
  if (L.nb == 0) return;
  require(ro == L.br && co == L.bc, "project_coupling: dim mismatch");
  if (pt.counts(l)) flops += fl.gemm(double(L.nb), rn, co, ro) + fl.gemm(double(L.nb), rn, cn, co);
  const int64_t n = R.off[l + 1] - R.off[l];
  if (rn == 0 || cn == 0 || n == 0) return;
  ProjTable P{};
  P.tri = tri ? 1 : 0;
  P.max_row = R.max_row;
  P.rowsum = want_sum ? R.rsum + R.off[l] : nullptr;
  ProjLevel& d = P.L[l];
  d.S = L.val;
  d.rp = L.rp;
  d.ci = L.ci;
  d.mirror = sym_T ? mirror_of(A, l) : nullptr;
  d.T = const_cast<TreePool&>(T).at(l);
  d.Tc = const_cast<TreePool&>(Tc).at(l);
  d.ro = ro;
  d.rn = rn;
  d.co = co;
  d.cn = cn;
  d.ld_old = L.ld;
  d.ld_new = pad2(rn);
  d.istride = L.block_stride();
  d.out = out ? out : L.val;  // default: in the old slots
  d.ostride = out ? ostride : L.block_stride();
  // TMA staging when every tile source is a 16-byte aligned pool of even-ld
  // blocks (odd ranks keep the 8-byte cp.async path)
  const auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  const int64_t nT = A.nodes(l), nTc = A.col_basis().nodes(l);
  if (kProjTma && (L.ld & 1) == 0 && (rn & 1) == 0 && (cn & 1) == 0 && al(d.S) && al(d.T) && al(d.Tc) &&
      L.nb > 0) {
    tma::encode_blocks3d(&P.mS, d.S, uint64_t(L.ld), uint64_t(co), uint64_t(L.nb), kPLd, 64);
    tma::encode_blocks3d(&P.mT, d.T, uint64_t(rn), uint64_t(ro), uint64_t(std::max<int64_t>(1, nT)), kPLd, 64);
    tma::encode_blocks3d(&P.mTc, d.Tc, uint64_t(cn), uint64_t(co), uint64_t(std::max<int64_t>(1, nTc)), kPLd, 64);
    P.tma = 1;
  }
  const size_t smax = size_t(3) * 64 * kPLd * sizeof(double) + (32 + 3 * size_t(P.max_row)) * sizeof(int);
  check_smem(smax, "project_coupling");
  set_smem(k_project, smax);
  k_project<<<unsigned(n), kThreads, smax, st>>>(P, R.d + R.off[l]);
  H2B_CUDA(cudaGetLastError());
}

// ||S||_F^2 of the projected coupling (replicated top levels: rank 0 only);
// the projection launches must be complete.
double project_rowsum(const ProjRows& R, const Part& pt, cudaStream_t s) {
  std::vector<double> h(R.h.size());
  if (!R.h.empty())
    H2B_CUDA(cudaMemcpyAsync(h.data(), R.rsum, R.h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  H2B_CUDA(cudaStreamSynchronize(s));
  double acc = 0.0;
  for (size_t i = 0; i < R.h.size(); ++i)
    if (pt.counts(R.h[i].level)) acc += h[i];
  return acc;
}

// After every level's launch completed (stream order on s): compaction of the
// shrunken blocks (not in_place) and the new layer shapes.
// level_done(l) (optional): makes s wait for level l's projection, so level
// l is compacted while the projections of the levels after it still run
// (compaction of level l touches only addresses below level l + 1's old slots).
void project_finish(Matrix& A, const TreePool& T, const TreePool& Tc, bool in_place, Arena& ar, cudaStream_t s,
                    const LevelHook& level_done = nullptr) {
  const int q = A.q;
  std::vector<int64_t> new_off(q + 2, 0);
  for (int l = 0; l <= q; ++l)
    new_off[l + 1] = new_off[l] + A.cpl[l].nb * int64_t(pad2(T.rows[l])) * Tc.rows[l];
  if (!in_place) {
    // compaction: level by level, block order, chunks staged in the arena
    double* temp = ar.base + ar.off;
    const int64_t cap = int64_t(ar.cap - ar.off);
    for (int l = 0; l <= q; ++l) {
      const Layer& L = A.cpl[l];
      const int64_t bs_new = int64_t(pad2(T.rows[l])) * Tc.rows[l], bs_old = L.block_stride();
      if (level_done) level_done(l);
      if (L.nb == 0 || bs_new == 0) continue;
      const int64_t per = std::max<int64_t>(1, cap / bs_new);
      const int64_t old_off = L.val - A.cpl_val.p;
      for (int64_t b0 = 0; b0 < L.nb;) {
        double* dst = A.cpl_val.p + new_off[l] + b0 * bs_new;
        const double* src = L.val + b0 * bs_old;
        // room between this chunk's destination and its (unread) sources:
        // chunks that fit in it are copied directly, the rest through temp
        const int64_t gap = (old_off + b0 * bs_old) - (new_off[l] + b0 * bs_new);
        int64_t nb = std::min(L.nb - b0, gap / bs_new);
        auto move = [&](double* d, const double* sp, int64_t so, int64_t cnt) {
          const unsigned grid = unsigned(std::min<int64_t>(cnt, 148 * 8));
          k_compact<<<grid, kThreads, 0, s>>>(d, sp, bs_new, so, cnt);
          H2B_CUDA(cudaGetLastError());
        };
        if (nb >= 1) {
          move(dst, src, bs_old, nb);
        } else {
          nb = std::min(per, L.nb - b0);
          move(temp, src, bs_old, nb);
          move(dst, temp, bs_new, nb);
        }
        b0 += nb;
      }
    }
  }
  H2B_CUDA(cudaStreamSynchronize(s));
  for (int l = 0; l <= q; ++l) {
    Layer& L = A.cpl[l];
    L.br = T.rows[l];
    L.bc = Tc.rows[l];
    L.ld = pad2(L.br);
    L.val = A.cpl_val.p + new_off[l];
  }
}

double sumsq(const double* v, int64_t n, cudaStream_t s, double* part) {
  if (n == 0) return 0.0;
  const int blocks = 1024;
  k_sumsq<<<blocks, kThreads, 0, s>>>(v, n, part);
  H2B_CUDA(cudaGetLastError());
  std::vector<double> h(blocks);
  H2B_CUDA(cudaMemcpyAsync(h.data(), part, blocks * sizeof(double), cudaMemcpyDeviceToHost, s));
  H2B_CUDA(cudaStreamSynchronize(s));
  double acc = 0.0;
  for (double v2 : h) acc += v2;
  return acc;
}

// Warps the weight-tree kernel keeps resident on the device (persistent).
int weights_slots(int device, int kc) {
  int sms = 0, per_sm = 0;
  H2B_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  constexpr int CR = 32;
  const size_t sm = kWWarps * (size_t(((kc * (kc + 1)) / 2 + 1) & ~1) + 2 * size_t(CR + 2)) * sizeof(double);
  if (kc > 32) {
    set_smem(k_weights<2, CR, true>, sm);
    set_smem(k_weights<2, CR, false>, sm);
    H2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_weights<2, CR, true>, 32 * kWWarps, sm));
  } else {
    set_smem(k_weights<1, CR, true>, sm);
    set_smem(k_weights<1, CR, false>, sm);
    H2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_weights<1, CR, true>, 32 * kWWarps, sm));
  }
  return sms * std::max(1, per_sm) * kWWarps;
}

size_t weights_arena_need(const Matrix& A) {
  size_t pmax = 1, items = 2;
  const int slots = weights_slots(A.device, 64);
  const Matrix& Cb = A.col_basis();
  for (int l = 1; l <= A.q; ++l) {
    pmax = std::max({pmax, size_t(A.nodes(l)) * A.rank[l - 1] * A.rank[l],
                     size_t(A.nodes(l)) * Cb.rank[l - 1] * Cb.rank[l]});
    items = std::max(items, size_t(std::max<int64_t>(A.own_count(l), slots)) + 2);
  }
  size_t nbmax = 1;
  for (int l = 1; l <= A.q; ++l) nbmax = std::max(nbmax, size_t(A.cpl[l].nb));
  // P, segment R's (<= slots + nodes), two item lists + counters, column-stack block list
  return Arena::need(pmax, sizeof(double)) + Arena::need(size_t(2 * items) * 64 * 64, sizeof(double)) +
         2 * Arena::need(items * sizeof(WItem) / sizeof(int32_t) + 4, sizeof(int32_t)) +
         Arena::need(4, 4) + Arena::need(nbmax, sizeof(int32_t));
}

// Weight tree (generate_weight_tree, compression.hpp:213-256), level by level
// top-down.  A level with fewer nodes than resident warps is split: every
// node's stack is cut into nseg contiguous segments processed by separate
// warps (partial R's, stored transposed), then a merge launch re-triangularises
// [R_0; ...; R_{nseg-1}] per node -- the same kernel, reading the partial R's
// as blocks.  Items are issued longest first (LPT).
// Transposed structure of a coupling level (the column stacks of a
// non-symmetric matrix, compression.hpp:497-520): for block column c, the
// blocks (r, c) in increasing r at [cp[c], cp[c + 1]) of cb.
void transpose_structure(const Layer& L, std::vector<int32_t>& cp, std::vector<int32_t>& cb, int& max_col) {
  cp.assign(L.rows + 1, 0);
  for (int64_t b = 0; b < L.nb; ++b) ++cp[L.h_ci[b] + 1];
  for (int64_t c = 0; c < L.rows; ++c) cp[c + 1] += cp[c];
  max_col = 0;
  for (int64_t c = 0; c < L.rows; ++c) max_col = std::max(max_col, cp[c + 1] - cp[c]);
  std::vector<int32_t> cur(cp.begin(), cp.end() - 1);
  cb.assign(L.nb, 0);
  for (int64_t r = 0; r < L.rows; ++r)
    for (int32_t b = L.h_rp[r]; b < L.h_rp[r + 1]; ++b) cb[cur[L.h_ci[b]]++] = b;
}

// Weight tree of basis B (generate_weight_tree, compression.hpp:213-256):
// B = A (row basis, row stacks of S^T) or, with col, A's column basis over
// the transposed layers (column stacks of S).
// before(l), when set, is called right before level l's weight-tree launches
// (after the parent products): the overlapped compression makes the chain
// stream wait there for level l's projection only.
void weights(Matrix& A, Matrix& B, bool col, TreePool& R, cudaStream_t s, Flops& fl, double& flops, const Part& pt,
             double* tree_mem, Arena& ar, const std::function<void(int)>& before = nullptr) {
  const int q = A.q;
  R.alloc(B, B.rank, B.rank, tree_mem);
  H2B_CUDA(cudaMemsetAsync(R.at(0), 0, sizeof(double) * B.rank[0] * B.rank[0], s));
  size_t pmax = 1, nbmax = 1;
  for (int l = 1; l <= q; ++l) {
    pmax = std::max(pmax, size_t(B.nodes(l)) * B.rank[l - 1] * B.rank[l]);
    nbmax = std::max(nbmax, size_t(A.cpl[l].nb));
  }
  ar.off = 0;
  double* Pall = ar.take<double>(pmax);
  const int slots = weights_slots(A.device, 64);
  size_t maxitems = 2;
  for (int l = 1; l <= q; ++l) maxitems = std::max(maxitems, size_t(std::max<int64_t>(A.own_count(l), slots)) + 2);
  double* segR = ar.take<double>(2 * maxitems * 64 * 64);
  WItem* ditems = ar.take<WItem>(maxitems);
  WItem* dmerge = ar.take<WItem>(maxitems);
  int* counters = ar.take<int>(4);
  int32_t* dcb = col ? ar.take<int32_t>(nbmax) : nullptr;
  std::vector<WItem> items, merge;
  std::vector<int32_t> cp, cb;
  for (int l = 1; l <= q; ++l) {
    const int kc = B.rank[l], kp = B.rank[l - 1];
    const Layer& L = A.cpl[l];
    int max_row = L.max_row;
    if (col) transpose_structure(L, cp, cb, max_row);
    const std::vector<int32_t>& ptr = col ? cp : L.h_rp;
    const int ld_ref = kp + max_row * kc;  // the reference's padded stack height
    flops += fl.gemm(double(B.nodes(l)), kp, kc, kp) + fl.qr(double(B.nodes(l)), ld_ref, kc);
    require(ld_ref >= kc, "qr_r_only_batched: requires rows >= cols");
    if (kc == 0) continue;
    require(L.nb == 0 || (col ? L.bc : L.br) == kc, "generate_weight_tree: dim mismatch");
    const int64_t r0 = A.own_begin(l), nn = A.own_count(l);  // r0 is even unless l == s (one node)
    if (nn == 0) continue;
    if (kp > 0) {
      k_weights_parent<<<unsigned(nn), kThreads, 0, s>>>(
          B.transfer.p + B.tr_off[l] + (r0 - B.tr_begin(l)) * B.tr_stride(l), B.ld(l), kc, kp,
          R.at(l - 1) + (r0 >> 1) * int64_t(kp) * kp, Pall);
      H2B_CUDA(cudaGetLastError());
    }
    if (col && L.nb)
      H2B_CUDA(cudaMemcpyAsync(dcb, cb.data(), cb.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    const WSrc src{L.val, L.ld, L.block_stride(), col ? L.br : L.bc, col ? 0 : 1, col ? dcb : nullptr};
    const int lslots = weights_slots(A.device, kc);
    int nseg = 1;
    if (nn < lslots) nseg = int(std::min<int64_t>((lslots + nn - 1) / nn, std::max(1, max_row / 4)));
    nseg = std::max(1, std::min(nseg, int(maxitems / std::max<int64_t>(1, nn))));
    items.clear();
    merge.clear();
    for (int64_t i = 0; i < nn; ++i) {
      const int32_t b0 = ptr[r0 + i], b1 = ptr[r0 + i + 1];
      if (nseg == 1) {
        items.push_back({int32_t(i), b0, b1, int32_t(i), 1});
      } else {
        for (int g = 0; g < nseg; ++g)
          items.push_back({int32_t(i), b0 + int32_t((int64_t(b1 - b0) * g) / nseg),
                           b0 + int32_t((int64_t(b1 - b0) * (g + 1)) / nseg), int32_t(i * nseg + g), g == 0});
        merge.push_back({int32_t(i), int32_t(i * nseg), int32_t((i + 1) * nseg), int32_t(i), 0});
      }
    }
    std::stable_sort(items.begin(), items.end(), [](const WItem& x, const WItem& y) {
      return (x.b1 - x.b0) + x.par > (y.b1 - y.b0) + y.par;
    });
    H2B_CUDA(cudaMemcpyAsync(ditems, items.data(), items.size() * sizeof(WItem), cudaMemcpyHostToDevice, s));
    H2B_CUDA(cudaMemsetAsync(counters, 0, 4 * sizeof(int), s));
    if (!merge.empty())
      H2B_CUDA(cudaMemcpyAsync(dmerge, merge.data(), merge.size() * sizeof(WItem), cudaMemcpyHostToDevice, s));
    constexpr int CR = 32;
    const size_t sm = kWWarps * (size_t(((kc * (kc + 1)) / 2 + 1) & ~1) + 2 * size_t(CR + 2)) * sizeof(double);
    double* Rl = R.at(l) + r0 * int64_t(kc) * kc;
    auto launch = [&](const WSrc& src, double* Rout, int out_t, const WItem* it, int64_t n, int* next) {
      const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>((n + kWWarps - 1) / kWWarps,
                                                                          lslots / kWWarps)));
      if (src.trans) {
        if (kc > 32)
          k_weights<2, CR, true><<<grid, 32 * kWWarps, sm, s>>>(Pall, kc, kp, src, Rout, out_t, it, n, next);
        else
          k_weights<1, CR, true><<<grid, 32 * kWWarps, sm, s>>>(Pall, kc, kp, src, Rout, out_t, it, n, next);
      } else {
        if (kc > 32)
          k_weights<2, CR, false><<<grid, 32 * kWWarps, sm, s>>>(Pall, kc, kp, src, Rout, out_t, it, n, next);
        else
          k_weights<1, CR, false><<<grid, 32 * kWWarps, sm, s>>>(Pall, kc, kp, src, Rout, out_t, it, n, next);
      }
      H2B_CUDA(cudaGetLastError());
    };
    if (before) before(l);
    if (nseg == 1) {
      launch(src, Rl, 0, ditems, int64_t(items.size()), counters);
    } else {
      launch(src, segR, 1, ditems, int64_t(items.size()), counters);
      // the partial R's, stored transposed, read as kc x kc "blocks"
      launch(WSrc{segR, kc, int64_t(kc) * kc, kc, 1, nullptr}, Rl, 0, dmerge, int64_t(merge.size()), counters + 1);
    }
    // the next level's uploads reuse the item buffers: keep stream order
    H2B_CUDA(cudaStreamSynchronize(s));
  }
}

double sum_host(const double* d, int64_t n, cudaStream_t s) {
  std::vector<double> h(n);
  if (n) H2B_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  H2B_CUDA(cudaStreamSynchronize(s));
  double acc = 0.0;
  for (double v : h) acc += v;
  return acc;
}

// Stages B (Jacobi) and C (Q1 application, tall) of a batch of nb SVDs of
// rows x cols matrices whose stage A wrote J, V, tau.
void svd_finish(const double* J, const double* V, const double* tau, int rows, int cols, double* U,
                double* sig, double eps, int* kmax, int64_t nb, cudaStream_t s) {
  const int sl = std::min(rows, cols);
  k_jacobi64<<<unsigned(nb), 64, 0, s>>>(J, sl, U, rows, int64_t(rows) * sl, sig, eps, kmax);
  H2B_CUDA(cudaGetLastError());
  if (rows >= cols) {
    const size_t sm = (size_t(rows) * cols + size_t(cols) * cols + 64) * sizeof(double);
    check_smem(sm, "truncate_basis");
    set_smem(k_svd_apply, sm);
    k_svd_apply<<<unsigned(nb), kThreads, sm, s>>>(V, tau, rows, cols, U);
    H2B_CUDA(cudaGetLastError());
  }
}

// H2B_TRACE=1: per-level wall-clock trace of the truncation on stderr.
struct Trace {
  bool on = std::getenv("H2B_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void at(cudaStream_t s, const char* tag, int l) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "  [trace] %8.2f ms %s l=%d\n", ms, tag, l);
  }
};

// Returns the discarded energy; fills Tt (new x old per node) and replaces
// the leaf / transfer pools and ranks.
// Scratch of truncate() (new ranks bounded by the old ones): the new
// transfers of every level, the per-level SVD batch (reused level to level)
// and the new leaf pool.
struct TruncSizes {
  std::vector<int64_t> ntoff;
  size_t lvl = 0, total = 0;
};
TruncSizes truncate_sizes(const Matrix& A) {
  TruncSizes z;
  const int q = A.q, m = A.m;
  const std::vector<int>& old = A.rank;
  z.ntoff.assign(q + 2, 0);
  for (int l = 1; l <= q; ++l) z.ntoff[l + 1] = z.ntoff[l] + A.tr_count(l) * int64_t(pad2(old[l])) * old[l - 1];
  const int64_t nlo = std::max<int64_t>(1, A.own_count(q));
  // per batch entry: U (rows x s), sigma, energy, J (s x s), Q1 (rows x cols + 64 tau)
  auto svd_need = [](size_t nb, int rows, int cols) {
    const int sl = std::min(rows, cols);
    return Arena::need(nb * rows * sl, 8) + Arena::need(nb * sl, 8) + Arena::need(nb, 8) +
           Arena::need(nb * sl * sl, 8) + Arena::need(nb * rows * cols, 8) + Arena::need(nb * 64, 8);
  };
  z.lvl = svd_need(size_t(nlo), m, old[q]);
  for (int l = q; l >= 1; --l) {
    const int64_t np = std::max<int64_t>(1, A.own_count(l - 1));
    const int zr = 2 * old[l], kp = old[l - 1];
    z.lvl = std::max(z.lvl, Arena::need(size_t(np) * zr * kp, 8) + svd_need(size_t(np), zr, kp));
  }
  z.total = Arena::need(size_t(std::max<int64_t>(1, z.ntoff[q + 1])), 8) + Arena::need(2, 4) +
            Arena::need(size_t(nlo) * pad2(m) * old[q], 8) + z.lvl;
  return z;
}

// on_t(l) (optional): called once Tt(l) (new x old per node) is final in
// stream order on s; Tt.rows[l] holds the new rank by then.
double truncate(Matrix& A, TreePool& R, double eps, TreePool& Tt, cudaStream_t s, Flops& fl,
                double& flops, const Part& pt, double* tree_mem, Arena& ar, const LevelHook& on_t_user = nullptr,
                std::vector<double>* level_energy = nullptr) {
  require(eps >= 0.0, "truncate_basis: eps must be non-negative");
  // partitioned: Tt(l) of a level > s gets its remote column bases from the
  // all-gather after the loop, Tt(s) from the one at the top of level s
  std::vector<int> deferred;
  bool gathered_s = !pt.dist(), gathered_all = !pt.dist();
  const LevelHook on_t = !on_t_user ? LevelHook() : LevelHook([&](int l) {
    if ((l > pt.s && !gathered_all) || (l == pt.s && !gathered_s))
      deferred.push_back(l);
    else
      on_t_user(l);
  });
  Trace tr;
  const int q = A.q, m = A.m;
  const std::vector<int> old = A.rank;
  std::vector<int> nr(q + 1, 0);
  std::vector<double> lev_e(q + 1, 0.0);
  const int64_t nl = A.nodes(q);
  // ---- all scratch up front (new ranks are bounded by the old ones) ----
  // Tt (new x old per node): level offsets sized for the old ranks, filled
  // in place; the new transfers: one region per level, compacted at the end.
  Tt.alloc(A, old, old, tree_mem);
  const TruncSizes sz = truncate_sizes(A);
  const std::vector<int64_t>& ntoff = sz.ntoff;
  const int sl_leaf = std::min(m, old[q]);
  const int64_t nlo = std::max<int64_t>(1, A.own_count(q)), l0 = A.own_begin(q);  // owned leaves
  ar.off = 0;
  double* newtr = ar.take<double>(std::max<int64_t>(1, ntoff[q + 1]));
  int* dk = ar.take<int>(2);  // [0] = kmax, [1] = non-finite flag
  double* newleaf = ar.take<double>(size_t(nlo) * pad2(m) * old[q]);
  const size_t lvl_base = ar.off;
  {
    const int kq = old[q];
    const int sl = sl_leaf;
    flops += fl.gemm(double(nl), m, kq, kq) + fl.svd(double(nl), m, kq);
    ar.off = lvl_base;
    const int64_t no = A.own_count(q);
    double* Uq = ar.take<double>(size_t(nlo) * m * sl);
    double* sg = ar.take<double>(size_t(nlo) * sl);
    double* en = ar.take<double>(size_t(nlo));
    double* Js = ar.take<double>(size_t(nlo) * sl * sl);
    double* Vs = ar.take<double>(size_t(nlo) * m * kq);
    double* ts = ar.take<double>(size_t(nlo) * 64);
    H2B_CUDA(cudaMemsetAsync(dk, 0, 2 * sizeof(int), s));
    if (sl > 0 && no > 0) {
      const size_t sm = (kSvdScratch + size_t(m) * kq + size_t(std::max(sl * sl, kq * m))) * sizeof(double);
      check_smem(sm, "truncate_basis");
      set_smem(k_trunc_leaf_pre, sm);
      k_trunc_leaf_pre<<<unsigned(no), kThreads, sm, s>>>(A.leaf.p, A.ldm, m, kq, R.at(q) + l0 * int64_t(kq) * kq,
                                                          Js, Vs, ts, dk + 1);
      H2B_CUDA(cudaGetLastError());
      svd_finish(Js, Vs, ts, m, kq, Uq, sg, eps, dk, no, s);
    }
    tr.at(s, "leaf svd", q);
    int flags[2] = {0, 0};
    H2B_CUDA(cudaMemcpyAsync(flags, dk, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    H2B_CUDA(cudaStreamSynchronize(s));
    pt.max_i32(flags, 2);  // the level rank is the max over ALL leaves
    require(flags[1] == 0, "svd_truncated_batched: non-finite input");
    const int kt = std::min(flags[0], sl);
    nr[q] = kt;
    flops += fl.gemm(double(nl), kt, kq, m);
    const int ldn = pad2(m);
    if (no > 0) {
      k_trunc_leaf_apply<<<unsigned(no), kThreads, 0, s>>>(A.leaf.p, A.ldm, m, kq, sl, kt, Uq, sg,
                                                           Tt.at(q) + l0 * int64_t(kt) * kq, newleaf, ldn, en);
      H2B_CUDA(cudaGetLastError());
    }
    Tt.rows[q] = kt;
    if (on_t) on_t(q);
    lev_e[q] = sum_host(en, no, s);
    tr.at(s, "leaf apply", q);
  }
  for (int l = q; l >= 1; --l) {
    const int ktc = nr[l], kc = old[l], kp = old[l - 1];
    const int64_t np = A.nodes(l - 1);
    const int zr = 2 * ktc;
    const int sl = std::min(zr, kp);
    flops += fl.gemm(double(A.nodes(l)), ktc, kp, kc) + fl.gemm(double(np), zr, kp, kp) +
             fl.svd(double(np), zr, kp);
    if (l == pt.s) {  // the replicated top needs every level-s child's T
      pt.allgather(Tt.at(l), int64_t(ktc) * kc, s);
      gathered_s = true;
      for (size_t d = 0; d < deferred.size();)
        if (deferred[d] == pt.s) {
          on_t_user(pt.s);
          deferred.erase(deferred.begin() + d);
        } else {
          ++d;
        }
    }
    const int64_t p0 = A.own_begin(l - 1), npo = A.own_count(l - 1);  // parents here
    ar.off = lvl_base;
    double* Z = ar.take<double>(size_t(npo) * zr * kp);
    double* U = ar.take<double>(size_t(npo) * zr * sl);
    double* sg = ar.take<double>(size_t(npo) * sl);
    double* en = ar.take<double>(size_t(npo));
    double* Js = ar.take<double>(size_t(npo) * sl * sl);
    double* Vs = ar.take<double>(size_t(npo) * zr * kp);
    double* ts = ar.take<double>(size_t(npo) * 64);
    H2B_CUDA(cudaMemsetAsync(dk, 0, 2 * sizeof(int), s));
    const int64_t es = A.tr_stride(l);
    if (sl > 0 && npo > 0) {
      const size_t sm = (kSvdScratch + size_t(zr) * kp + size_t(std::max(sl * sl, kp * zr))) * sizeof(double);
      check_smem(sm, "truncate_basis");
      set_smem(k_trunc_level_pre, sm);
      k_trunc_level_pre<<<unsigned(npo), kLevelThreads, sm, s>>>(
          A.transfer.p + A.tr_off[l] + (2 * p0 - A.tr_begin(l)) * es, A.ld(l), kc, kp, ktc,
          Tt.at(l) + 2 * p0 * int64_t(ktc) * kc, R.at(l - 1) + p0 * int64_t(kp) * kp, Z, Js, Vs, ts, dk + 1);
      H2B_CUDA(cudaGetLastError());
      svd_finish(Js, Vs, ts, zr, kp, U, sg, eps, dk, npo, s);
    }
    tr.at(s, "level svd", l);
    int flags[2] = {0, 0};
    H2B_CUDA(cudaMemcpyAsync(flags, dk, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    H2B_CUDA(cudaStreamSynchronize(s));
    if (l - 1 >= pt.s) pt.max_i32(flags, 2);  // (replicated parents agree already)
    require(flags[1] == 0, "svd_truncated_batched: non-finite input");
    const int ktp = std::min(flags[0], sl);
    nr[l - 1] = ktp;
    flops += fl.gemm(double(np), ktp, kp, zr);
    const int ldn = pad2(ktc);
    if (npo > 0) {
      k_trunc_level_apply<<<unsigned(npo), kThreads, 0, s>>>(
          ktc, kp, sl, ktp, Z, U, sg, Tt.at(l - 1) + p0 * int64_t(ktp) * kp,
          newtr + ntoff[l] + (2 * p0 - A.tr_begin(l)) * int64_t(ldn) * ktp, ldn, en);
      H2B_CUDA(cudaGetLastError());
    }
    Tt.rows[l - 1] = ktp;
    if (on_t) on_t(l - 1);
    const double el = sum_host(en, npo, s);
    lev_e[l - 1] = pt.counts(l - 1) ? el : 0.0;
    tr.at(s, "level apply", l);
  }
  // the projection with the rectangular T needs remote column bases too
  for (int l = pt.s + 1; l <= q; ++l)
    pt.allgather(Tt.at(l), (int64_t(1) << (l - pt.s)) * nr[l] * old[l], s);
  gathered_all = gathered_s = true;
  for (int l : deferred) on_t_user(l);
  Tt.rows = nr;  // per node: new x old, at the old-rank level offsets
  // new transfer pool with padded ld for the new ranks
  A.rank = nr;
  std::vector<int64_t> toff(q + 2, 0);
  int64_t t = 0;
  for (int l = 1; l <= q; ++l) {
    toff[l] = t;
    t += A.tr_count(l) * A.tr_stride(l);
  }
  toff[q + 1] = t;
  // the new (smaller) pools overwrite the old allocations
  require(size_t(t) <= std::max<size_t>(A.transfer.n, 1), "truncate: transfer pool grew");
  for (int l = 1; l <= q; ++l) {
    const int64_t n = A.tr_count(l) * A.tr_stride(l);
    if (n) H2B_CUDA(cudaMemcpyAsync(A.transfer.p + toff[l], newtr + ntoff[l], n * sizeof(double),
                                    cudaMemcpyDeviceToDevice, s));
  }
  const int64_t nleaf = A.own_count(q) * int64_t(pad2(m)) * nr[q];
  if (nleaf) H2B_CUDA(cudaMemcpyAsync(A.leaf.p, newleaf, nleaf * sizeof(double), cudaMemcpyDeviceToDevice, s));
  H2B_CUDA(cudaStreamSynchronize(s));
  A.tr_off = toff;
  if (level_energy) *level_energy = lev_e;
  double energy = 0.0;
  for (double e : lev_e) energy += e;
  return energy;
}

// Highest-priority stream ordered after `user` on construction; `user` is
// ordered after it on destruction.
struct ChainStream {
  cudaStream_t user, s = nullptr;
  cudaEvent_t e = nullptr;
  explicit ChainStream(cudaStream_t u) : user(u) {
    int lo = 0, hi = 0;
    H2B_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    H2B_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi));
    H2B_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    H2B_CUDA(cudaEventRecord(e, user));
    H2B_CUDA(cudaStreamWaitEvent(s, e, 0));
  }
  ~ChainStream() {
    cudaEventRecord(e, s);
    cudaStreamWaitEvent(user, e, 0);
    cudaStreamSynchronize(s);
    cudaEventDestroy(e);
    cudaStreamDestroy(s);
  }
};

// Side stream of compress(): fork(l) makes it wait for the main stream's
// work issued so far (T(l) final), join() makes the main stream wait for it.
// Disabled: b is the main stream itself and both are no-ops.
// Side streams for the projections, ONE PER LEVEL, below the main stream's
// priority: the producers (orthogonalization, truncation) finish the levels
// bottom-up, the weight tree consumes them top-down, so a small top level's
// projection must not queue behind the big bottom levels' in one in-order
// stream -- nor behind their CTAs in the block scheduler: the stream of the
// level d above the leaves has priority lo - d (clamped one below the main
// stream), so once the leaf level's projection (the biggest, issued first)
// holds the GPU, every upper level's CTAs still go first as slots free up.
// The stream sets are indexed by d, created on first use and recycled through
// a per-device free list (creating 15 streams per call left the GPU idle for
// ms).
struct SideSet {
  std::vector<cudaStream_t> bs = std::vector<cudaStream_t>(kMaxLevels + 1, nullptr);
  std::vector<cudaEvent_t> ev = std::vector<cudaEvent_t>(kMaxLevels + 1, nullptr);   // fork points
  std::vector<cudaEvent_t> lev = std::vector<cudaEvent_t>(kMaxLevels + 1, nullptr);  // per-level completion
};
struct SidePool {
  std::mutex mu;
  std::map<int, std::vector<SideSet*>> free;  // never destroyed: device teardown frees the streams
};
SidePool& side_pool() {
  static SidePool p;
  return p;
}
SideSet* side_acquire(int device) {
  SidePool& p = side_pool();
  std::lock_guard<std::mutex> g(p.mu);
  auto& f = p.free[device];
  if (f.empty()) return new SideSet;
  SideSet* r = f.back();
  f.pop_back();
  return r;
}
void side_release(int device, SideSet* set) {
  SidePool& p = side_pool();
  std::lock_guard<std::mutex> g(p.mu);
  p.free[device].push_back(set);
}

struct SideStream {
  cudaStream_t s;
  bool on;
  int device = 0;
  SideSet* set = nullptr;
  std::vector<char> used = std::vector<char>(kMaxLevels + 1, 0);
  int q = 0;  // leaf level: level l uses slot q - l
  SideStream(bool enable, cudaStream_t main, int leaf_level) : s(main), on(enable), q(leaf_level) {
    if (!on) return;
    H2B_CUDA(cudaGetDevice(&device));
    set = side_acquire(device);
  }
  ~SideStream() {
    if (!on) return;
    for (int l = 0; l <= kMaxLevels; ++l)
      if (used[l]) cudaStreamSynchronize(set->bs[l]);
    side_release(device, set);
  }
  SideStream(const SideStream&) = delete;
  SideStream& operator=(const SideStream&) = delete;
  // the stream level l's side work goes to (the main stream when off)
  cudaStream_t b(int l) {
    if (!on) return s;
    const int d = q - l;
    if (!set->bs[d]) {
      int lo = 0, hi = 0;
      H2B_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      const int prio = hi < lo ? std::max(hi + 1, lo - d) : lo;
      H2B_CUDA(cudaStreamCreateWithPriority(&set->bs[d], cudaStreamNonBlocking, prio));
      H2B_CUDA(cudaEventCreateWithFlags(&set->ev[d], cudaEventDisableTiming));
      H2B_CUDA(cudaEventCreateWithFlags(&set->lev[d], cudaEventDisableTiming));
    }
    used[d] = 1;
    return set->bs[d];
  }
  // level l's side work starts after everything enqueued on the main stream so far
  void fork(int l) {
    if (!on) return;
    cudaStream_t st = b(l);
    H2B_CUDA(cudaEventRecord(set->ev[q - l], s));
    H2B_CUDA(cudaStreamWaitEvent(st, set->ev[q - l], 0));
  }
  // level l's side work is enqueued: mark its completion
  void mark(int l) {
    if (!on) return;
    cudaStream_t st = b(l);
    H2B_CUDA(cudaEventRecord(set->lev[q - l], st));
  }
  // the main stream waits for level l's side work only
  void wait(int l) {
    if (!on || !used[q - l]) return;
    H2B_CUDA(cudaStreamWaitEvent(s, set->lev[q - l], 0));
  }
  // the main stream waits for all side work
  void join() {
    if (!on) return;
    for (int l = 0; l <= kMaxLevels; ++l)
      if (used[l]) {
        H2B_CUDA(cudaEventRecord(set->lev[l], set->bs[l]));
        H2B_CUDA(cudaStreamWaitEvent(s, set->lev[l], 0));
      }
  }
};

// Resize the workspace and rebuild the BSR work list after ranks changed.
void relayout(Matrix& A) {
  const int q = A.q;
  A.vec_off.assign(q + 2, 0);
  for (int l = 0; l <= q; ++l) A.vec_off[l + 1] = A.vec_off[l] + A.nodes(l) * A.rank[l];
  if (!A.symmetric) {  // x^ follows the column basis
    Matrix& C = *A.colb;
    C.vec_off.assign(q + 2, 0);
    for (int l = 0; l <= q; ++l) C.vec_off[l + 1] = C.vec_off[l] + C.nodes(l) * C.rank[l];
  }
  // every workspace (the handle's and any h2b_context) re-sizes on next use
  ++A.layout_version;
  // the block pattern (row_ptr / col_idx, the symmetric mirror map) is
  // unchanged; only the work list's row costs changed with the ranks (the full
  // upload_structure rebuilt the mirror map on the host: 16-19 ms of idle GPU)
  rebuild_work_list(A);
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    H2B_CUDA(cudaSetDevice(d));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

// Free the cached compression workspaces of a device (h2b_release_cached_memory).
void release_workspaces(int device) {
  std::lock_guard<std::mutex> lk(ws_cache().mu);
  auto& fr = ws_cache().free;
  if (device >= 0 && device < int(fr.size())) fr[device].clear();
}

// memory_footprint (h2_matrix.hpp:90-102) of the part of the matrix this
// rank accounts for: its own blocks, replicated top levels on rank 0 only
uint64_t counted_footprint(const Matrix& A, const Part& pt) {
  uint64_t e = uint64_t(A.dense.nb) * A.dense.br * A.dense.bc + uint64_t(A.own_count(A.q)) * A.m * A.rank[A.q];
  for (int l = 0; l <= A.q; ++l)
    if (pt.counts(l)) e += uint64_t(A.cpl[l].nb) * A.cpl[l].br * A.cpl[l].bc;
  for (int l = 1; l <= A.q; ++l)
    if (l > pt.s || pt.counts(0)) e += uint64_t(A.tr_count(l)) * A.rank[l] * A.rank[l - 1];
  if (!A.symmetric) {  // the column basis (h2_matrix.hpp:97-100; never partitioned)
    const Matrix& C = *A.colb;
    e += uint64_t(C.own_count(C.q)) * C.m * C.rank[C.q];
    for (int l = 1; l <= C.q; ++l) e += uint64_t(C.tr_count(l)) * C.rank[l] * C.rank[l - 1];
  }
  return e * sizeof(double);
}

// The compression kernels (register Householder, 64-thread Jacobi, 64 x 64
// DMMA projection tiles) cover ranks and leaf sizes up to 64; the mat-vec
// kernels go to 128 (k_hmv_big.cu).
void require_compress_dims(const Matrix& B, const char* what) {
  if (big_basis(B))
    throw Error(H2B_UNSUPPORTED, std::string(what) + ": rank or leaf size > 64 not supported by the compression kernels");
}

void compress_matrix(Matrix& A, double eps, h2b_compress_report* rep, const h2b_comm* comm) {
  require(eps >= 0.0, "truncate_basis: eps must be non-negative");
  require_compress_dims(A, "compress");
  if (!A.symmetric) require_compress_dims(*A.colb, "compress");
  DeviceGuard g(A.device);
  // The dependency chain (orthogonalization, weights, truncation) runs on a
  // highest-priority stream ordered after the handle's stream; the
  // projections on lower-priority per-level side streams soak up the SMs it leaves
  // idle (SideStream).
  ChainStream chain(A.stream);
  cudaStream_t s = chain.s;
  // One workspace for the whole call (cached per device, see WsCache):
  // region A holds the projection trees (To, then Tt), region B the weight
  // tree R, region C the phase scratch (weights, truncation, the chunked
  // compaction of the coupling pool).
  // (non-symmetric: the column basis' trees follow the row basis' in A and B)
  const bool sym = A.symmetric;
  Matrix& Cb = A.col_basis();
  const size_t tree_row = TreePool::need(A, A.rank, A.rank);
  const size_t tree_need = tree_row + (sym ? 0 : TreePool::need(Cb, Cb.rank, Cb.rank));
  const size_t arena_need = std::max({weights_arena_need(A), truncate_sizes(A).total,
                                      sym ? size_t(0) : truncate_sizes(Cb).total, size_t(1) << 25});
  const size_t proj_need = ProjRows::need(A);
  Workspace ws{A.device};
  ws.buf = ws_checkout(A.device, 2 * tree_need + arena_need + proj_need);
  ws.trees = ws.buf.p;
  ws.rtree = ws.buf.p + tree_need;
  double* trees_col = ws.trees + tree_row;
  double* rtree_col = ws.rtree + tree_row;
  ws.arena = ws.buf.p + 2 * tree_need;
  ws.arena_cap = ws.buf.n - 2 * tree_need - proj_need;  // all the rest (projection chunks)
  Arena ar, par;  // phase scratch; the projection work lists (at the end: live across phases)
  ar.reserve(ws.arena, ws.arena_cap);
  par.reserve(ws.arena + ws.arena_cap, proj_need);
  if (std::getenv("H2B_TRACE"))
    fprintf(stderr, "  [trace] compress workspace %.2f GB (arena %.2f GB)\n", ws.buf.n * 8e-9,
            ws.arena_cap * 8e-9);
  Part pt;
  pt.comm = comm;
  pt.s = comm ? A.part_s : 0;
  pt.g = comm ? A.part_g : 0;
  Flops fl;
  h2b_compress_report r{};
  for (int l = 0; l <= A.q; ++l) r.old_ranks[l] = A.rank[l];
  // the reference's padded weight-stack height uses the GLOBAL longest block row
  std::vector<int32_t> mrow(A.q + 1);
  for (int l = 0; l <= A.q; ++l) mrow[l] = A.cpl[l].max_row;
  pt.max_i32(mrow.data(), A.q + 1);
  std::vector<int> saved_max(A.q + 1);
  for (int l = 0; l <= A.q; ++l) {
    saved_max[l] = A.cpl[l].max_row;
    A.cpl[l].max_row = mrow[l];
  }
  double sums[3] = {double(counted_footprint(A, pt)), 0.0, 0.0};

  // The projections run level by level on a side stream as soon as T(l) is
  // final, overlapping the (bottom-up, increasingly latency-bound) chains of
  // the orthogonalization and of the truncation on the main stream.  Phase
  // times are therefore boundary to boundary on the main stream: a
  // projection phase is what remains of it after its producer phase.
  // Partitioned compression: a partitioned level's projection starts once the
  // all-gather has brought the remote column bases (orthogonalize / truncate
  // defer its hook until then).
  const bool overlap = sym;
  SideStream side(overlap, s, A.q);
  ProjRows PR;
  project_rows(A, par, PR, s);
  TreePool To, R, Tt, Toc, Rc, Ttc;  // row basis; column basis (non-symmetric)
  TreePool& To_c = sym ? To : Toc;
  TreePool& Tt_c = sym ? Tt : Ttc;
  double n2 = 0.0;  // ||A||_F^2 after the orthogonal projection (compression.hpp:487)
  Matrix* Ap = &A;
  auto hook = [Ap, &PR, &fl, &pt, &side](TreePool& T, bool tri, bool want_sum, double& fl_acc) -> LevelHook {
    TreePool* Tp = &T;
    double* fa = &fl_acc;
    return [Ap, Tp, fa, tri, want_sum, &PR, &fl, &pt, &side](int l) {
      side.fork(l);
      project_level(*Ap, *Tp, *Tp, PR, l, tri, want_sum, fl, *fa, pt, side.b(l));
      side.mark(l);
    };
  };
  {
    NvtxRange nv("h2b compress: orthogonalize");
    Timer t(s);
    orthogonalize(A, To, s, fl, r.flops_orthogonalize, pt, ws.trees,
                  overlap ? hook(To, true, true, r.flops_project_orth) : nullptr);
    if (!sym) orthogonalize(Cb, Toc, s, fl, r.flops_orthogonalize, pt, trees_col);
    r.time_orthogonalize_ms = t.stop();
  }
  if (!overlap) {
    {
      NvtxRange nv("h2b compress: project (orthogonal)");
      Timer t(s);
      for (int l = A.q; l >= 0; --l) project_level(A, To, To_c, PR, l, true, true, fl, r.flops_project_orth, pt, s);
      n2 = project_rowsum(PR, pt, s);
      project_finish(A, To, To_c, /*in_place=*/true, ar, s);
      r.time_project_orth_ms = t.stop();
    }
    n2 += sumsq(A.dense.val, A.dense.nb * A.dense.block_stride(), s, ws.arena);
    pt.sum_f64(&n2, 1);
    {
      NvtxRange nv("h2b compress: weight tree");
      Timer t(s);
      weights(A, A, false, R, s, fl, r.flops_weights, pt, ws.rtree, ar);
      if (!sym) weights(A, Cb, true, Rc, s, fl, r.flops_weights, pt, rtree_col, ar);  // transposed layers
      r.time_weights_ms = t.stop();
    }
  } else {
    // The weight tree goes top-down and level l needs only level l's projected
    // blocks: its launches wait for that level's projection (side.wait), so
    // the small, latency-bound top levels run while the big bottom levels are
    // still being projected.  The projection phase then has no time of its
    // own (reported as 0; its kernels run inside the orthogonalization and
    // weight-tree phases).  The in-place orthogonal projection changes no
    // layer shape, so project_finish and ||A||_F come after the weight tree.
    NvtxRange nv("h2b compress: weight tree (overlapping the orthogonal projection)");
    Timer t(s);
    weights(A, A, false, R, s, fl, r.flops_weights, pt, ws.rtree, ar, [&side](int l) { side.wait(l); });
    side.join();
    r.time_weights_ms = t.stop();
    r.time_project_orth_ms = 0.0;
    n2 = project_rowsum(PR, pt, s);
    project_finish(A, To, To_c, /*in_place=*/true, ar, s);
    n2 += sumsq(A.dense.val, A.dense.nb * A.dense.block_stride(), s, ws.arena);
    pt.sum_f64(&n2, 1);
  }
  r.frobenius_norm = std::sqrt(n2);
  for (int l = 0; l <= A.q; ++l) A.cpl[l].max_row = saved_max[l];
  double energy = 0.0;
  {
    NvtxRange nv("h2b compress: truncate");
    Timer t(s);
    energy = truncate(A, R, eps, Tt, s, fl, r.flops_truncate, pt, ws.trees, ar,
                      overlap ? hook(Tt, false, false, r.flops_project_trunc) : nullptr);
    if (!sym) energy += truncate(Cb, Rc, eps, Ttc, s, fl, r.flops_truncate, pt, trees_col, ar);
    r.time_truncate_ms = t.stop();
  }
  {
    NvtxRange nv("h2b compress: project (truncated)");
    Timer t(s);
    if (!overlap)
      for (int l = A.q; l >= 0; --l)
        project_level(A, Tt, Tt_c, PR, l, false, false, fl, r.flops_project_trunc, pt, s);
    // levels are compacted in address order as their projections complete:
    // the upper levels (finished first, see SideStream) while the leaf
    // level's projection still runs
    project_finish(A, Tt, Tt_c, /*in_place=*/false, ar, s, [&side](int l) { side.wait(l); });
    side.join();
    r.time_project_trunc_ms = t.stop();
  }
  relayout(A);
  for (int l = 0; l <= A.q; ++l) r.new_ranks[l] = A.rank[l];
  // global sums: footprints, discarded energy, projection flops (local rows)
  double g5[5] = {sums[0], double(counted_footprint(A, pt)), energy, r.flops_project_orth, r.flops_project_trunc};
  pt.sum_f64(g5, 5);
  r.bytes_before = uint64_t(g5[0]);
  r.bytes_after = uint64_t(g5[1]);
  energy = g5[2];
  r.flops_project_orth = g5[3];
  r.flops_project_trunc = g5[4];
  r.frobenius_error = r.frobenius_norm > 0 ? std::sqrt(energy) / r.frobenius_norm : 0.0;
  if (A.part_s > 0) A.global_footprint = r.bytes_after;

  if (rep) *rep = r;
#ifdef H2B_SWEEP_HIST
  int hist[64];
  H2B_CUDA(cudaMemcpyFromSymbol(hist, cta::g_sweep_hist, sizeof(hist)));
  fprintf(stderr, "jacobi sweeps:");
  for (int i = 0; i <= 60; ++i)
    if (hist[i]) fprintf(stderr, " %d:%d", i + 1, hist[i]);
  fprintf(stderr, "\n");
  std::fill(hist, hist + 64, 0);
  H2B_CUDA(cudaMemcpyToSymbol(cta::g_sweep_hist, hist, sizeof(hist)));
#endif
}

// ---------------------------------------------------------------- phase API
// The reference's compression phases on component objects (phases.cu):
// B a basis-only Matrix (BasisTree), S a coupling-only Matrix (MatrixTree).
// Trees (ProjectionTree / WeightTree pools) are level-concatenated device
// arrays, rows[l] x cols[l] per node, column-major, like the reference's pools.

// orthogonalize_basis(B) (compression.hpp:69-126): t_dev gets T (k_l x k_l per node).
void phase_orthogonalize(Matrix& B, double* t_dev, cudaStream_t s) {
  require_compress_dims(B, "orthogonalize_basis");
  Flops fl;
  double f = 0;
  TreePool T;
  orthogonalize(B, T, s, fl, f, Part{}, t_dev);
  H2B_CUDA(cudaStreamSynchronize(s));
}

// project_coupling(Trow, Tcol, S) (compression.hpp:130-169) into a fresh pool
// (the new block shapes may be larger than the old ones); same: Tcol is Trow.
void phase_project(Matrix& S, const double* tr, const std::vector<int>& tr_rows, const std::vector<int>& tr_cols,
                   const double* tc, const std::vector<int>& tc_rows, const std::vector<int>& tc_cols, bool same,
                   cudaStream_t s) {
  const int q = S.q;
  TreePool Tr, Tc;
  Tr.alloc(S, tr_rows, tr_cols, const_cast<double*>(tr));
  Tc.alloc(S, tc_rows, tc_cols, const_cast<double*>(tc));
  for (int l = 0; l <= q; ++l) {
    const Layer& L = S.cpl[l];
    if (L.nb == 0) continue;
    require(tr_cols[l] == L.br && tc_cols[l] == L.bc, "project_coupling: dim mismatch");
    if (tr_rows[l] > kMaxDim || tc_rows[l] > kMaxDim)
      throw Error(H2B_UNSUPPORTED, "project_coupling: rank > 64 not supported by the compiled kernels");
  }
  std::vector<int64_t> noff(q + 2, 0);
  for (int l = 0; l <= q; ++l) noff[l + 1] = noff[l] + S.cpl[l].nb * int64_t(pad2(tr_rows[l])) * tc_rows[l];
  DevBuf<double> out;
  out.alloc(std::max<int64_t>(1, noff[q + 1]));
  Workspace ws{S.device};
  ws.buf = ws_checkout(S.device, ProjRows::need(S) + 64);
  Arena par;
  par.reserve(ws.buf.p, ws.buf.n);
  ProjRows PR;
  project_rows(S, par, PR, s, same);
  Flops fl;
  double f = 0;
  for (int l = 0; l <= q; ++l)
    project_level(S, Tr, Tc, PR, l, /*tri=*/false, /*want_sum=*/false, fl, f, Part{}, s, same, out.p + noff[l],
                  int64_t(pad2(tr_rows[l])) * tc_rows[l]);
  H2B_CUDA(cudaStreamSynchronize(s));
  S.cpl_val = std::move(out);
  for (int l = 0; l <= q; ++l) {
    Layer& L = S.cpl[l];
    L.br = tr_rows[l];
    L.bc = tc_rows[l];
    L.ld = pad2(L.br);
    L.val = S.cpl_val.p + noff[l];
  }
}

// generate_weight_tree(B, S) (compression.hpp:213-256): r_dev gets R (k_l x k_l
// per node, upper triangular; R^0 = 0).
void phase_weights(Matrix& S, Matrix& B, double* r_dev, cudaStream_t s) {
  require_compress_dims(B, "generate_weight_tree");
  require(S.q == B.q, "generate_weight_tree: depth mismatch");
  for (int l = 1; l <= S.q; ++l)
    require(S.cpl[l].nb == 0 || S.cpl[l].br == B.rank[l], "generate_weight_tree: dim mismatch");
  Flops fl;
  double f = 0;
  TreePool R;
  Workspace ws{S.device};
  const size_t need = weights_arena_need(S) + 64;
  ws.buf = ws_checkout(S.device, need);
  Arena ar;
  ar.reserve(ws.buf.p, ws.buf.n);
  weights(S, B, false, R, s, fl, f, Part{}, r_dev, ar);
  H2B_CUDA(cudaStreamSynchronize(s));
}

// truncate_basis(B, R, eps, Tout) (compression.hpp:267-420): B is truncated in
// place; t_dev gets Tout level-concatenated, new_rank[l] x old_rank[l] per node;
// energy[l] the discarded energy of level l.
void phase_truncate(Matrix& B, const double* r_dev, double eps, double* t_dev, std::vector<double>& energy,
                    cudaStream_t s) {
  require_compress_dims(B, "truncate_basis");
  require(eps >= 0.0, "truncate_basis: eps must be non-negative");
  const std::vector<int> old = B.rank;
  Flops fl;
  double f = 0;
  TreePool R, Tt;
  R.alloc(B, B.rank, B.rank, const_cast<double*>(r_dev));
  const size_t tree = TreePool::need(B, old, old);
  Workspace ws{B.device};
  const size_t arena = truncate_sizes(B).total + 64;
  ws.buf = ws_checkout(B.device, tree + arena);
  Arena ar;
  ar.reserve(ws.buf.p + tree, ws.buf.n - tree);
  truncate(B, R, eps, Tt, s, fl, f, Part{}, ws.buf.p, ar, nullptr, &energy);
  int64_t o = 0;
  for (int l = 0; l <= B.q; ++l) {
    const int64_t c = B.nodes(l) * int64_t(Tt.rows[l]) * old[l];
    if (c) H2B_CUDA(cudaMemcpyAsync(t_dev + o, Tt.at(l), c * sizeof(double), cudaMemcpyDeviceToDevice, s));
    o += c;
  }
  H2B_CUDA(cudaStreamSynchronize(s));
  B.vec_off.assign(B.q + 2, 0);
  for (int l = 0; l <= B.q; ++l) B.vec_off[l + 1] = B.vec_off[l] + B.nodes(l) * B.rank[l];
  ++B.layout_version;
}

// col: the column basis (non-symmetric matrices; the row basis itself when
// symmetric).  The coupling is not projected (the reference's contract).
void orthogonalize_matrix(Matrix& A, double* t_out, bool col) {
  DeviceGuard g(A.device);
  cudaStream_t s = A.stream;
  Matrix& B = col ? A.col_basis() : A;
  require_compress_dims(B, "orthogonalize_basis");
  Flops fl;
  double f = 0;
  TreePool T;
  Workspace ws{A.device};
  ws.buf = ws_checkout(A.device, TreePool::need(B, B.rank, B.rank));
  orthogonalize(B, T, s, fl, f, Part{}, ws.buf.p);
  if (t_out && T.off[A.q + 1])
    H2B_CUDA(cudaMemcpyAsync(t_out, T.p, T.off[A.q + 1] * sizeof(double), cudaMemcpyDeviceToHost, s));
  H2B_CUDA(cudaStreamSynchronize(s));
}

}  // namespace h2b
