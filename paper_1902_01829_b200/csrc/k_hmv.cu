// HMV kernels for sm_100a (FP64).  One warp owns one small matrix at a time;
// lane L owns the row pair (2L, 2L+1) of every block it touches, so a column
// of a 64-row block is one fully coalesced 512-byte warp load (32 x 128-bit).
//
// Phase map (reference include/h2kit/hmv.hpp, Appendix B of SURVEY.md):
//   k_up_leaf    : xc = x[perm] (hmv.hpp:179) fused with x^q = V^T xc (hmv.hpp:86-97)
//   k_up_level   : x^{l-1}_p = F_2p^T x^l_2p + F_2p+1^T x^l_2p+1 (hmv.hpp:98-110)
//   k_bsr        : yc = D xc (hmv.hpp:180) and y^l = S^l x^l for every level
//                  (hmv.hpp:114-125) in ONE launch over a flattened row list
//   k_down_level : y^l_c += E_c y^{l-1}_{c/2} (hmv.hpp:136-146)
//   k_down_leaf  : yc += U y^q (hmv.hpp:147-156) fused with the alpha/beta
//                  scatter y[perm[t]] = alpha yc[t] + beta y[perm[t]] (hmv.hpp:184-187)
// All matrix bytes are read exactly once per phase with streaming
// (evict-first) 128-bit loads; node vectors stay L2-resident.
#include "dataflow.cuh"
#include "h2b_internal.hpp"
#include "tma.cuh"
#include "warp_gemv.cuh"

#include <algorithm>
#include <numeric>

namespace h2b {
namespace {

#ifndef H2B_TMA_BSR1
#define H2B_TMA_BSR1 1
#endif
constexpr bool kTmaBsr = H2B_TMA_BSR1;
// fused sweeps: 0 claim an item after the previous one and prefetch its
// transfers into L2 before its flag wait; 1 claim the next item ahead and
// prefetch it while this one runs -- measured 1.10 -> 1.58 ms per sweep at C4
// (an item claimed ahead holds back the items that wait on it); -1 no prefetch
#ifndef H2B_SWEEP_AHEAD
#define H2B_SWEEP_AHEAD 0
#endif
constexpr int kSweepAhead = H2B_SWEEP_AHEAD;
#ifndef H2B_TMA_FORCE
#define H2B_TMA_FORCE 0
#endif  // k_bsr_tma (else the register-fed k_bsr)

constexpr int kThreads = 256;  // 8 warps per CTA
using namespace wg;

__global__ void __launch_bounds__(kThreads, 2) k_up_leaf(const double* __restrict__ x,
                                                      const int32_t* __restrict__ perm,
                                                      const double* __restrict__ leaf, int m,
                                                      int ldm, int k, int64_t nleaves, int64_t leaf0,
                                                      double* __restrict__ xc,
                                                      double* __restrict__ xh) {
  const int r = 2 * lane_id();
  const int64_t stride = int64_t(ldm) * k;
  for (int64_t il = warp_global(); il < nleaves; il += warp_count()) {
    const int64_t i = leaf0 + il;  // global leaf index; the pool holds owned leaves only
    const int64_t base = i * m;
    double v0 = 0.0, v1 = 0.0;
    // perm == nullptr: x is already in cluster order (phase API).
    if (r < m) {
      v0 = __ldg(x + (perm ? __ldg(perm + base + r) : base + r));
      xc[base + r] = v0;
    }
    if (r + 1 < m) {
      v1 = __ldg(x + (perm ? __ldg(perm + base + r + 1) : base + r + 1));
      xc[base + r + 1] = v1;
    }
    if (k == 0) continue;
    const double* V = leaf + il * stride;
    const double o0 = gemvT_group<false>(V, nullptr, ldm, k, 0, v0, v1, 0, 0, r < ldm);
    const double o1 = gemvT_group<false>(V, nullptr, ldm, k, 1, v0, v1, 0, 0, r < ldm);
    if (r < k) xh[i * k + r] = o0;
    if (r + 1 < k) xh[i * k + r + 1] = o1;
  }
}

__global__ void __launch_bounds__(kThreads, 2) k_up_level(const double* __restrict__ F, int ldc,
                                                       int kc, int kp, int64_t p0, int64_t p1,
                                                       int64_t cbegin,
                                                       const double* __restrict__ xl,
                                                       double* __restrict__ xp) {
  const int r = 2 * lane_id();
  const int64_t stride = int64_t(ldc) * kp;
  for (int64_t p = p0 + warp_global(); p < p1; p += warp_count()) {
    const double* x0 = xl + (2 * p) * kc;
    const double* x1 = x0 + kc;
    const double v0 = r < kc ? x0[r] : 0.0, v1 = r + 1 < kc ? x0[r + 1] : 0.0;
    const double w0 = r < kc ? x1[r] : 0.0, w1 = r + 1 < kc ? x1[r + 1] : 0.0;
    const double* A = F + (2 * p - cbegin) * stride;
    const double o0 = gemvT_group<true>(A, A + stride, ldc, kp, 0, v0, v1, w0, w1, r < ldc);
    const double o1 = gemvT_group<true>(A, A + stride, ldc, kp, 1, v0, v1, w0, w1, r < ldc);
    if (r < kp) xp[p * kp + r] = o0;
    if (r + 1 < kp) xp[p * kp + r + 1] = o1;
  }
}

__global__ void __launch_bounds__(kThreads) k_down_level(const double* __restrict__ E, int ldc,
                                                         int kc, int kp, int64_t c0, int64_t c1,
                                                         int64_t cbegin,
                                                         const double* __restrict__ yp_all,
                                                         double* __restrict__ yl) {
  const int r = 2 * lane_id();
  const int64_t stride = int64_t(ldc) * kp;
  for (int64_t c = c0 + warp_global(); c < c1; c += warp_count()) {
    const double* yp = yp_all + (c >> 1) * kp;
    const double a0 = r < kp ? yp[r] : 0.0, a1 = r + 1 < kp ? yp[r + 1] : 0.0;
    double acc0, acc1;
    gemvN_pair(E + (c - cbegin) * stride, ldc, kp, a0, a1, r < ldc, acc0, acc1);
    double* y = yl + c * kc;
    if (r < kc) y[r] = acc0 + y[r];
    if (r + 1 < kc) y[r + 1] = acc1 + y[r + 1];
  }
}

__global__ void __launch_bounds__(kThreads) k_down_leaf(
    const double* __restrict__ U, int ldm, int m, int k, int64_t nleaves, int64_t leaf0,
    const double* __restrict__ yh, const double* __restrict__ yc,
    const int32_t* __restrict__ perm, double* __restrict__ y, double alpha, double beta,
    int to_user) {
  const int r = 2 * lane_id();
  const int64_t stride = int64_t(ldm) * k;
  for (int64_t il = warp_global(); il < nleaves; il += warp_count()) {
    const int64_t i = leaf0 + il;  // global leaf index; the pool holds owned leaves only
    const double* yq = yh + i * k;
    const double a0 = r < k ? yq[r] : 0.0, a1 = r + 1 < k ? yq[r + 1] : 0.0;
    double acc0 = 0.0, acc1 = 0.0;
    if (k > 0) gemvN_pair(U + il * stride, ldm, k, a0, a1, r < ldm, acc0, acc1);
    const int64_t base = i * m;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int rr = r + h;
      if (rr >= m) continue;
      const double v = (h ? acc1 : acc0) + yc[base + rr];
      if (to_user) {
        const int64_t o = perm[base + rr];
        y[o] = alpha * v + (beta == 0.0 ? 0.0 : beta * y[o]);
      } else {
        y[il * m + rr] = v;  // cluster-order slice starting at the first owned leaf
      }
    }
  }
}

// ---- fused dataflow sweeps ------------------------------------------------
// Items are the nodes of all levels in dependency order; a warp claims the
// next item with an atomic ticket (reset before each launch), waits on
// the flags of the nodes it reads, computes exactly like k_up_level /
// k_down_level, and publishes its node's flag.  Claimed items only ever wait
// for items claimed earlier, whose warps are running: deadlock-free at any
// residency.  Flags hold an epoch (2e: up done, 2e + 1: down done) so they are
// never cleared.  Node vectors written by other SMs are read with ld.cg.
struct SweepLevel {
  const double* T;   // transfers of the child level (block (c - cbegin) * stride)
  int64_t stride, cbegin;
  int ldc, kc, kp, l;  // child level l, parent level l - 1
  const double* in;  // up: x^ of level l;   down: y^ of level l - 1
  double* out;       // up: x^ of level l-1; down: y^ of level l
  int64_t n, i0;     // items (up: parents i0.., down: children i0..)
};
struct SweepTable {
  SweepLevel L[kMaxLevels];
  int64_t start[kMaxLevels + 1];
  int nl;
  int q;  // up: the deepest child level (its x^ is input); down: the top parent level (its y^ is input)
};

using df::node_id;
using df::set_flag;
using df::wait_flag;

__device__ __forceinline__ int claim(unsigned long long* ticket, unsigned long long base) {
  return int(df::claim(ticket) - int64_t(base));
}

__global__ void __launch_bounds__(kThreads, 2) k_up_fused(const __grid_constant__ SweepTable S,
                                                       uint32_t* __restrict__ flag,
                                                       const unsigned long long* __restrict__ ep,
                                                       unsigned long long* __restrict__ ticket,
                                                       unsigned long long base) {
  const uint32_t epoch = 2u * uint32_t(__ldcg(ep));  // up flags of this mat-vec
  const int r = 2 * lane_id();
  const int64_t total = S.start[S.nl];
  // bulk L2 prefetch of an item's two child transfers ahead of its flag waits
  // (C4 mat-vec 12.41 -> 12.34 ms, C2 1.850 -> 1.815 ms; three A/B pairs)
  auto prefetch = [&](int64_t i) {
    if (kSweepAhead < 0 || i >= total || lane_id() != 0) return;
    int e = 0;
    while (i >= S.start[e + 1]) ++e;
    const SweepLevel& L = S.L[e];
    if (L.kc > 0 && L.kp > 0) {
      const double* pf = L.T + (2 * (L.i0 + (i - S.start[e])) - L.cbegin) * L.stride;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf), "r"(uint32_t(2 * L.stride * 8)) : "memory");
    }
  };
  int64_t next = claim(ticket, base);
  prefetch(next);
  for (;;) {
    const int64_t it = next;
    if (it >= total) break;
    if (kSweepAhead > 0) {
      next = claim(ticket, base);
      prefetch(next);
    }
    int e = 0;
    while (it >= S.start[e + 1]) ++e;
    const SweepLevel& L = S.L[e];
    const int64_t p = L.i0 + (it - S.start[e]);
    if (L.l < S.q) {  // children computed by this launch (level q: input, e.g. by k_up_leaf)
      wait_flag(flag + node_id(L.l, 2 * p), epoch);
      wait_flag(flag + node_id(L.l, 2 * p + 1), epoch);
    }
    if (L.kp > 0) {
      double o0 = 0.0, o1 = 0.0;
      if (L.kc > 0) {
        const double* x0 = L.in + (2 * p) * L.kc;
        const double* x1 = x0 + L.kc;
        const double v0 = r < L.kc ? __ldcg(x0 + r) : 0.0, v1 = r + 1 < L.kc ? __ldcg(x0 + r + 1) : 0.0;
        const double w0 = r < L.kc ? __ldcg(x1 + r) : 0.0, w1 = r + 1 < L.kc ? __ldcg(x1 + r + 1) : 0.0;
        const double* A = L.T + (2 * p - L.cbegin) * L.stride;
        o0 = gemvT_group<true>(A, A + L.stride, L.ldc, L.kp, 0, v0, v1, w0, w1, r < L.ldc);
        o1 = gemvT_group<true>(A, A + L.stride, L.ldc, L.kp, 1, v0, v1, w0, w1, r < L.ldc);
      }
      if (r < L.kp) L.out[p * L.kp + r] = o0;
      if (r + 1 < L.kp) L.out[p * L.kp + r + 1] = o1;
    }
    set_flag(flag + node_id(L.l - 1, p), epoch);
    if (kSweepAhead <= 0) {
      next = claim(ticket, base);
      prefetch(next);
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_down_fused(const __grid_constant__ SweepTable S,
                                                         uint32_t* __restrict__ flag,
                                                         const unsigned long long* __restrict__ ep,
                                                         unsigned long long* __restrict__ ticket,
                                                         unsigned long long base) {
  const uint32_t epoch = 2u * uint32_t(__ldcg(ep)) + 1u;  // down flags of this mat-vec
  const int r = 2 * lane_id();
  const int64_t total = S.start[S.nl];
  auto prefetch = [&](int64_t i) {  // the transfer block, ahead of the flag wait (see k_up_fused)
    if (kSweepAhead < 0 || i >= total || lane_id() != 0) return;
    int e = 0;
    while (i >= S.start[e + 1]) ++e;
    const SweepLevel& L = S.L[e];
    if (L.kc > 0 && L.kp > 0) {
      const double* pf = L.T + (L.i0 + (i - S.start[e]) - L.cbegin) * L.stride;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf), "r"(uint32_t(L.stride * 8)) : "memory");
    }
  };
  int64_t next = claim(ticket, base);
  prefetch(next);
  for (;;) {
    const int64_t it = next;
    if (it >= total) break;
    if (kSweepAhead > 0) {
      next = claim(ticket, base);
      prefetch(next);
    }
    int e = 0;
    while (it >= S.start[e + 1]) ++e;
    const SweepLevel& L = S.L[e];
    const int64_t c = L.i0 + (it - S.start[e]);
    if (L.l - 1 > S.q) wait_flag(flag + node_id(L.l - 1, c >> 1), epoch);  // (top parent level: input)
    if (L.kc > 0 && L.kp > 0) {
      const double* yp = L.in + (c >> 1) * L.kp;
      const double a0 = r < L.kp ? __ldcg(yp + r) : 0.0, a1 = r + 1 < L.kp ? __ldcg(yp + r + 1) : 0.0;
      double acc0, acc1;
      gemvN_pair(L.T + (c - L.cbegin) * L.stride, L.ldc, L.kp, a0, a1, r < L.ldc, acc0, acc1);
      double* y = L.out + c * L.kc;
      if (r < L.kc) y[r] = acc0 + __ldcg(y + r);
      if (r + 1 < L.kc) y[r + 1] = acc1 + __ldcg(y + r + 1);
    }
    set_flag(flag + node_id(L.l, c), epoch);
    if (kSweepAhead <= 0) {
      next = claim(ticket, base);
      prefetch(next);
    }
  }
}

__global__ void k_epoch_next(unsigned long long* e) { *e += 1; }

struct LayerDesc {
  const double* val;
  const int32_t* rp;
  const int32_t* ci;
  const double* x;
  double* y;
  int64_t stride;
  int br, bc, ld;
  int tma;  // rows of this layer go to k_bsr_tma (full 64 x 64 blocks), else to k_bsr
};
struct LayerTable {
  LayerDesc L[kMaxLevels + 2];
};

// Fused block-sparse multiply over every (layer, block row) work item:
// y_r = sum_b B_b x_{col(b)} in col_idx order (bsr.hpp:50-73, beta = 0).
// A row of ld/2 lanes covers one block column; small blocks put
// G = 32 / (ld/2) column groups side by side and reduce them at the end.
__global__ void __launch_bounds__(kThreads) k_bsr(const __grid_constant__ LayerTable T,
                                                  const uint32_t* __restrict__ work,
                                                  int64_t nwork) {
  const int lane = lane_id();
  for (int64_t it = warp_global(); it < nwork; it += warp_count()) {
    const uint32_t u = __ldg(work + it);
    const LayerDesc& D = T.L[u >> kLayerShift];
    if (D.tma) continue;  // streamed by k_bsr_tma
    const int row = int(u & ((1u << kLayerShift) - 1));
    const int lpc = D.ld >> 1;
    const int G = 32 / lpc;
    const int grp = lane / lpc;
    const int pr = lane - grp * lpc;
    const bool act = grp < G;
    const int r = 2 * pr;
    int b = __ldg(D.rp + row);
    const int b1 = __ldg(D.rp + row + 1);
    double y0 = 0.0, y1 = 0.0;
    int col = b < b1 ? __ldg(D.ci + b) : 0;
    for (; b < b1; ++b) {
      const double* xs = D.x + int64_t(col) * D.bc;
      const double xr0 = lane < D.bc ? __ldg(xs + lane) : 0.0;
      const double xr1 = lane + 32 < D.bc ? __ldg(xs + lane + 32) : 0.0;
      col = b + 1 < b1 ? __ldg(D.ci + b + 1) : 0;
      const double* blk = D.val + int64_t(b) * D.stride + r;
      for (int j0 = 0; j0 < D.bc; j0 += 8 * G) {
        double2 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int j = j0 + q * G + grp;
          v[q] = (act && j < D.bc) ? ld_stream(blk + int64_t(j) * D.ld) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int jb = j0 + q * G;  // warp-uniform
          const int j = jb + grp;
          // bc > 32 implies G == 1: active lanes have j == jb, and the source
          // lane's register choice must depend on the uniform jb only.
          const double xj = __shfl_sync(kFull, jb < 32 ? xr0 : xr1, j & 31);
          if (j < D.bc) {
            y0 += v[q].x * xj;
            y1 += v[q].y * xj;
          }
        }
      }
    }
    if (G > 1) {
      double t0 = y0, t1 = y1;
      for (int g = 1; g < G; ++g) {
        t0 += __shfl_down_sync(kFull, y0, g * lpc);
        t1 += __shfl_down_sync(kFull, y1, g * lpc);
      }
      y0 = t0;
      y1 = t1;
    }
    if (act && grp == 0) {
      double* yr = D.y + int64_t(row) * D.br;
      if (r < D.br) yr[r] = y0;
      if (r + 1 < D.br) yr[r + 1] = y1;
    }
  }
}

// The same product with the blocks streamed by the tensor-memory accelerator
// (k_bsr_tma): a read-only 64 GB stream measured 7.44 TB/s through a TMA ring
// against 7.06-7.09 TB/s with 16-byte evict-first loads
// (tools/microbench/tma_stream.cu).  One CTA walks its rows of the LPT list; a
// producer lane loads each block as one tensor-map box of 64 x 64 (zero fill
// out of range; column-major, 64-double column stride) plus the x segment of
// its block column (1D tensor map, from an even element: TMA boxes start
// 16-byte aligned), completion on the stage's mbarrier; four consumer warps
// own a box each: lane (rp, cq) accumulates rows 16w + 2rp and 16w + 2rp + 1
// over the columns [16cq, 16cq + 16), one 16-byte shared load per column (a
// box line holds the 16 rows of one column; a quarter warp reads 8 distinct
// swizzled chunks of a line: conflict-free), the column quarters meet by two
// shuffles at the end of the row.  (One row per lane with 8-byte loads: 2-3%
// slower, twice the shared loads.)  Measured at C4, ms per mat-vec: one
// unswizzled 64 x 64 box per block = four swizzled 16 x 64 boxes (11.94);
// stages x CTAs/SM 2 x 2 12.0, 4 x 1 12.0, 1 x 4 12.04, 2 x 3 12.45, 3 x 2
// 12.47 -- four blocks (128 KB) in flight per SM is the sweet spot.
#ifndef H2B_BSTAGES
#define H2B_BSTAGES 2
#endif
#ifndef H2B_BBOX64
#define H2B_BBOX64 1
#endif
constexpr bool kBBox64 = H2B_BBOX64;  // one unswizzled 64 x 64 box per block (else 4 swizzled 16 x 64)
#ifndef H2B_BCTAS
#define H2B_BCTAS 2
#endif
constexpr int kBStages = H2B_BSTAGES, kBCtas = H2B_BCTAS, kBWarps = 4;
constexpr int kBBox = 16 * 64;
constexpr int kBXBox = 66;  // x segment: 64 doubles from an even start (one more when it is odd)
constexpr int kBStage = 4 * kBBox + 128;  // + the x segment, padded: every stage 1024-byte aligned (swizzle)
constexpr size_t kBSmem = size_t(kBStages) * kBStage * sizeof(double) + 1024;
struct TmaTable {
  CUtensorMap S[kMaxLevels + 2];  // per layer: 3D {ld, bc, nb} blocks, box {64, 64, 1}
  CUtensorMap X[2];               // [0] x^ pool, [1] x_c (dense layer): 1D, box 66
  int64_t xrow0[kMaxLevels + 2];  // per layer: offset of its x^ in X[0]
  int dense;                      // the dense layer's index
};

__global__ void __launch_bounds__(32 * (kBWarps + 1), kBCtas) k_bsr_tma(const __grid_constant__ LayerTable T,
                                                                     const __grid_constant__ TmaTable M,
                                                                     const uint32_t* __restrict__ work,
                                                                     int64_t nwork) {
  using namespace tma;
  extern __shared__ double ring_raw[];
  double* ring = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(ring_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kBStages], empty[kBStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < kBStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kBWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int stage = 0;
  uint32_t phase = 0;
  if (warp == kBWarps) {  // producer: one elected lane
    if (lane == 0) {
      const uint64_t pol_s = l2_policy_evict_first(), pol_x = l2_policy_evict_last();
      for (int64_t it = blockIdx.x; it < nwork; it += gridDim.x) {
        const uint32_t u = __ldg(work + it);
        const int li = int(u >> kLayerShift);
        const LayerDesc& D = T.L[li];
        if (!D.tma) continue;  // small blocks: k_bsr
        const int row = int(u & ((1u << kLayerShift) - 1));
        const int b0 = __ldg(D.rp + row), b1 = __ldg(D.rp + row + 1);
        const CUtensorMap* xm = &M.X[li == M.dense ? 1 : 0];
        for (int b = b0; b < b1; ++b) {
          const int col = __ldg(D.ci + b);
          mbar_wait(&empty[stage], phase ^ 1u);
          if (D.br > 0 && D.bc > 0) {
            // 4 boxes + the x segment; the segment starts at an even element
            // (a TMA box must start 16-byte aligned): consumers skip x0 & 1
            mbar_expect_tx(&full[stage], uint32_t((4 * kBBox + kBXBox) * sizeof(double)));
            double* dst = ring + stage * kBStage;
            if (kBBox64)
              tma_3d(dst, &M.S[li], 0, b, &full[stage], pol_s);
            else
#pragma unroll
              for (int h = 0; h < 4; ++h) tma_3d(dst + h * kBBox, &M.S[li], 16 * h, b, &full[stage], pol_s);
            const int64_t x0 = M.xrow0[li] + int64_t(col) * D.bc;
            tma_1d(dst + 4 * kBBox, xm, int(x0 & ~int64_t(1)), &full[stage], pol_x);
          } else {  // rank-0 blocks: nothing to load
            mbar_arrive(&full[stage]);
          }
          if (++stage == kBStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    return;
  }
  // lane = 8 cq + rp: rows 16w + 2rp, 16w + 2rp + 1 (one 16-byte load per
  // column: two rows of a box line), columns [16cq, 16cq + 16)
  const int rp = lane & 7, cq = lane >> 3;
  const int r = 16 * warp + 2 * rp;
  for (int64_t it = blockIdx.x; it < nwork; it += gridDim.x) {
    const uint32_t u = __ldg(work + it);
    const LayerDesc& D = T.L[u >> kLayerShift];
    if (!D.tma) continue;
    const int row = int(u & ((1u << kLayerShift) - 1));
    const int b0 = __ldg(D.rp + row), b1 = __ldg(D.rp + row + 1);
    const int br = D.br, bc = D.bc;
    const bool live = 16 * warp < br && bc > 0;  // warp-uniform
    double a0[2] = {0.0, 0.0}, a1[2] = {0.0, 0.0};  // rows r, r + 1; two FMA chains each
    for (int b = b0; b < b1; ++b) {
      const int xo = int((M.xrow0[u >> kLayerShift] + int64_t(__ldg(D.ci + b)) * bc) & 1);
      mbar_wait(&full[stage], phase);
      if (live) {
        const double* Sx = ring + stage * kBStage + (kBBox64 ? 16 * warp : warp * kBBox);
        const double* xs = ring + stage * kBStage + 4 * kBBox + xo + 16 * cq;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int j = 16 * cq + jj;
          if (j < bc) {
            const double2 sv = *reinterpret_cast<const double2*>(Sx + (kBBox64 ? 64 * j + 2 * rp : swz(j, 2 * rp)));
            const double xj = xs[jj];
            a0[jj & 1] = fma(sv.x, xj, a0[jj & 1]);
            a1[jj & 1] = fma(sv.y, xj, a1[jj & 1]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kBStages) {
        stage = 0;
        phase ^= 1u;
      }
    }
    double y0 = a0[0] + a0[1], y1 = a1[0] + a1[1];
    y0 += __shfl_xor_sync(kFull, y0, 8);
    y1 += __shfl_xor_sync(kFull, y1, 8);
    y0 += __shfl_xor_sync(kFull, y0, 16);
    y1 += __shfl_xor_sync(kFull, y1, 16);
    if (cq == 0) {
      double* yr = D.y + int64_t(row) * br;
      if (r < br) yr[r] = y0;
      if (r + 1 < br) yr[r + 1] = y1;
    }
  }
}

// block_sparse_mv(L, x, y, alpha, beta) for one generic layer (any block_rows x
// block_cols, brows / bcols <= 128), in the reference's exact arithmetic
// (bsr.hpp:50-73): y_r = (beta == 0 ? 0 : beta y_r), then for every block in
// col_idx order and every column j, y_r += col_j * (alpha x_j) -- unfused
// multiply and add, so the result is bitwise the reference's.  Warp per block
// row, lane per row pair; the phase API's instance, not the mat-vec's.
__global__ void __launch_bounds__(kThreads) k_bsr_exact(const double* __restrict__ val, int64_t stride, int ld,
                                                        int br, int bc, const int32_t* __restrict__ rp,
                                                        const int32_t* __restrict__ ci, int64_t rows,
                                                        const double* __restrict__ x, double* __restrict__ y,
                                                        double alpha, double beta) {
  const int lane = lane_id();
  for (int64_t r = warp_global(); r < rows; r += warp_count()) {
    double* yr = y + r * br;
    double acc[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int i = lane + 32 * h;
      acc[h] = (i < br && beta != 0.0) ? __dmul_rn(beta, yr[i]) : 0.0;
    }
    for (int b = rp[r]; b < rp[r + 1]; ++b) {
      const double* blk = val + int64_t(b) * stride;
      const double* xs = x + int64_t(ci[b]) * bc;
      for (int j = 0; j < bc; ++j) {
        const double xv = __dmul_rn(alpha, __ldg(xs + j));
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int i = lane + 32 * h;
          if (i < br) acc[h] = __dadd_rn(acc[h], __dmul_rn(blk[i + int64_t(j) * ld], xv));
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 4; ++h)
      if (lane + 32 * h < br) yr[lane + 32 * h] = acc[h];
  }
}

__global__ void k_gather(const int32_t* __restrict__ perm, const double* __restrict__ x,
                         double* __restrict__ xc, int64_t n) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n;
       t += int64_t(gridDim.x) * blockDim.x)
    xc[t] = x[perm[t]];
}

__global__ void k_scatter(const int32_t* __restrict__ perm, const double* __restrict__ ys,
                          double* __restrict__ y, int64_t n, double alpha, double beta) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n;
       t += int64_t(gridDim.x) * blockDim.x) {
    double* o = y + perm[t];
    *o = alpha * ys[t] + (beta == 0.0 ? 0.0 : beta * *o);
  }
}

__global__ void k_repack(const double* __restrict__ src, int64_t ss, int ld_src,
                         double* __restrict__ dst, int64_t sd, int ld_dst, int rows, int cols,
                         int64_t count) {
  const int64_t per = int64_t(ld_dst) * cols;
  const int64_t total = per * count;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = e / per;
    const int64_t w = e - b * per;
    const int j = int(w / ld_dst);
    const int i = int(w - int64_t(j) * ld_dst);
    dst[b * sd + int64_t(j) * ld_dst + i] = i < rows ? src[b * ss + int64_t(j) * ld_src + i] : 0.0;
  }
}

int sm_count() {
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return sms;
}

// Grid for a grid-stride warp loop over `items` warps of work: at most 8
// resident 256-thread CTAs per SM.
unsigned warp_grid(int64_t items) {
  const int64_t want = (items + 7) / 8;
  const int64_t cap = int64_t(sm_count()) * 8;
  return unsigned(std::max<int64_t>(1, std::min(want, cap)));
}

unsigned flat_grid(int64_t n) {
  const int64_t want = (n + kThreads - 1) / kThreads;
  const int64_t cap = int64_t(sm_count()) * 16;
  return unsigned(std::max<int64_t>(1, std::min(want, cap)));
}

}  // namespace

void launch_up_leaf(const Matrix& B, const double* x, double* xc, double* xhat, cudaStream_t s,
                    bool cluster_order) {
  if (big_basis(B)) return launch_up_leaf_big(B, x, xc, xhat, s, cluster_order);
  const int64_t nl = B.own_count(B.q);
  k_up_leaf<<<warp_grid(nl), kThreads, 0, s>>>(x, cluster_order ? nullptr : B.perm.p, B.leaf.p, B.m, B.ldm,
                                               B.rank[B.q], nl, B.own_begin(B.q), xc, xhat + B.vec_off[B.q]);
  H2B_CUDA(cudaGetLastError());
}

void launch_up_level(const Matrix& B, int l, double* xhat, cudaStream_t s, int64_t p0, int64_t p1) {
  const int kc = B.rank[l], kp = B.rank[l - 1];
  if (p1 < 0) p1 = B.nodes(l - 1);
  double* xp = xhat + B.vec_off[l - 1];
  const int64_t np = p1 - p0;
  if (kp == 0 || np <= 0) return;
  if (kc == 0) {
    H2B_CUDA(cudaMemsetAsync(xp + p0 * kp, 0, size_t(np) * kp * sizeof(double), s));
    return;
  }
  if (big_basis(B)) return launch_up_level_big(B, l, xhat, s, p0, p1);
  k_up_level<<<warp_grid(np), kThreads, 0, s>>>(B.transfer.p + B.tr_off[l], B.ld(l), kc, kp, p0, p1,
                                                B.tr_begin(l), xhat + B.vec_off[l], xp);
  H2B_CUDA(cudaGetLastError());
}

namespace {
unsigned persistent_grid(const void* kernel) {
  int per_sm = 0;
  H2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0));
  return unsigned(std::max(1, per_sm) * sm_count());
}
}  // namespace

void sweep_begin(Work& w, const Matrix& A, cudaStream_t s) {
  const int64_t nodes = int64_t(4) << A.q;  // 2^(q+1) - 1 nodes, x 2 for the split 16-vector sweeps
  if (w.flag.n < size_t(nodes) || !w.ticket.p) {
    // stream-ordered zeroing: the kernels of this mat-vec run after it
    w.flag.alloc(nodes);
    H2B_CUDA(cudaMemsetAsync(w.flag.p, 0, nodes * sizeof(uint32_t), s));
    w.ticket.alloc(3);  // [0] up ticket, [1] down ticket, [2] epoch
    H2B_CUDA(cudaMemsetAsync(w.ticket.p, 0, 3 * sizeof(unsigned long long), s));
  }
  // this mat-vec's epoch (up flags 2e, down flags 2e + 1), advanced on the
  // device so that a captured CUDA graph replays correctly
  k_epoch_next<<<1, 1, 0, s>>>(w.ticket.p + 2);
  H2B_CUDA(cudaGetLastError());
}

void launch_up_fused(Work& w, const Matrix& B, double* xhat, cudaStream_t s, int l_hi, int l_lo, bool own) {
  if (big_basis(B)) {  // blocks > 64: one launch per level (k_hmv_big.cu)
    for (int l = l_hi; l >= l_lo; --l)
      launch_up_level(B, l, xhat, s, own ? B.own_begin(l - 1) : 0, own ? B.own_end(l - 1) : B.nodes(l - 1));
    return;
  }
  SweepTable T{};
  T.q = l_hi;
  int64_t tot = 0;
  for (int l = l_hi; l >= l_lo; --l) {
    SweepLevel& L = T.L[T.nl];
    L.T = B.transfer.p + B.tr_off[l];
    L.stride = B.tr_stride(l);
    L.cbegin = B.tr_begin(l);
    L.ldc = B.ld(l);
    L.kc = B.rank[l];
    L.kp = B.rank[l - 1];
    L.l = l;
    L.in = xhat + B.vec_off[l];
    L.out = xhat + B.vec_off[l - 1];
    L.i0 = own ? B.own_begin(l - 1) : 0;
    L.n = own ? B.own_count(l - 1) : B.nodes(l - 1);
    T.start[T.nl] = tot;
    tot += L.n;
    ++T.nl;
  }
  T.start[T.nl] = tot;
  if (tot == 0) return;
  require(w.flag.n >= (size_t(2) << B.q), "launch_up_fused: sweep_begin missing");
  H2B_CUDA(cudaMemsetAsync(w.ticket.p, 0, sizeof(unsigned long long), s));
  k_up_fused<<<persistent_grid((const void*)k_up_fused), kThreads, 0, s>>>(T, w.flag.p, w.ticket.p + 2, w.ticket.p,
                                                                          0ull);
  H2B_CUDA(cudaGetLastError());
}

void launch_down_fused(Work& w, const Matrix& A, double* yhat, cudaStream_t s, bool own) {
  if (big_basis(A)) {  // blocks > 64: one launch per level (k_hmv_big.cu)
    for (int l = 1; l <= A.q; ++l)
      launch_down_level(A, l, yhat, s, own ? A.own_begin(l) : 0, own ? A.own_end(l) : A.nodes(l));
    return;
  }
  const int q = A.q;
  SweepTable T{};
  T.q = 0;  // the root's y^ is final (after the coupling multiply)
  int64_t tot = 0;
  for (int l = 1; l <= q; ++l) {
    SweepLevel& L = T.L[T.nl];
    L.T = A.transfer.p + A.tr_off[l];
    L.stride = A.tr_stride(l);
    L.cbegin = A.tr_begin(l);
    L.ldc = A.ld(l);
    L.kc = A.rank[l];
    L.kp = A.rank[l - 1];
    L.l = l;
    L.in = yhat + A.vec_off[l - 1];
    L.out = yhat + A.vec_off[l];
    L.i0 = own ? A.own_begin(l) : 0;
    L.n = own ? A.own_count(l) : A.nodes(l);
    T.start[T.nl] = tot;
    tot += L.n;
    ++T.nl;
  }
  T.start[T.nl] = tot;
  if (tot == 0) return;
  require(w.flag.n >= (size_t(2) << A.q), "launch_down_fused: sweep_begin missing");
  H2B_CUDA(cudaMemsetAsync(w.ticket.p + 1, 0, sizeof(unsigned long long), s));
  k_down_fused<<<persistent_grid((const void*)k_down_fused), kThreads, 0, s>>>(T, w.flag.p, w.ticket.p + 2,
                                                                              w.ticket.p + 1, 0ull);
  H2B_CUDA(cudaGetLastError());
}

void launch_down_level(const Matrix& A, int l, double* yhat, cudaStream_t s, int64_t c0, int64_t c1) {
  const int kc = A.rank[l], kp = A.rank[l - 1];
  if (c1 < 0) c1 = A.nodes(l);
  const int64_t nc = c1 - c0;
  if (kc == 0 || kp == 0 || nc <= 0) return;
  if (big_basis(A)) return launch_down_level_big(A, l, yhat, s, c0, c1);
  k_down_level<<<warp_grid(nc), kThreads, 0, s>>>(A.transfer.p + A.tr_off[l], A.ld(l), kc, kp, c0, c1,
                                                  A.tr_begin(l), yhat + A.vec_off[l - 1], yhat + A.vec_off[l]);
  H2B_CUDA(cudaGetLastError());
}

void launch_down_leaf(const Matrix& A, const double* yhat, const double* yc, double* y, double alpha,
                      double beta, bool to_user, cudaStream_t s) {
  if (big_basis(A)) return launch_down_leaf_big(A, yhat, yc, y, alpha, beta, to_user, s);
  const int64_t nl = A.own_count(A.q);
  k_down_leaf<<<warp_grid(nl), kThreads, 0, s>>>(A.leaf.p, A.ldm, A.m, A.rank[A.q], nl, A.own_begin(A.q),
                                                 yhat + A.vec_off[A.q], yc, A.perm.p, y, alpha, beta,
                                                 to_user ? 1 : 0);
  H2B_CUDA(cudaGetLastError());
}

void launch_bsr(const Matrix& A, const uint32_t* work, int64_t nwork, const double* xdense,
                double* ydense, const double* xh, double* yh, cudaStream_t s, const Matrix* xb) {
  if (nwork == 0) return;
  if (big_matrix(A)) return launch_bsr_big(A, work, nwork, xdense, ydense, xh, yh, s, xb);
  const std::vector<int64_t>& xoff = xb ? xb->vec_off : A.vec_off;
  LayerTable T{};
  for (int l = 0; l <= A.q; ++l) {
    const Layer& L = A.cpl[l];
    LayerDesc& d = T.L[l];
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
  LayerDesc& d = T.L[A.q + 1];
  d.val = A.dense.val;
  d.rp = A.dense.rp;
  d.ci = A.dense.ci;
  d.x = xdense;
  d.y = ydense;
  d.stride = A.dense.block_stride();
  d.br = A.dense.br;
  d.bc = A.dense.bc;
  d.ld = std::max(2, A.dense.ld);
  // the tensor maps need 16-byte aligned bases (user device pointers of the
  // phase API may not be): the register-fed kernel takes any alignment
  const auto aligned = [](const double* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  // k_bsr_tma (3D block views, a block costs only its own bytes) when the big
  // blocks (>= 48 x 48 entries) carry at least 3/4 of the bytes, else k_bsr for
  // everything: small blocks keep too few bytes in flight in a 4-block ring,
  // and splitting a launch by layer loses the interleaving of big and small
  // rows.  ms per mat-vec, same box (tools/microbench/hmv_configs.py): C3
  // 8.65-8.66 on the ring vs 9.06-9.12 register-fed; C2 (k = 36, half the
  // bytes in 36 x 36 blocks) 2.00 vs 1.92 (2.01 split by layer); C3 compressed
  // at 1e-6 (ranks 34-60) 6.16-6.21 vs 6.09-6.14.  k_bsr also takes layers
  // whose x is absent (phase calls) and misaligned phase-API pointers.
  double big = 0.0, all = 0.0;
  for (int l = 0; l <= A.q + 1; ++l) {
    const Layer& L = l <= A.q ? A.cpl[l] : A.dense;
    const double b = double(L.nb) * L.ld * L.bc;
    all += b;
    if (L.ld * L.bc >= 48 * 48) big += b;
  }
  bool any_tma = false;
  if (kTmaBsr && aligned(xh) && aligned(xdense) && (H2B_TMA_FORCE || big >= 0.75 * all))
    for (int l = 0; l <= A.q + 1; ++l) {
      const Layer& L = l <= A.q ? A.cpl[l] : A.dense;
      T.L[l].tma = l <= A.q ? xh != nullptr : xdense != nullptr;
      any_tma = any_tma || (T.L[l].tma && L.nb > 0);
    }
  if (!any_tma)
    for (int l = 0; l <= A.q + 1; ++l) T.L[l].tma = 0;
  bool any_reg = false;
  for (int l = 0; l <= A.q + 1; ++l) {
    const Layer& L = l <= A.q ? A.cpl[l] : A.dense;
    any_reg = any_reg || (!T.L[l].tma && L.rows > 0);
  }
  if (any_tma) {
    TmaTable M{};
    if (xh) tma::encode_1d(&M.X[0], xh, uint64_t(std::max<int64_t>(1, xoff[A.q + 1])), kBXBox);
    if (xdense) tma::encode_1d(&M.X[1], xdense, uint64_t(std::max(1, A.n)), kBXBox);
    M.dense = A.q + 1;
    for (int l = 0; l <= A.q + 1; ++l) {
      const Layer& L = l <= A.q ? A.cpl[l] : A.dense;
      M.xrow0[l] = l <= A.q ? xoff[l] : 0;
      if (T.L[l].tma && L.nb > 0)
        tma::encode_blocks3d(&M.S[l], L.val, uint64_t(std::max(2, L.ld)), uint64_t(L.bc), uint64_t(L.nb),
                             kBBox64 ? 64 : 16, 64, !kBBox64);
    }
    H2B_CUDA(cudaFuncSetAttribute(k_bsr_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kBSmem)));
    k_bsr_tma<<<unsigned(std::min<int64_t>(nwork, int64_t(kBCtas) * sm_count())), 32 * (kBWarps + 1), kBSmem, s>>>(
        T, M, work, nwork);
    H2B_CUDA(cudaGetLastError());
  }
  if (any_reg) k_bsr<<<warp_grid(nwork), kThreads, 0, s>>>(T, work, nwork);
  H2B_CUDA(cudaGetLastError());
}

void launch_bsr_exact(const Layer& L, const double* x, double* y, double alpha, double beta, cudaStream_t s) {
  if (L.rows == 0 || L.br == 0) return;
  k_bsr_exact<<<warp_grid(L.rows), kThreads, 0, s>>>(L.val, L.block_stride(), std::max(1, L.ld), L.br, L.bc, L.rp,
                                                     L.ci, L.rows, x, y, alpha, beta);
  H2B_CUDA(cudaGetLastError());
}

void launch_gather(const int32_t* perm, const double* x, double* xc, int64_t n, cudaStream_t s) {
  k_gather<<<flat_grid(n), kThreads, 0, s>>>(perm, x, xc, n);
  H2B_CUDA(cudaGetLastError());
}

void launch_scatter(const int32_t* perm, const double* ys, double* y, int64_t n, double alpha, double beta,
                    cudaStream_t s) {
  if (n == 0) return;
  k_scatter<<<flat_grid(n), kThreads, 0, s>>>(perm, ys, y, n, alpha, beta);
  H2B_CUDA(cudaGetLastError());
}

void launch_repack(const double* src, int64_t ss, int ld_src, double* dst, int64_t sd, int ld_dst,
                   int rows, int cols, int64_t count, cudaStream_t s) {
  const int64_t total = int64_t(ld_dst) * cols * count;
  if (total == 0) return;
  k_repack<<<flat_grid(total), kThreads, 0, s>>>(src, ss, ld_src, dst, sd, ld_dst, rows, cols,
                                                 count);
  H2B_CUDA(cudaGetLastError());
}

std::vector<uint32_t> make_work_list(const std::vector<const Layer*>& layers) {
  struct Item {
    uint32_t code;
    int32_t cost;
  };
  std::vector<Item> items;
  for (size_t li = 0; li < layers.size(); ++li) {
    const Layer* L = layers[li];
    if (!L) continue;
    const int64_t r1 = L->row1 < 0 ? L->rows : L->row1;
    for (int64_t r = L->row0; r < r1; ++r) {
      const int32_t nb = L->h_rp.empty() ? 0 : L->h_rp[r + 1] - L->h_rp[r];
      // cost ~ bytes of the row; empty rows still write zeros
      const int64_t bytes = int64_t(nb) * L->ld * L->bc;
      items.push_back({uint32_t(li) << kLayerShift | uint32_t(r), int32_t(std::min<int64_t>(bytes, 1 << 30))});
    }
  }
  std::stable_sort(items.begin(), items.end(),
                   [](const Item& a, const Item& b) { return a.cost > b.cost; });
  std::vector<uint32_t> out(items.size());
  for (size_t i = 0; i < items.size(); ++i) out[i] = items[i].code;
  return out;
}

}  // namespace h2b
