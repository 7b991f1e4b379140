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
// straight into the A fragments with evict-first 128-bit loads:
//   * transposed products (V^T x, F^T x^) pair their k-steps: lane k-slot fk
//     of a pair of k-steps covers the two ADJACENT contraction rows 2j, 2j+1
//     (j = j0 + fk), so one 16-byte load feeds two DMMAs and a block column is
//     read in 64-byte pieces (the 8-byte form fetched every sector twice);
//   * untransposed products (E y^, U y^, S x^) pair their row tiles: tiles
//     2z / 2z+1 hold the rows 16z + 2fr / 16z + 2fr + 1, one 16-byte load per
//     lane and k-step feeds both.
// Phases: k_up_leaf_mv (perm gather fused, coalesced through shared memory),
// k_up_fused_mv (levels q..1, one dataflow launch), k_bsr_mv (dense + every
// coupling level), k_down_fused_mv (levels 1..q, one dataflow launch),
// k_down_leaf_mv (alpha/beta scatter fused, coalesced through shared memory).
#include "dataflow.cuh"
#include "h2b_internal.hpp"
#include "tma.cuh"

#ifndef H2B_TSTAGES
#define H2B_TSTAGES 2
#endif
#ifndef H2B_TCTAS
#define H2B_TCTAS 2
#endif

#include <algorithm>

namespace h2b {
namespace {

using namespace tma;

constexpr int kThreads = 256;
constexpr int NV = 16;        // vectors per pass (2 DMMA column tiles)
constexpr int kLeafWarps = 4; // leaf kernels: 4 warps x 8 KB shared panel
#ifndef H2B_MV_PREFETCH
#define H2B_MV_PREFETCH 1
#endif
// Bulk L2 prefetch of the downsweep's transfer block ahead of its flag wait
// (C4: k_down_fused_mv 1.49 -> 1.41 ms).  The same for the upsweep and the
// leaf kernels (the next leaf of the warp) raised their DRAM reads 1.5-1.7x
// and their times (profiles/r02_mv16_launches.txt): not used there.
constexpr bool kPrefetch = H2B_MV_PREFETCH;
// fused 16-vector sweeps: claim the next item before this one (1) or after it
// (0).  C4, same box: k_down_fused_mv 1.50-1.53 ms claiming ahead, 1.37-1.38
// after (an item claimed ahead holds back the items that wait on it);
// k_up_fused_mv 1.25 either way.
#ifndef H2B_MV_CLAIM_AHEAD
#define H2B_MV_CLAIM_AHEAD 0
#endif
constexpr bool kMvClaimAhead = H2B_MV_CLAIM_AHEAD;
// bulk L2 prefetch of the upsweep items' child transfers: measured 1.25 ->
// 1.55 ms (C4, claim-after order too); off
#ifndef H2B_MV_UP_PREFETCH
#define H2B_MV_UP_PREFETCH 0
#endif
constexpr bool kUpPrefetch = H2B_MV_UP_PREFETCH;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int64_t warp_global() {
  return (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
}
__device__ __forceinline__ int64_t warp_count() { return (int64_t(gridDim.x) * blockDim.x) >> 5; }

// Bulk L2 prefetch of a contiguous matrix block (16-byte aligned, size a
// multiple of 16): the TMA unit streams it into L2 while the warp waits on
// flags or works on the previous block, beyond what its registers can hold
// in flight.
__device__ __forceinline__ void prefetch_l2(const double* p, int64_t count) {
  if ((threadIdx.x & 31) == 0 && count > 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(uint32_t(count * sizeof(double)))
                 : "memory");
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Streaming 16-byte matrix loads.  POL: 0 evict-first, 1 non-coherent,
// 2 non-coherent + L2::256B prefetch, 3 evict-first + L2::256B prefetch
// (measured: see hmv_multi_device).
template <int POL = 0>
__device__ __forceinline__ double2 ld_stream2(const double* p) {
  if (POL == 0) return __ldcs(reinterpret_cast<const double2*>(p));
  if (POL == 1) return __ldg(reinterpret_cast<const double2*>(p));
  double2 v;
  if (POL == 2)
    asm("ld.global.nc.L2::256B.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  else
    asm("ld.global.cs.L2::256B.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// 8 row tiles (M <= 64) x NY column tiles (8 NY vectors)
template <int NY>
struct AccT {
  double c[8][NY][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int x = 0; x < 8; ++x)
#pragma unroll
      for (int y = 0; y < NY; ++y) c[x][y][0] = c[x][y][1] = 0.0;
  }
};
using Acc = AccT<2>;  // 16 vectors

// acc (M x 16) += op(A) (M x K) * B (K x 16), B vector-minor (B[p * 16 + v]).
// op(A)(i, p) = TA ? A[p + i * lda] : A[i + p * lda]; A streamed (evict-first).
// Natural tile layout (row tile x = rows 8x .. 8x+7).  Used by k_bsr_mv.
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

// out (M x 8 NY of a vector-minor panel) = acc (+ out when add); natural tile layout.
template <int NY>
__device__ __forceinline__ void store_panel(const AccT<NY>& acc, double* __restrict__ out, int M, bool add) {
  const int lane = lane_id();
  const int fr = lane >> 2, fc = 2 * (lane & 3);
#pragma unroll
  for (int x = 0; x < 8; ++x) {
    const int i = 8 * x + fr;
    if (i >= M) continue;
#pragma unroll
    for (int y = 0; y < NY; ++y) {
      double2* o = reinterpret_cast<double2*>(out + i * NV + 8 * y + fc);
      double2 v = make_double2(acc.c[x][y][0], acc.c[x][y][1]);
      if (add) {
        const double2 old = __ldcg(o);
        v.x += old.x;
        v.y += old.y;
      }
      *o = v;
    }
  }
}

// ---- transposed products with paired k-steps ------------------------------
// acc (M x 16) += A^T (M x K) * B (K x 16) with A column-major (K x M, lda
// even, rows K..lda-1 may be padding), i.e. acc(i, :) += sum_p A[p + i lda] B(p, :).
// Lane k-slot fk of pair-step j0 takes the contraction rows 2j, 2j+1
// (j = j0 + fk): A by one 16-byte load per row tile, B by the callback
// bpair(j, y) -> (B(2j, 8y + fr), B(2j + 1, 8y + fr)), which must return 0
// for rows >= K.  UNROLL pair-steps (8 contraction rows each) in flight.
template <int UNROLL, int POL, int NY = 2, class BPair>
__device__ __forceinline__ void mma_T_pairs(AccT<NY>& acc, const double* __restrict__ A, int lda, int M, int K,
                                            BPair bpair) {
  const int lane = lane_id();
  const int fr = lane >> 2, fk = lane & 3;
  const int np = (K + 1) >> 1;
#pragma unroll UNROLL
  for (int j0 = 0; j0 < np; j0 += 4) {
    const int j = j0 + fk;
    const bool ok = j < np;
    const bool hi = 2 * j + 1 < K;
    double2 b[NY];
#pragma unroll
    for (int y = 0; y < NY; ++y) b[y] = bpair(j, y, ok);
    double2 a[8];
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const int i = 8 * x + fr;
      a[x] = (ok && i < M) ? ld_stream2<POL>(A + 2 * j + int64_t(i) * lda) : make_double2(0.0, 0.0);
      if (!hi) a[x].y = 0.0;  // padding row of an odd K
    }
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      if (8 * x < M) {  // warp-uniform
#pragma unroll
        for (int y = 0; y < NY; ++y) dmma(acc.c[x][y][0], acc.c[x][y][1], a[x].x, b[y].x);
#pragma unroll
        for (int y = 0; y < NY; ++y) dmma(acc.c[x][y][0], acc.c[x][y][1], a[x].y, b[y].y);
      }
    }
  }
}

// ---- untransposed products with paired row tiles -------------------------
// acc += A (M x K, column-major, lda even >= M) * B (K x 16, vector-minor).
// Row tile 2z holds rows 16z + 2fr, tile 2z + 1 rows 16z + 2fr + 1 (lane
// row fr): one 16-byte load per tile pair and k-step.
__device__ __forceinline__ int prow(int x, int fr) { return 16 * (x >> 1) + 2 * fr + (x & 1); }

template <int UNROLL, int POL, int NY = 2>
__device__ __forceinline__ void mma_N_pairs(AccT<NY>& acc, const double* __restrict__ A, int lda, int M, int K,
                                            const double* __restrict__ B) {
  const int lane = lane_id();
  const int fr = lane >> 2, fk = lane & 3;
#pragma unroll UNROLL
  for (int p0 = 0; p0 < K; p0 += 4) {
    const int p = p0 + fk;
    const bool pk = p < K;
    double b[NY];
#pragma unroll
    for (int y = 0; y < NY; ++y) b[y] = pk ? __ldcg(B + p * NV + 8 * y + fr) : 0.0;
    double2 a[4];
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      const int r = 16 * z + 2 * fr;
      a[z] = (pk && r < M) ? ld_stream2<POL>(A + r + int64_t(p) * lda) : make_double2(0.0, 0.0);
      if (r + 1 >= M) a[z].y = 0.0;  // padding row of an odd M
    }
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      if (16 * z < M) {  // warp-uniform
#pragma unroll
        for (int y = 0; y < NY; ++y) dmma(acc.c[2 * z][y][0], acc.c[2 * z][y][1], a[z].x, b[y]);
#pragma unroll
        for (int y = 0; y < NY; ++y) dmma(acc.c[2 * z + 1][y][0], acc.c[2 * z + 1][y][1], a[z].y, b[y]);
      }
    }
  }
}

// out (M x 8 NY of a vector-minor panel) = acc (+ out when add); paired-row tile layout.
template <int NY>
__device__ __forceinline__ void store_panel_pr(const AccT<NY>& acc, double* __restrict__ out, int M, bool add) {
  const int lane = lane_id();
  const int fr = lane >> 2, fc = 2 * (lane & 3);
#pragma unroll
  for (int x = 0; x < 8; ++x) {
    const int i = prow(x, fr);
    if (i >= M) continue;
#pragma unroll
    for (int y = 0; y < NY; ++y) {
      double2* o = reinterpret_cast<double2*>(out + i * NV + 8 * y + fc);
      double2 v = make_double2(acc.c[x][y][0], acc.c[x][y][1]);
      if (add) {
        const double2 old = __ldcg(o);
        v.x += old.x;
        v.y += old.y;
      }
      *o = v;
    }
  }
}

// acc = in (M x 16, vector-minor; paired-row tile layout), zero above M: the
// accumulator starts from the values the product is added to, so their loads
// overlap the first A-operand loads instead of trailing the product.
__device__ __forceinline__ void load_panel_pr(Acc& acc, const double* __restrict__ in, int M) {
  const int lane = lane_id();
  const int fr = lane >> 2, fc = 2 * (lane & 3);
#pragma unroll
  for (int x = 0; x < 8; ++x) {
    const int i = prow(x, fr);
#pragma unroll
    for (int y = 0; y < 2; ++y) {
      const double2 v = i < M ? __ldcg(reinterpret_cast<const double2*>(in + i * NV + 8 * y + fc))
                              : make_double2(0.0, 0.0);
      acc.c[x][y][0] = v.x;
      acc.c[x][y][1] = v.y;
    }
  }
}

// ---- shared 64 x 16 panel of one leaf ------------------------------------
// Pair-interleaved and swizzled: rows 2j, 2j+1 of vector v form one 16-byte
// unit at j * 16 + (v ^ ((j & 3) << 1)).  The B fragments of mma_T_pairs read
// 8 distinct bank slots per quarter warp; the gather below writes them so too.
__device__ __forceinline__ int punit(int j, int v) { return j * NV + (v ^ ((j & 3) << 1)); }

// Leaf i: xc16[t][v] = X[perm[t] + v ldx] (fused gather, hmv.hpp:179), then
// x^q_i = V_i^T xc_i (hmv.hpp:86-97) for 16 vectors.
template <int POL, int UNR>
__global__ void __launch_bounds__(32 * kLeafWarps) k_up_leaf_mv(
    const double* __restrict__ leaf, int ldm, int m, int k, int64_t nleaves, int64_t leaf0,
    const int32_t* __restrict__ perm, const double* __restrict__ X, int64_t ldx, int nv, int write_xc,
    double* __restrict__ xc, double* __restrict__ xh) {
  __shared__ double2 panel_all[kLeafWarps][32 * NV];
  double2* panel = panel_all[threadIdx.x >> 5];
  const int lane = lane_id();
  const int64_t stride = int64_t(ldm) * k;
  for (int64_t il = warp_global(); il < nleaves; il += warp_count()) {
    const int64_t i = leaf0 + il;  // global leaf; the pool holds the owned leaves only
    const int64_t base = i * m;
    // gather: lane L owns rows 2L, 2L + 1; the vector order is rotated by L / 4
    // so the 16-byte smem stores of a quarter warp hit 8 distinct slots
    const int t0 = 2 * lane, t1 = t0 + 1;
    const int64_t o0 = t0 < m ? int64_t(__ldg(perm + base + t0)) : -1;
    const int64_t o1 = t1 < m ? int64_t(__ldg(perm + base + t1)) : -1;
    // all 32 loads in flight before the first store
    double2 g[NV];
#pragma unroll
    for (int s = 0; s < NV; ++s) {
      const int v = (s + (lane >> 2)) & (NV - 1);
      const bool vok = v < nv;
      g[s].x = (vok && o0 >= 0) ? __ldg(X + o0 + v * ldx) : 0.0;
      g[s].y = (vok && o1 >= 0) ? __ldg(X + o1 + v * ldx) : 0.0;
    }
#pragma unroll
    for (int s = 0; s < NV; ++s) panel[punit(lane, (s + (lane >> 2)) & (NV - 1))] = g[s];
    __syncwarp();
    // xc16 rows of this leaf, coalesced 16-byte stores (unless a full gather
    // already wrote them: partitions, whose dense blocks read remote rows)
    const double* pd = reinterpret_cast<const double*>(panel);
    double* xo = xc + base * NV;
#pragma unroll 4
    for (int s = 0; s < NV && write_xc; ++s) {
      const int e = 2 * (s * 32 + lane);  // element (t, v) = (e / 16, e % 16), v even
      const int t = e >> 4, v = e & (NV - 1);
      if (t < m) {
        const int j = t >> 1, h = t & 1;
        *reinterpret_cast<double2*>(xo + e) =
            make_double2(pd[2 * punit(j, v) + h], pd[2 * punit(j, v + 1) + h]);
      }
    }
    if (k > 0) {
      Acc acc;
      acc.zero();
      const int fr = lane >> 2;
      mma_T_pairs<UNR, POL>(acc, leaf + il * stride, ldm, k, m, [&](int j, int y, bool ok) {
        return ok ? panel[punit(j, 8 * y + fr)] : make_double2(0.0, 0.0);
      });
      store_panel(acc, xh + i * k * NV, k, false);
    }
    __syncwarp();
  }
}

// ---- fused dataflow sweeps (see dataflow.cuh) -----------------------------
struct SweepLevelMV {
  const double* T;  // transfers of the child level l (block (c - cbegin) * stride)
  int64_t stride, cbegin;
  int ldc, kc, kp, l;
  const double* in;  // up: x^ of level l (vector-minor); down: y^ of level l - 1
  double* out;       // up: x^ of level l - 1;             down: y^ of level l
  int64_t n, i0;     // items (up: parents i0.., down: children i0..)
};
struct SweepTableMV {
  SweepLevelMV L[kMaxLevels];
  int64_t start[kMaxLevels + 1];
  int nl;
  int q;  // up: the deepest child level (input); down: the top parent level (input)
};

// The fused sweeps optionally split every node into two items, one per
// 8-vector half (SPLIT = 1): the halves of the 16-vector pass are independent
// dataflows (half h of a parent needs only half h of its children), a warp
// holds half the accumulators and fragments, and twice as many warps fit an
// SM (both halves stream the node's matrix; the second read hits L2).  Flags
// are per (node, half).
template <int SPLIT>
__device__ __forceinline__ uint32_t* flag_of(uint32_t* flag, int level, int64_t node, int h) {
  return flag + ((df::node_id(level, node) << SPLIT) + h);
}

// x^{l-1}_p = F_2p^T x^l_2p + F_2p+1^T x^l_2p+1 (hmv.hpp:98-110), levels q..1.
template <int POL, int UNR, int SPLIT>
__global__ void __launch_bounds__(kThreads) k_up_fused_mv(const __grid_constant__ SweepTableMV S,
                                                          uint32_t* __restrict__ flag,
                                                          const unsigned long long* __restrict__ ep,
                                                          unsigned long long* __restrict__ ticket) {
  const uint32_t epoch = 2u * uint32_t(__ldcg(ep));  // up flags of this pass
  constexpr int NY = SPLIT ? 1 : 2;
  const int fr = lane_id() >> 2;
  const int64_t total = S.start[S.nl];
  int64_t next = df::claim(ticket);
  for (;;) {
    const int64_t it = next;
    if (it >= total) break;
    if (kMvClaimAhead) next = df::claim(ticket);  // claimed ahead: its atomic overlaps this item
    int e = 0;
    while (it >= S.start[e + 1]) ++e;
    const SweepLevelMV& L = S.L[e];
    const int64_t loc = it - S.start[e];
    const int64_t p = L.i0 + (loc >> SPLIT);
    const int h = int(loc) & SPLIT, v0 = 8 * h;
    if (kUpPrefetch && L.kc > 0 && L.kp > 0 && h == 0)  // both child transfers, ahead of the flag waits
      prefetch_l2(L.T + (2 * p - L.cbegin) * L.stride, 2 * L.stride);
    if (L.l < S.q) {
      df::wait_flag(flag_of<SPLIT>(flag, L.l, 2 * p, h), epoch);
      df::wait_flag(flag_of<SPLIT>(flag, L.l, 2 * p + 1, h), epoch);
    }
    if (L.kp > 0) {
      AccT<NY> acc;
      acc.zero();
      if (L.kc > 0) {
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          const double* xin = L.in + (2 * p + c) * L.kc * NV + v0;
          const int kc = L.kc;
          mma_T_pairs<UNR, POL, NY>(acc, L.T + (2 * p + c - L.cbegin) * L.stride, L.ldc, L.kp, kc,
                                    [&](int j, int y, bool ok) {
            const int r = 2 * j;
            const double lo = (ok && r < kc) ? __ldcg(xin + r * NV + 8 * y + fr) : 0.0;
            const double hi = (ok && r + 1 < kc) ? __ldcg(xin + (r + 1) * NV + 8 * y + fr) : 0.0;
            return make_double2(lo, hi);
          });
        }
      }
      store_panel(acc, L.out + p * L.kp * NV + v0, L.kp, false);
    }
    df::set_flag(flag_of<SPLIT>(flag, L.l - 1, p, h), epoch);
    if (!kMvClaimAhead) next = df::claim(ticket);
  }
}

// y^l_c += E_c y^{l-1}_{c/2} (hmv.hpp:136-146), levels 1..q.
template <int POL, int UNR, int SPLIT>
__global__ void __launch_bounds__(kThreads) k_down_fused_mv(const __grid_constant__ SweepTableMV S,
                                                            uint32_t* __restrict__ flag,
                                                            const unsigned long long* __restrict__ ep,
                                                            unsigned long long* __restrict__ ticket) {
  const uint32_t epoch = 2u * uint32_t(__ldcg(ep)) + 1u;  // down flags of this pass
  constexpr int NY = SPLIT ? 1 : 2;
  const int64_t total = S.start[S.nl];
  int64_t next = df::claim(ticket);
  for (;;) {
    const int64_t it = next;
    if (it >= total) break;
    if (kMvClaimAhead) next = df::claim(ticket);  // claimed ahead: its atomic overlaps this item
    int e = 0;
    while (it >= S.start[e + 1]) ++e;
    const SweepLevelMV& L = S.L[e];
    const int64_t loc = it - S.start[e];
    const int64_t c = L.i0 + (loc >> SPLIT);
    const int h = int(loc) & SPLIT, v0 = 8 * h;
    if (kPrefetch && L.kc > 0 && L.kp > 0 && h == 0)  // the transfer block, ahead of the flag wait
      prefetch_l2(L.T + (c - L.cbegin) * L.stride, L.stride);
    if (L.l - 1 > S.q) df::wait_flag(flag_of<SPLIT>(flag, L.l - 1, c >> 1, h), epoch);
    if (L.kc > 0 && L.kp > 0) {
      AccT<NY> acc;
      acc.zero();
      mma_N_pairs<UNR, POL, NY>(acc, L.T + (c - L.cbegin) * L.stride, L.ldc, L.kc, L.kp,
                                L.in + (c >> 1) * L.kp * NV + v0);
      // y^l_c (coupling product) += E_c y^{l-1}: added at the end (starting
      // the accumulator from it, as k_down_leaf_mv does with yc, measured
      // 1.49 -> 1.70 ms at C4)
      store_panel_pr(acc, L.out + c * L.kc * NV + v0, L.kc, true);
    }
    df::set_flag(flag_of<SPLIT>(flag, L.l, c, h), epoch);
    if (!kMvClaimAhead) next = df::claim(ticket);
  }
}

struct LayerDescMV {
  const double* val;
  const int32_t* rp;
  const int32_t* ci;
  const double* x;  // vector-minor panel base
  double* y;
  int64_t stride;
  int br, bc, ld;
  int tma;  // rows of this layer go to k_bsr_mv_tma (full 64 x 64 blocks), else to k_bsr_mv
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
    if (D.tma) continue;  // streamed by k_bsr_mv_tma
    const int row = int(u & ((1u << kLayerShift) - 1));
    const int b0 = __ldg(D.rp + row), b1 = __ldg(D.rp + row + 1);
    Acc acc;
    acc.zero();
    for (int b = b0; b < b1; ++b) {
      const int col = __ldg(D.ci + b);
      // the whole 64-deep block unrolled: its 128 fragment loads per lane are
      // in flight together (measured at n = 2^22: 8 k-steps 19.35 ms per
      // 16 vectors, 16 k-steps 18.39 ms, 4 k-steps at 2 CTAs/SM 19.78 ms)
      mma_panel<false, 16>(acc, D.val + int64_t(b) * D.stride, D.ld, D.br, D.bc, D.x + int64_t(col) * D.bc * NV);
    }
    store_panel(acc, D.y + int64_t(row) * D.br * NV, D.br, false);
  }
}

// ---- TMA-fed coupling / dense product of the 16-vector pass ---------------
// One CTA per SM walks its rows of the LPT list (static round robin).  A
// producer warp streams every block of the row, and the x^ panel of its block
// column, through a kTStages-deep ring in shared memory with tensor-map TMA
// loads (cp.async.bulk.tensor.2d, 128-byte swizzle): a block is 4 boxes of
// 16 rows x 64 columns, the panel one box of 64 rows x 16 vectors (8 KB each;
// out-of-range rows / columns are zero-filled by the TMA unit), completion
// signalled on the stage's mbarrier by the transaction bytes.  Four consumer
// warps (one per SM sub-partition) each own one box, i.e. the 16 rows
// [16w, 16w + 16) of the block row, as two DMMA row tiles (even / odd rows)
// times two vector tiles (even / odd vectors): one 16-byte shared load gives
// a lane its A values of both row tiles (rows 2fr, 2fr + 1 of a column) and
// another its B values of both vector tiles (vectors 2fr, 2fr + 1).  The last
// read of a stage arrives on its empty barrier.  The ring, not the registers,
// holds the bytes in flight.
//
// Fragment k-order: in k-step kk lane (fr, fk) takes column
//   p = 8 (kk / 2) + 2 fk + kk % 2,
// a bijection onto 0..63 per block with p % 8 = 2 fk + kk % 2: under the
// 128-byte swizzle (16-byte chunk ^= line % 8) the 8 lanes of a quarter warp
// read 8 distinct chunks -- every 16-byte fragment load is 4 conflict-free
// wavefronts.
constexpr int kTStages = H2B_TSTAGES;
constexpr int kTCtas = H2B_TCTAS;  // resident CTAs per SM
constexpr int kTWarps = 4;
constexpr int kTBox = 16 * 64;                      // doubles per box (8 KB)
constexpr int kTStageDoubles = 5 * kTBox;           // 4 block boxes + the x^ panel
constexpr size_t kTSmem = size_t(kTStages) * kTStageDoubles * sizeof(double) + 1024;  // + alignment

struct TmaTableMV {
  CUtensorMap S[kMaxLevels + 2];  // per layer: 3D {ld, bc, nb} blocks, box {16, 64, 1}, 128-byte swizzle
  CUtensorMap X[2];               // [0] x^ pool, [1] xc (dense layer): {16, rows}, box {16, 64}
  int64_t xrow0[kMaxLevels + 2];  // per layer: first row of its x panels in X
  int dense;                      // the dense layer's index
};

__global__ void __launch_bounds__(32 * (kTWarps + 1), kTCtas) k_bsr_mv_tma(const __grid_constant__ LayerTableMV T,
                                                                     const __grid_constant__ TmaTableMV M,
                                                                     const uint32_t* __restrict__ work,
                                                                     int64_t nwork) {
  extern __shared__ double ring_raw[];
  double* ring = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(ring_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kTStages], empty[kTStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < kTStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int stage = 0;
  uint32_t phase = 0;
  if (warp == kTWarps) {  // producer: one elected lane
    if (lane == 0) {
      const uint64_t pol_s = l2_policy_evict_first(), pol_x = l2_policy_evict_last();
      for (int64_t it = blockIdx.x; it < nwork; it += gridDim.x) {
        const uint32_t u = __ldg(work + it);
        const int li = int(u >> kLayerShift);
        const LayerDescMV& D = T.L[li];
        if (!D.tma) continue;  // small blocks: k_bsr_mv
        const int row = int(u & ((1u << kLayerShift) - 1));
        const int b0 = __ldg(D.rp + row), b1 = __ldg(D.rp + row + 1);
        const CUtensorMap* xm = &M.X[li == M.dense ? 1 : 0];
        for (int b = b0; b < b1; ++b) {
          const int col = __ldg(D.ci + b);
          mbar_wait(&empty[stage], phase ^ 1u);
          if (D.br == 0 || D.bc == 0) {  // rank-0 blocks: nothing to load, the rows are zero
            mbar_arrive(&full[stage]);
            if (++stage == kTStages) {
              stage = 0;
              phase ^= 1u;
            }
            continue;
          }
          mbar_expect_tx(&full[stage], 5u * kTBox * sizeof(double));
          double* dst = ring + stage * kTStageDoubles;
#pragma unroll
          for (int h = 0; h < 4; ++h) tma_3d(dst + h * kTBox, &M.S[li], 16 * h, b, &full[stage], pol_s);
          tma_2d(dst + 4 * kTBox, xm, 0, int(M.xrow0[li] + int64_t(col) * D.bc), &full[stage], pol_x);
          if (++stage == kTStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    return;
  }
  const int fr = lane >> 2, fk = lane & 3;
  const int r0 = 16 * warp + 2 * fr;  // this lane's A rows: r0 (even tile), r0 + 1 (odd tile)
  for (int64_t it = blockIdx.x; it < nwork; it += gridDim.x) {
    const uint32_t u = __ldg(work + it);
    const LayerDescMV& D = T.L[u >> kLayerShift];
    if (!D.tma) continue;
    const int row = int(u & ((1u << kLayerShift) - 1));
    const int b0 = __ldg(D.rp + row), b1 = __ldg(D.rp + row + 1);
    const int br = D.br, bc = D.bc;
    const bool live = 16 * warp < br;  // warp-uniform
    double c[2][2][2] = {};  // [row tile][vector tile][pair]
    for (int b = b0; b < b1; ++b) {
      mbar_wait(&full[stage], phase);
      if (live) {
        const double* S = ring + stage * kTStageDoubles + warp * kTBox;
        const double* X = ring + stage * kTStageDoubles + 4 * kTBox;
        double2 av[16], xv[16];
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
          const int p = 8 * (kk >> 1) + 2 * fk + (kk & 1);
          const bool pk = p < bc;
          av[kk] = pk ? *reinterpret_cast<const double2*>(S + swz(p, 2 * fr)) : make_double2(0.0, 0.0);
          xv[kk] = pk ? *reinterpret_cast<const double2*>(X + swz(p, 2 * fr)) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
          dmma(c[0][0][0], c[0][0][1], av[kk].x, xv[kk].x);
          dmma(c[0][1][0], c[0][1][1], av[kk].x, xv[kk].y);
          dmma(c[1][0][0], c[1][0][1], av[kk].y, xv[kk].x);
          dmma(c[1][1][0], c[1][1][1], av[kk].y, xv[kk].y);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kTStages) {
        stage = 0;
        phase ^= 1u;
      }
    }
    // lane (fr, fk) of tile (t, y) holds rows r0 + t, vectors 2 (2 fk + j) + y:
    // four consecutive vectors 4 fk .. 4 fk + 3 of each of its two rows
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (live && r0 + t < br) {
        double* yo = D.y + (int64_t(row) * br + r0 + t) * NV + 4 * fk;
        *reinterpret_cast<double2*>(yo) = make_double2(c[t][0][0], c[t][1][0]);
        *reinterpret_cast<double2*>(yo + 2) = make_double2(c[t][0][1], c[t][1][1]);
      }
    }
  }
}

// Leaf i: Y[perm[t] + v ldy] = alpha (U_i y^q_i + yc)[t][v] + beta Y[...]
// (hmv.hpp:147-156, 184-187).  The result rows go through a shared [v][t]
// panel so the scatter is coalesced along t.
constexpr int kSLd = 68;  // shared [v][t] leading dimension (2-way store conflicts, conflict-free reads)
template <int POL, int UNR>
__global__ void __launch_bounds__(32 * kLeafWarps) k_down_leaf_mv(
    const double* __restrict__ U, int ldm, int m, int k, int64_t nleaves, int64_t leaf0,
    const double* __restrict__ yh, const double* __restrict__ yc, const int32_t* __restrict__ perm,
    double* __restrict__ Y, int64_t ldy, int nv, double alpha, double beta, double* __restrict__ yslice) {
  __shared__ __align__(16) double panel_all[kLeafWarps][NV * kSLd];
  double* panel = panel_all[threadIdx.x >> 5];
  const int lane = lane_id();
  const int fr = lane >> 2, fc = 2 * (lane & 3);
  const int64_t stride = int64_t(ldm) * k;
  for (int64_t il = warp_global(); il < nleaves; il += warp_count()) {
    const int64_t i = leaf0 + il;  // global leaf; the pool holds the owned leaves only
    Acc acc;
    load_panel_pr(acc, yc + i * m * NV, m);  // yc (dense product) + U y^ (0.88 -> 0.76 ms at C4)
    if (k > 0) mma_N_pairs<UNR, POL>(acc, U + il * stride, ldm, m, k, yh + i * k * NV);
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const int r = prow(x, fr);
      if (r >= m) continue;
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int h = 0; h < 2; ++h) panel[(8 * y + fc + h) * kSLd + r] = acc.c[x][y][h];
    }
    __syncwarp();
    const int64_t base = i * m;
    if (yslice) {  // partition: the cluster-order slice (vector-minor), alpha / beta applied by the scatter
      double* yo = yslice + il * m * NV;
      for (int e = lane; e < m * NV; e += 32) yo[e] = panel[(e & (NV - 1)) * kSLd + (e >> 4)];
      __syncwarp();
      continue;
    }
    const int t0 = 2 * lane, t1 = t0 + 1;
    const int64_t o0 = t0 < m ? int64_t(__ldg(perm + base + t0)) : -1;
    const int64_t o1 = t1 < m ? int64_t(__ldg(perm + base + t1)) : -1;
#pragma unroll 2
    for (int v = 0; v < nv; ++v) {
      const double2 u = *reinterpret_cast<const double2*>(panel + v * kSLd + t0);
      if (o0 >= 0) {
        double* d = Y + o0 + v * ldy;
        const double val = u.x;
        *d = alpha * val + (beta == 0.0 ? 0.0 : beta * *d);
      }
      if (o1 >= 0) {
        double* d = Y + o1 + v * ldy;
        const double val = u.y;
        *d = alpha * val + (beta == 0.0 ? 0.0 : beta * *d);
      }
    }
    __syncwarp();
  }
}

// xc16[t][v] = X[perm[t] + v ldx] for every t (partitions: dense blocks read
// the rows of remote leaves).  Thread per 16-byte output.
__global__ void k_gather_mv(const int32_t* __restrict__ perm, const double* __restrict__ X, int64_t ldx, int nv,
                            int64_t n, double* __restrict__ xc) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n * (NV / 2);
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = e >> 3;
    const int v = 2 * int(e & 7);
    const int64_t o = __ldg(perm + t);
    const double a = v < nv ? __ldg(X + o + v * ldx) : 0.0;
    const double b = v + 1 < nv ? __ldg(X + o + (v + 1) * ldx) : 0.0;
    reinterpret_cast<double2*>(xc)[e] = make_double2(a, b);
  }
}

// Y[perm[t] + v ldy] = alpha yc[t][v] + beta Y[...] for every t (the
// replicated-output scatter of a gathered cluster-order panel).
__global__ void k_scatter_mv(const int32_t* __restrict__ perm, const double* __restrict__ yc, int64_t n, int nv,
                             double* __restrict__ Y, int64_t ldy, double alpha, double beta) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n * NV;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = e >> 4;
    const int v = int(e & (NV - 1));
    if (v >= nv) continue;
    double* d = Y + __ldg(perm + t) + v * ldy;
    *d = alpha * yc[e] + (beta == 0.0 ? 0.0 : beta * *d);
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

unsigned leaf_grid(int64_t items) {
  return unsigned(
      std::max<int64_t>(1, std::min<int64_t>((items + kLeafWarps - 1) / kLeafWarps, int64_t(sms()) * 16)));
}

unsigned persistent_grid_mv(const void* kernel) {
  int per_sm = 0;
  H2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0));
  return unsigned(std::max(1, per_sm) * sms());
}

}  // namespace

namespace {

// Fused sweeps with one item per (node, 8-vector half) (kSplit = 1): 80
// registers and twice the warps per SM, but measured slower at C4
// (k_up_fused_mv 1.46 -> 1.56 ms, k_down_fused_mv 1.49 -> 1.94 ms: every
// fragment load now feeds half the DMMAs).  Kept switchable.
constexpr int kSplit = 0;
#ifndef H2B_TMA_BSR
#define H2B_TMA_BSR 1
#endif
constexpr bool kTmaBsr = H2B_TMA_BSR;
#ifndef H2B_UNR_DOWN
#define H2B_UNR_DOWN 2
#endif
constexpr int kUnrDown = H2B_UNR_DOWN;
#ifndef H2B_UNR_UP
#define H2B_UNR_UP 4  // C4: 1.25 ms at 1, 1.45 at 2, 1.22 at 4
#endif
constexpr int kUnrUp = H2B_UNR_UP;  // pair-steps in flight of the fused upsweep  // pair-steps in flight of the fused downsweep (see kUnr)

unsigned flat_grid_mv(int64_t items) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, int64_t(sms()) * 16)));
}

void ensure_mv_work(Matrix& A, Work& w) {
  const Matrix& C = A.col_basis();
  const int q = A.q;
  const int64_t nvec_pool = std::max<int64_t>({1, A.vec_off[q + 1], C.vec_off[q + 1]}) * NV;
  if (w.xc16.n < size_t(A.n) * NV) {
    w.xc16.alloc(size_t(A.n) * NV);
    w.yc16.alloc(size_t(A.n) * NV);
  }
  if (w.xh16.n < size_t(nvec_pool)) {
    w.xh16.alloc(nvec_pool);
    w.yh16.alloc(nvec_pool);
  }
}

// Upsweep of the 16-vector pass over this handle's nodes: gather + leaves,
// then levels q .. part_s + 1 (whole matrix: q .. 1) in one dataflow launch.
template <int POL, int UNR>
void mv_up_local(Matrix& A, Work& w, const double* X, int64_t ldx, int nv, cudaStream_t s) {
  const int q = A.q;
  const Matrix& C = A.col_basis();  // upsweep on the column basis (hmv.hpp:182)
  double* xh = w.xh16.p;
  const int64_t nl = C.own_count(q);
  const bool part = A.part_s > 0;
  if (part) {  // dense blocks crossing the partition read remote rows of xc
    k_gather_mv<<<flat_grid_mv(int64_t(A.n) * (NV / 2)), 256, 0, s>>>(A.perm.p, X, ldx, nv, A.n, w.xc16.p);
    H2B_CUDA(cudaGetLastError());
  }
  k_up_leaf_mv<POL, UNR><<<leaf_grid(nl), 32 * kLeafWarps, 0, s>>>(C.leaf.p, C.ldm, C.m, C.rank[q], nl,
                                                                   C.own_begin(q), A.perm.p, X, ldx, nv,
                                                                   part ? 0 : 1, w.xc16.p, xh + C.vec_off[q] * NV);
  H2B_CUDA(cudaGetLastError());
  if (q > A.part_s) {
    SweepTableMV T{};
    T.q = q;
    int64_t tot = 0;
    for (int l = q; l > A.part_s; --l) {
      SweepLevelMV& L = T.L[T.nl];
      L.T = C.transfer.p + C.tr_off[l];
      L.stride = C.tr_stride(l);
      L.cbegin = C.tr_begin(l);
      L.ldc = C.ld(l);
      L.kc = C.rank[l];
      L.kp = C.rank[l - 1];
      L.l = l;
      L.in = xh + C.vec_off[l] * NV;
      L.out = xh + C.vec_off[l - 1] * NV;
      L.i0 = C.own_begin(l - 1);
      L.n = C.own_count(l - 1);
      T.start[T.nl++] = tot;
      tot += L.n << kSplit;
    }
    T.start[T.nl] = tot;
    H2B_CUDA(cudaMemsetAsync(w.ticket.p, 0, sizeof(unsigned long long), s));
    k_up_fused_mv<POL, kUnrUp, kSplit><<<persistent_grid_mv((const void*)k_up_fused_mv<POL, kUnrUp, kSplit>), kThreads, 0, s>>>(
        T, w.flag.p, w.ticket.p + 2, w.ticket.p);
    H2B_CUDA(cudaGetLastError());
  }
}

// Replicated top of a partition: levels part_s .. 1, every node (level
// part_s's x^ gathered from all partitions).
template <int POL, int UNR>
void mv_up_top(Matrix& A, Work& w, cudaStream_t s) {
  if (A.part_s < 1) return;
  double* xh = w.xh16.p;
  SweepTableMV T{};
  T.q = A.part_s;
  int64_t tot = 0;
  for (int l = A.part_s; l >= 1; --l) {
    SweepLevelMV& L = T.L[T.nl];
    L.T = A.transfer.p + A.tr_off[l];
    L.stride = A.tr_stride(l);
    L.cbegin = A.tr_begin(l);
    L.ldc = A.ld(l);
    L.kc = A.rank[l];
    L.kp = A.rank[l - 1];
    L.l = l;
    L.in = xh + A.vec_off[l] * NV;
    L.out = xh + A.vec_off[l - 1] * NV;
    L.i0 = 0;
    L.n = A.nodes(l - 1);
    T.start[T.nl++] = tot;
    tot += L.n << kSplit;
  }
  T.start[T.nl] = tot;
  H2B_CUDA(cudaMemsetAsync(w.ticket.p, 0, sizeof(unsigned long long), s));
  k_up_fused_mv<POL, kUnrUp, kSplit><<<persistent_grid_mv((const void*)k_up_fused_mv<POL, kUnrUp, kSplit>), kThreads, 0, s>>>(
      T, w.flag.p, w.ticket.p + 2, w.ticket.p);
  H2B_CUDA(cudaGetLastError());
}

// Coupling + dense rows of this handle, downsweep (replicated top + own
// subtree), leaf expansion: Y (original order, alpha / beta) or, when yslice,
// the cluster-order vector-minor slice of the owned leaves.
template <int POL, int UNR>
void mv_finish(Matrix& A, Work& w, double* Y, int64_t ldy, int nv, double alpha, double beta, double* yslice,
               cudaStream_t s) {
  const int q = A.q;
  const Matrix& C = A.col_basis();
  double* xh = w.xh16.p;
  double* yh = w.yh16.p;
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
    // The LPT-ordered work list (make_work_list).  Layer / row order keeps
    // neighbouring rows' x panels in L2 (DRAM read 75.4 -> 72.6 GB at C4) but
    // loses the balance: 12.18 -> 12.71 ms; claimed dynamically (atomic row
    // ticket, claim-ahead) in that order: 72.8 GB but 15.6 ms.  16-byte paired-row loads
    // (mma_N_pairs) instead of the 8-byte fragments: 17.3 ms (fewer loads in
    // flight at 255 registers); non-coherent / L2::256B loads: 12.6 ms,
    // 79.4 GB read.  The evict-first 8-byte form stays.
    // every layer through the TMA ring (3D block views: a compressed level's
    // smaller blocks cost only their bytes).  Measured on C3 compressed at
    // 1e-6 (ranks 34-60, odd ld): 9.0-9.2 ms per pass against 12.9 ms with the
    // register-fed k_bsr_mv, 12.8 ms with only the full 64 x 64 levels on the
    // ring; uncompressed C3 10.4 vs 11.6 ms.  k_bsr_mv remains the H2B_TMA_BSR=0
    // build's kernel.
    bool any_tma = false, any_reg = false;
    for (int l = 0; l <= q + 1; ++l) {
      const Layer& L = l <= q ? A.cpl[l] : A.dense;
      T.L[l].tma = kTmaBsr;
      any_tma = any_tma || (T.L[l].tma && L.nb > 0);
    }
    if (!any_tma)
      for (int l = 0; l <= q + 1; ++l) T.L[l].tma = 0;
    for (int l = 0; l <= q + 1; ++l) any_reg = any_reg || (!T.L[l].tma && (l <= q ? A.cpl[l] : A.dense).rows > 0);
    if (any_tma) {
      TmaTableMV M{};
      const int64_t xrows = std::max<int64_t>(1, std::max(A.vec_off[q + 1], C.vec_off[q + 1]));
      encode_box16x64(&M.X[0], xh, NV, uint64_t(xrows), NV);
      encode_box16x64(&M.X[1], w.xc16.p, NV, uint64_t(std::max(1, A.n)), NV);
      M.dense = q + 1;
      for (int l = 0; l <= q + 1; ++l) {
        const Layer& L = l <= q ? A.cpl[l] : A.dense;
        M.xrow0[l] = l <= q ? C.vec_off[l] : 0;
        if (T.L[l].tma && L.nb > 0)
          encode_blocks3d(&M.S[l], L.val, uint64_t(std::max(2, L.ld)), uint64_t(L.bc), uint64_t(L.nb), 16, 64, true);
      }
      H2B_CUDA(cudaFuncSetAttribute(k_bsr_mv_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTSmem)));
      k_bsr_mv_tma<<<unsigned(std::min<int64_t>(A.nwork, int64_t(kTCtas) * sms())), 32 * (kTWarps + 1), kTSmem, s>>>(T, M, A.work.p,
                                                                                                   A.nwork);
      H2B_CUDA(cudaGetLastError());
    }
    if (any_reg) k_bsr_mv<<<wgrid(A.nwork), kThreads, 0, s>>>(T, A.work.p, A.nwork);
    H2B_CUDA(cudaGetLastError());
  }
  if (q >= 1) {  // levels 1..q in one dataflow launch (the root's y^ is final)
    SweepTableMV S{};
    S.q = 0;
    int64_t tot = 0;
    for (int l = 1; l <= q; ++l) {
      SweepLevelMV& L = S.L[S.nl];
      L.T = A.transfer.p + A.tr_off[l];
      L.stride = A.tr_stride(l);
      L.cbegin = A.tr_begin(l);
      L.ldc = A.ld(l);
      L.kc = A.rank[l];
      L.kp = A.rank[l - 1];
      L.l = l;
      L.in = yh + A.vec_off[l - 1] * NV;
      L.out = yh + A.vec_off[l] * NV;
      L.i0 = A.own_begin(l);
      L.n = A.own_count(l);
      S.start[S.nl++] = tot;
      tot += L.n << kSplit;
    }
    S.start[S.nl] = tot;
    H2B_CUDA(cudaMemsetAsync(w.ticket.p + 1, 0, sizeof(unsigned long long), s));
    k_down_fused_mv<POL, kUnrDown, kSplit><<<persistent_grid_mv((const void*)k_down_fused_mv<POL, kUnrDown, kSplit>), kThreads, 0, s>>>(
        S, w.flag.p, w.ticket.p + 2, w.ticket.p + 1);
    H2B_CUDA(cudaGetLastError());
  }
  const int64_t nl = A.own_count(q);
  k_down_leaf_mv<POL, UNR><<<leaf_grid(nl), 32 * kLeafWarps, 0, s>>>(
      A.leaf.p, A.ldm, A.m, A.rank[q], nl, A.own_begin(q), yh + A.vec_off[q] * NV, w.yc16.p, A.perm.p, Y, ldy, nv,
      alpha, beta, yslice);
  H2B_CUDA(cudaGetLastError());
}

// Load policy and unroll measured at C4 (n = 2^22, k = 64, 16 vectors; ncu
// launch lists, tools/mv16_launches.sh): the evict-first 16-byte loads of the
// transposed products fetched 1.5-1.8x their bytes from DRAM (the other half
// of each 128-byte line was evicted before its second 64-byte piece was
// used): k_up_fused_mv 2.13 ms / 8.73 GB read, k_up_leaf_mv 0.87 ms / 4.00 GB.
// Non-coherent loads with the 256-byte L2 prefetch hint read exactly the
// algorithmic bytes: 1.45 ms / 5.36 GB and 0.68 ms / 2.70 GB.  Two pair-steps
// in flight beat four (registers / occupancy) except for the leaf (0.67 vs
// 0.68 ms, noise).  The untransposed products are insensitive to the policy.
// One pair-step in flight (kUnr = 1) beat two for the leaves and the upsweep
// once the loads were non-coherent (k_up_fused_mv 1.46 -> 1.24 ms, the leaf
// kernels 0.69 / 0.76 -> 0.64 / 0.68 ms); the downsweep keeps two (1.41 vs
// 1.49 ms with its L2 prefetch).  With the sweeps claiming items after the
// current one, the fused upsweep runs best at four (1.22 vs 1.25 ms at one,
// 1.45 at two; kUnrUp).
constexpr int kPol = 2, kUnr = 1;

}  // namespace

// Y (n x nv, ld ldy) <- alpha A X + beta Y for nv <= 16 vectors, device pointers.
void hmv_multi_device(Matrix& A, Work& w, const double* X, int64_t ldx, double* Y, int64_t ldy, int nv,
                      double alpha, double beta, cudaStream_t s) {
  require(nv >= 1 && nv <= NV, "hmv_multi: 1..16 vectors per pass");
  require(A.part_s == 0, "hmv_multi_device: partition handle");
  ensure_mv_work(A, w);
  sweep_begin(w, A, s);
  mv_up_local<kPol, kUnr>(A, w, X, ldx, nv, s);
  mv_finish<kPol, kUnr>(A, w, Y, ldy, nv, alpha, beta, nullptr, s);
}

// Partitioned 16-vector pass, phase 1: owned leaves and levels > part_s.
// Level l >= part_s of the vector-minor x^ panel pool (xh16) then holds this
// partition's nodes; the caller all-gathers them (part_exchange).
void part_mv_upsweep(Matrix& A, Work& w, const double* X, int64_t ldx, int nv, cudaStream_t s) {
  require(nv >= 1 && nv <= NV, "hmv_multi: 1..16 vectors per pass");
  ensure_mv_work(A, w);
  sweep_begin(w, A, s);
  mv_up_local<kPol, kUnr>(A, w, X, ldx, nv, s);
}

// Phase 2: replicated top, owned rows, downsweep, leaf expansion into Y
// (yslice == nullptr: owned rows of Y in original order) or the cluster-order
// vector-minor slice.
void part_mv_finish(Matrix& A, Work& w, double* Y, int64_t ldy, int nv, double alpha, double beta, double* yslice,
                    cudaStream_t s) {
  mv_up_top<kPol, kUnr>(A, w, s);
  mv_finish<kPol, kUnr>(A, w, Y, ldy, nv, alpha, beta, yslice, s);
}

void launch_scatter_mv(const int32_t* perm, const double* yc, int64_t n, int nv, double* Y, int64_t ldy,
                       double alpha, double beta, cudaStream_t s) {
  if (n == 0) return;
  k_scatter_mv<<<flat_grid_mv(n * NV), 256, 0, s>>>(perm, yc, n, nv, Y, ldy, alpha, beta);
  H2B_CUDA(cudaGetLastError());
}

}  // namespace h2b
