// Warp-level GEMV building blocks of the single-vector sweeps (k_hmv.cu,
// k_hmv_big.cu): a warp owns one small column-major block; lane L owns the
// row pair (2L, 2L+1), so a 64-row column is one coalesced 512-byte load.
#pragma once

#include <cstdint>

namespace h2b {
namespace wg {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double2 ld_stream(const double* p) {
  return __ldcs(reinterpret_cast<const double2*>(p));
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int64_t warp_global() {
  return (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
}
__device__ __forceinline__ int64_t warp_count() {
  return (int64_t(gridDim.x) * blockDim.x) >> 5;
}

// Transposed product for the column group g in {0,1}:
//   returns out[2*lane + g] = sum_r A[r, 2*lane+g] * v[r]  (+ B^T w when TWO)
// A, B: column-major, leading dim ld (even), `cols` columns; the lane's row
// pair (2*lane, 2*lane+1) is valid when row_ok.
template <bool TWO>
__device__ __forceinline__ double gemvT_group(const double* __restrict__ A,
                                              const double* __restrict__ B, int ld, int cols,
                                              int g, double v0, double v1, double w0, double w1,
                                              bool row_ok, bool row_ok_b = true) {
  const int lane = lane_id();
  const int r = 2 * lane;
  // Streaming reduce-scatter: each chunk of 8 columns is reduced over lane
  // bits 0..2 right away (7 shuffles), leaving one value per chunk; the 4
  // chunk values are then reduced over lane bits 3..4 (3 shuffles).  Lane L
  // ends with column index L of the group; 31 shuffles per 32 columns, and
  // only one chunk of loads is live at a time.
  double hv[4] = {0.0, 0.0, 0.0, 0.0};
  const int64_t step = 2 * int64_t(ld);
  const double* pa = A + int64_t(g) * ld + r;
  const double* pb = TWO ? B + int64_t(g) * ld + r : nullptr;
#pragma unroll 1
  for (int h = 0; h < 4; ++h) {
    double p[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int c = 2 * (8 * h + t) + g;
      const bool ok = c < cols && row_ok;
      const double2 a = ok ? ld_stream(pa) : make_double2(0.0, 0.0);
      pa += step;
      double acc = a.x * v0 + a.y * v1;
      if (TWO) {
        const double2 b = (ok && row_ok_b) ? ld_stream(pb) : make_double2(0.0, 0.0);
        pb += step;
        acc += b.x * w0 + b.y * w1;
      }
      p[t] = acc;
    }
#pragma unroll
    for (int s = 1, n = 8; s <= 4; s <<= 1, n >>= 1) {
      const bool up = (lane & s) != 0;
#pragma unroll
      for (int i = 0; i < n / 2; ++i) {
        const double keep = up ? p[2 * i + 1] : p[2 * i];
        const double send = up ? p[2 * i] : p[2 * i + 1];
        p[i] = keep + __shfl_xor_sync(kFull, send, s);
      }
    }
    hv[0] = h == 0 ? p[0] : hv[0];
    hv[1] = h == 1 ? p[0] : hv[1];
    hv[2] = h == 2 ? p[0] : hv[2];
    hv[3] = h == 3 ? p[0] : hv[3];
    if (2 * (8 * h + 8) + g >= cols) break;  // remaining chunks are all padding
  }
#pragma unroll
  for (int s = 8, n = 4; s <= 16; s <<= 1, n >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const double keep = up ? hv[2 * i + 1] : hv[2 * i];
      const double send = up ? hv[2 * i] : hv[2 * i + 1];
      hv[i] = keep + __shfl_xor_sync(kFull, send, s);
    }
  }
  return hv[0];
}

// Non-transposed product: returns (acc0, acc1) for rows (2*lane, 2*lane+1)
// of A (ld x cols) times v, where v is held in pair layout (lane L has
// v[2L], v[2L+1]) and broadcast with shuffles.
__device__ __forceinline__ void gemvN_pair(const double* __restrict__ A, int ld, int cols,
                                           double a0, double a1, bool row_ok, double& acc0,
                                           double& acc1) {
  const int r = 2 * lane_id();
  acc0 = 0.0;
  acc1 = 0.0;
  for (int c0 = 0; c0 < cols; c0 += 8) {
    double2 col[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = c0 + u;
      col[u] = (c < cols && row_ok) ? ld_stream(A + int64_t(c) * ld + r) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = c0 + u;  // warp-uniform
      if (c < cols) {
        const double s = __shfl_sync(kFull, (c & 1) ? a1 : a0, c >> 1);
        acc0 += col[u].x * s;
        acc1 += col[u].y * s;
      }
    }
  }
}

}  // namespace wg
}  // namespace h2b
