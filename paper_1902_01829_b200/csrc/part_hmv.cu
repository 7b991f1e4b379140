// Exchange buffers of the subtree-partitioned mat-vec.
//
// At every level l >= s the nodes a partition owns are one contiguous run of
// the level-concatenated x^ pool: [g 2^(l-s), (g+1) 2^(l-s)) x k_l entries
// (x width per entry: 1 for the single-vector pool, 16 for the vector-minor
// panels of the multi-vector pass).  One all-gather per mat-vec moves them
// all: pack the owned runs of every level into slice g of an exchange buffer
// (nparts equal slices), all-gather it in place, unpack the other slices.
#include "h2b_internal.hpp"

#include <algorithm>

namespace h2b {
namespace {

struct PackPlan {
  int64_t pool_off[kMaxLevels];  // level offset in the pool (elements, width included)
  int64_t run[kMaxLevels];       // owned run length of one partition (elements)
  int64_t start[kMaxLevels + 1]; // prefix of run: position within a slice
  int nl, s;
};

__device__ __forceinline__ int find_level(const PackPlan& P, int64_t e) {
  int l = 0;
  while (e >= P.start[l + 1]) ++l;
  return l;
}

// slice g of buf <- owned runs of partition g (pack: g = part only).
__global__ void k_pack(const __grid_constant__ PackPlan P, const double* __restrict__ pool, double* __restrict__ buf,
                       int part) {
  const int64_t total = P.start[P.nl];
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int l = find_level(P, e);
    buf[part * total + e] = pool[P.pool_off[l] + part * P.run[l] + (e - P.start[l])];
  }
}

// runs of every partition g != part <- slice g of buf.
__global__ void k_unpack(const __grid_constant__ PackPlan P, const double* __restrict__ buf, double* __restrict__ pool,
                         int nparts, int part) {
  const int64_t total = P.start[P.nl];
  for (int64_t x = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < total * nparts;
       x += int64_t(gridDim.x) * blockDim.x) {
    const int g = int(x / total);
    if (g == part) continue;
    const int64_t e = x - g * total;
    const int l = find_level(P, e);
    pool[P.pool_off[l] + g * P.run[l] + (e - P.start[l])] = buf[x];
  }
}

PackPlan make_plan(const Matrix& A, int width) {
  PackPlan P{};
  P.s = A.part_s;
  int64_t tot = 0;
  for (int l = A.part_s; l <= A.q; ++l) {
    if (A.rank[l] == 0) continue;
    P.pool_off[P.nl] = A.vec_off[l] * width;
    P.run[P.nl] = (int64_t(1) << (l - A.part_s)) * A.rank[l] * width;
    P.start[P.nl] = tot;
    tot += P.run[P.nl];
    ++P.nl;
  }
  P.start[P.nl] = tot;
  return P;
}

unsigned grid_for(int64_t n) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)));
}

}  // namespace

// Doubles per partition slice of the x^ exchange buffer.
int64_t part_exchange_count(const Matrix& A, int width) {
  const PackPlan P = make_plan(A, width);
  return P.start[P.nl];
}

void launch_pack_xhat(const Matrix& A, int width, const double* pool, double* buf, cudaStream_t s) {
  const PackPlan P = make_plan(A, width);
  const int64_t total = P.start[P.nl];
  if (total == 0) return;
  k_pack<<<grid_for(total), 256, 0, s>>>(P, pool, buf, A.part_g);
  H2B_CUDA(cudaGetLastError());
}

void launch_unpack_xhat(const Matrix& A, int width, const double* buf, double* pool, cudaStream_t s) {
  const PackPlan P = make_plan(A, width);
  const int64_t total = P.start[P.nl];
  const int nparts = 1 << A.part_s;
  if (total == 0 || nparts == 1) return;
  k_unpack<<<grid_for(total * nparts), 256, 0, s>>>(P, buf, pool, nparts, A.part_g);
  H2B_CUDA(cudaGetLastError());
}

}  // namespace h2b
