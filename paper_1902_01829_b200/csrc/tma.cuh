// Tensor-memory-accelerator (TMA) helpers shared by the streaming kernels
// (k_hmv.cu: k_bsr_tma, k_hmv_mv.cu: k_bsr_mv_tma): mbarrier ring
// primitives, tensor-map loads with L2 cache hints, the 128-byte swizzle
// addressing of a box of 16-double lines, and the host-side tensor-map
// encoding (cuTensorMapEncodeTiled through the runtime's driver entry point,
// no link-time libcuda dependency).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <string>

#include "h2b_internal.hpp"

namespace h2b {
namespace tma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// L2 policies of the TMA loads: the matrix stream evict-first (read once),
// the x^ panels evict-last (re-read by every block of their block column).
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                       uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// Element (line, e) of a 128-byte-swizzled box of 16-double lines.
__device__ __forceinline__ int swz(int line, int e) { return line * 16 + ((((e >> 1) ^ line) & 7) << 1) + (e & 1); }

// Block b of a 3D view {ld, cols, blocks} (see encode_blocks3d): rows from r0.
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, int r0, int b, uint64_t* bar,
                                       uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "0, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(r0), "r"(b), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_1d(void* dst, const CUtensorMap* map, int c0, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2}], "
      "[%3], %4;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    H2B_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    require(p != nullptr && q == cudaDriverEntryPointSuccess, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2D f64 tensor {inner, outer} (outer stride `ld` doubles), boxes of 16 x 64
// elements, 128-byte swizzle, out-of-range elements zero-filled.
inline void encode_box16x64(CUtensorMap* m, const double* base, uint64_t inner, uint64_t outer, uint64_t ld) {
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * sizeof(double)};
  const cuuint32_t box[2] = {16, 64};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = tensor_map_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                                          strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(H2B_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
}

// 2D f64 tensor {inner, outer} (outer stride `ld` doubles), boxes of 64 x 64
// elements without swizzle (one 32 KB block per load, column-major in shared
// memory with a 64-double column stride), out-of-range elements zero-filled.
inline void encode_box64x64(CUtensorMap* m, const double* base, uint64_t inner, uint64_t outer, uint64_t ld) {
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * sizeof(double)};
  const cuuint32_t box[2] = {64, 64};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = tensor_map_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                                          strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(H2B_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
}

// 3D f64 view {ld, cols, blocks} of a pool of column-major blocks (ld x cols
// each, consecutive), boxes {box_rows, box_cols, 1} without swizzle: one load
// puts a block into a box_rows-strided shared tile, rows >= ld and columns >=
// cols zero-filled -- a block narrower than the box costs only its own bytes
// (a 2D view would stream the next block's columns).  Needs 16-byte aligned
// base and ld even.
inline void encode_blocks3d(CUtensorMap* m, const double* base, uint64_t ld, uint64_t cols, uint64_t blocks,
                            uint32_t box_rows, uint32_t box_cols, bool swizzle128 = false) {
  const cuuint64_t dims[3] = {ld, cols, blocks};
  const cuuint64_t strides[2] = {ld * sizeof(double), ld * cols * sizeof(double)};
  const cuuint32_t box[3] = {box_rows, box_cols, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = tensor_map_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims,
                                          strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(H2B_CUDA_ERROR, "cuTensorMapEncodeTiled (3D) failed: " + std::to_string(int(r)));
}

// 1D f64 tensor of n elements, boxes of `box` elements (no swizzle), zero fill
// beyond n.
inline void encode_1d(CUtensorMap* m, const double* base, uint64_t n, uint32_t box) {
  const cuuint64_t dims[1] = {n};
  const cuuint64_t strides[1] = {n * sizeof(double)};  // unused for rank 1
  const cuuint32_t boxd[1] = {box};
  const cuuint32_t es[1] = {1};
  const CUresult r = tensor_map_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, const_cast<double*>(base), dims, strides,
                                          boxd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error(H2B_CUDA_ERROR, "cuTensorMapEncodeTiled (1D) failed: " + std::to_string(int(r)));
}

}  // namespace tma
}  // namespace h2b
