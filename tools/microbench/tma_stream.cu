// Read-bandwidth microbenchmark: a 64 GB f64 stream read (a) by 16-byte
// evict-first loads (the k_bsr pattern) and (b) by tensor-map TMA boxes
// through an mbarrier ring (the k_bsr_mv_tma pattern), trivial consumers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void k_ldg(const double* __restrict__ a, int64_t n, double* out) {
  double s = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x * 2;
  for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 2; i < n; i += stride) {
    double2 v = __ldcs(reinterpret_cast<const double2*>(a + i));
    s += v.x + v.y;
  }
  if (s == 1.2345) *out = s;
}

template <int STAGES, int CONS>
__global__ void __launch_bounds__(32 * (CONS + 1)) k_tma(const __grid_constant__ CUtensorMap map, int64_t nboxes, double* out) {
  extern __shared__ double raw[];
  double* ring = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(CONS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int stage = 0; uint32_t phase = 0;
  if (warp == CONS) {
    if (lane == 0) {
      for (int64_t b = blockIdx.x; b < nboxes; b += gridDim.x) {
        asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(su32(&empty[stage])), "r"(phase ^ 1u) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[stage])), "r"(4 * 8192) : "memory");
        for (int h = 0; h < 4; ++h)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                       ::"r"(su32(ring + stage * 4096 + h * 1024)), "l"(&map), "r"(16 * h), "r"(int(b * 64)), "r"(su32(&full[stage])) : "memory");
        if (++stage == STAGES) { stage = 0; phase ^= 1u; }
      }
    }
    return;
  }
  double s = 0;
  for (int64_t b = blockIdx.x; b < nboxes; b += gridDim.x) {
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(su32(&full[stage])), "r"(phase) : "memory");
    const double* t = ring + stage * 4096 + warp * 1024;
    for (int i = lane; i < 1024; i += 32) s += t[i];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[stage])) : "memory");
    if (++stage == STAGES) { stage = 0; phase ^= 1u; }
  }
  if (s == 1.2345) *out = s;
}

int main() {
  const int64_t n = (int64_t(64) << 30) / 8;  // 64 GB
  double* a; double* o;
  CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&o, 8));
  CK(cudaMemset(a, 0, n * 8));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k_ldg<<<sms * 8, 256>>>(a, n, o);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("ldcs16 %d: %.3f ms %.1f GB/s\n", rep, ms, n * 8 / (ms * 1e6));
  }
  void* fp; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  CUtensorMap map;
  cuuint64_t dims[2] = {64, cuuint64_t(n / 64)}, strides[1] = {64 * 8};
  cuuint32_t box[2] = {16, 64}, es[2] = {1, 1};
  CUresult r = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); return 1; }
  const int64_t nboxes = n / (64 * 64);  // 32 KB blocks
  auto run = [&](auto kern, int stages, int ctas, const char* name) {
    const size_t sm = size_t(stages) * 32768 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      kern<<<sms * ctas, 160, sm>>>(map, nboxes, o);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("%s %d: %.3f ms %.1f GB/s (%s)\n", name, rep, ms, n * 8 / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
    }
  };
  run(k_tma<2, 4>, 2, 2, "tma 2stg x2cta");
  run(k_tma<3, 4>, 3, 2, "tma 3stg x2cta");
  run(k_tma<6, 4>, 6, 1, "tma 6stg x1cta");
  return 0;
}
