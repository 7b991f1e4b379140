// Dependent-chain latencies (cycles) of FP64 ops on one warp: DFMA, DADD,
// DMUL, sqrt, division, rcp, shfl, LDS.  B200 microbenchmark for the
// compression kernels' critical-path model.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[64];
  sm[threadIdx.x] = a + threadIdx.x;
  __syncwarp();
  double x = a + threadIdx.x * 1e-9;
  long long t0, t1;
#define MEAS(idx, BODY)                     \
  t0 = clock64();                           \
  for (int i = 0; i < n; ++i) { BODY; }     \
  t1 = clock64();                           \
  if (threadIdx.x == 0) cyc[idx] = t1 - t0;
  MEAS(0, x = fma(x, b, a));
  MEAS(1, x = x + b);
  MEAS(2, x = x * b);
  MEAS(3, x = sqrt(x));
  MEAS(4, x = a / x);
  MEAS(5, x = __drcp_rn(x));
  MEAS(6, x = __shfl_xor_sync(0xffffffffu, x, 1));
  MEAS(7, x = sm[(__double_as_longlong(x) & 1) + threadIdx.x]);
  MEAS(8, x = sqrt(fma(x, x, b)); x = a / (x * b));
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 256); cudaMalloc(&c, 16 * 8);
  const int n = 1000;
  for (int r = 0; r < 2; ++r) k<<<1, 32>>>(o, c, 1.0000001, 0.9999999, n);
  long long h[16];
  cudaMemcpy(h, c, 9 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"DFMA", "DADD", "DMUL", "sqrt", "div", "drcp_rn", "shfl.f64", "LDS.64", "sqrt+mul+div"};
  for (int i = 0; i < 9; ++i) printf("%-14s %.1f cyc\n", nm[i], double(h[i]) / n);
}
