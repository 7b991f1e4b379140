// Verifies cta::gemm_tc (DMMA m8n8k4) against cta::gemm (DFMA) for all
// transpose combinations and ragged shapes; times both on 64^3 blocks.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_1902_01829_b200/csrc/cta_linalg.cuh"
using namespace h2b;

template <bool TA, bool TB, bool TC>
__global__ void k_gemm(double* C, const double* A, const double* B, int m, int n, int k, int reps) {
  extern __shared__ double sm[];
  const int la = cta::sld(TA ? k : m), lb = cta::sld(TB ? n : k), lc = cta::sld(m);
  double* As = sm; double* Bs = As + la * (TA ? m : k); double* Cs = Bs + lb * (TB ? k : n);
  const int ar = TA ? k : m, ac = TA ? m : k, br = TB ? n : k, bc = TB ? k : n;
  cta::copy_block(As, la, A + blockIdx.x * ar * ac, ar, ar, ac);
  cta::copy_block(Bs, lb, B + blockIdx.x * br * bc, br, br, bc);
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
    if (TC) cta::gemm_tc<TA, TB>(Cs, lc, As, la, Bs, lb, m, n, k);
    else cta::gemm<TA, TB>(Cs, lc, As, la, Bs, lb, m, n, k);
    __syncthreads();
  }
  cta::copy_block(C + blockIdx.x * m * n, m, Cs, lc, m, n);
}

template <bool TA, bool TB>
double check(int m, int n, int k) {
  const int nb = 4;
  std::vector<double> A(nb * m * k), B(nb * k * n), C1(nb * m * n), C2(nb * m * n);
  for (auto& v : A) v = drand48() - 0.5;
  for (auto& v : B) v = drand48() - 0.5;
  double *dA, *dB, *dC;
  cudaMalloc(&dA, A.size() * 8); cudaMalloc(&dB, B.size() * 8); cudaMalloc(&dC, C1.size() * 8);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
  const size_t sm = 8 * (size_t(cta::sld(TA ? k : m)) * (TA ? m : k) + size_t(cta::sld(TB ? n : k)) * (TB ? k : n) +
                         size_t(cta::sld(m)) * n);
  cudaFuncSetAttribute(k_gemm<TA, TB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  cudaFuncSetAttribute(k_gemm<TA, TB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  k_gemm<TA, TB, true><<<nb, 256, sm>>>(dC, dA, dB, m, n, k, 1);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("launch failed %s\n", cudaGetErrorString(cudaGetLastError())); exit(2); }
  cudaMemcpy(C1.data(), dC, C1.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemset(dC, 0, C1.size() * 8);
  k_gemm<TA, TB, false><<<nb, 256, sm>>>(dC, dA, dB, m, n, k, 1);
  cudaMemcpy(C2.data(), dC, C2.size() * 8, cudaMemcpyDeviceToHost);
  double err = 0, nrm = 0;
  for (size_t i = 0; i < C1.size(); ++i) { err = fmax(err, fabs(C1[i] - C2[i])); nrm = fmax(nrm, fabs(C2[i])); }
  cudaFree(dA); cudaFree(dB); cudaFree(dC);
  return err / nrm;
}

template <bool TC>
double timeit() {
  const int nb = 148 * 8, m = 64, reps = 50;
  double *dA, *dB, *dC;
  cudaMalloc(&dA, nb * m * m * 8); cudaMalloc(&dB, nb * m * m * 8); cudaMalloc(&dC, nb * m * m * 8);
  cudaMemset(dA, 0, nb * m * m * 8); cudaMemset(dB, 0, nb * m * m * 8);
  const size_t sm = 8 * (cta::sld(64) * 64 * 3);
  cudaFuncSetAttribute(k_gemm<false, false, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  k_gemm<false, false, TC><<<nb, 256, sm>>>(dC, dA, dB, m, m, m, 1);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_gemm<false, false, TC><<<nb, 256, sm>>>(dC, dA, dB, m, m, m, reps);
  cudaEventRecord(b); cudaEventSynchronize(b);
  if (cudaGetLastError() != cudaSuccess) { printf("timing launch failed\n"); exit(2); }
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaFree(dA); cudaFree(dB); cudaFree(dC);
  return 2.0 * m * m * m * double(nb) * reps / ms / 1e9;
}

int main() {
  int shapes[][3] = {{64, 64, 64}, {128, 64, 64}, {37, 21, 13}, {8, 8, 4}, {1, 1, 1}, {64, 60, 96}, {29, 35, 64}};
  double worst = 0;
  for (auto& s : shapes) {
    worst = fmax(worst, check<false, false>(s[0], s[1], s[2]));
    worst = fmax(worst, check<true, false>(s[0], s[1], s[2]));
    worst = fmax(worst, check<false, true>(s[0], s[1], s[2]));
    worst = fmax(worst, check<true, true>(s[0], s[1], s[2]));
  }
  printf("gemm_tc vs gemm max rel diff: %.3e %s\n", worst, worst < 1e-13 ? "OK" : "MISMATCH");
  printf("64^3 smem gemm: DFMA %.2f TFLOP/s, DMMA %.2f TFLOP/s\n", timeit<false>() / 1e3, timeit<true>() / 1e3);
  return worst < 1e-13 ? 0 : 1;
}
