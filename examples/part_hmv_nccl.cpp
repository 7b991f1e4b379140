// C++ host driver of the subtree-partitioned H^2 mat-vec over NCCL
// (north_star: "the host stays in C++ and calls CUDA through a
// thin C-ABI layer").  No Python, no torch: one host thread per GPU, one
// ncclComm_t per thread, libh2b.so does every kernel (upsweep, x^ pack /
// unpack, coupling + dense rows, downsweep, owner-row scatter), and the only
// communication is the stream-ordered ncclAllGather this file hands to
// h2b_part_hmv / h2b_part_hmv_multi through an h2b_dcomm.
//
//   part_hmv_nccl [--dim 2] [--n 4194304] [--order 8] [--gpus N] [--steps 20] [--warmup 3]
//                 [--nvec 1] [--owned] [--emulate P] [--check]
//
// --gpus N     N GPUs, NCCL all-gathers (default: every visible GPU, a power of two)
// --emulate P  P partitions on GPU 0, all-gathers host-staged between threads
//              (the CPU-side stand-in of NCCL used by the one-GPU tests; same
//              library calls, same callback contract)
// --check      compare with the whole-matrix h2b_hmv on GPU 0 (max rel error)
// Prints one JSON line: ms per mat-vec (max over ranks, CUDA events), GB/s in
// the reference byte convention (memory_footprint of the whole matrix).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <barrier>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "h2b.h"

#define CK(x)                                                                       \
  do {                                                                              \
    h2b_status s_ = (x);                                                            \
    if (s_ != H2B_OK) {                                                             \
      std::fprintf(stderr, "%s failed: %d %s\n", #x, int(s_), h2b_last_error());    \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)
#define CU(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      std::fprintf(stderr, "%s failed: %s\n", #x, cudaGetErrorString(e_));          \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)
#define NC(x)                                                                       \
  do {                                                                              \
    ncclResult_t r_ = (x);                                                          \
    if (r_ != ncclSuccess) {                                                        \
      std::fprintf(stderr, "%s failed: %s\n", #x, ncclGetErrorString(r_));          \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)

namespace {

struct Args {
  int dim = 2, n = 1 << 22, order = 8, gpus = 0, steps = 20, warmup = 3, nvec = 1, emulate = 0;
  bool owned = false, check = false;
};

// ---- NCCL communicator: in-place all-gather on the library's stream ----
struct NcclRank {
  ncclComm_t comm;
  int rank;
};
int nccl_allgather(void* ctx, double* buf, int64_t count, void* stream) {
  auto* r = static_cast<NcclRank*>(ctx);
  return ncclAllGather(buf + r->rank * count, buf, size_t(count), ncclDouble, r->comm,
                       static_cast<cudaStream_t>(stream)) == ncclSuccess
             ? 0
             : 1;
}

// ---- host-staged stand-in for P partitions on one GPU ----
struct Emulated {
  int P;
  std::barrier<>* bar;
  std::vector<double*>* bufs;  // each rank's exchange buffer
};
struct EmuRank {
  Emulated* e;
  int rank;
};
int emu_allgather(void* ctx, double* buf, int64_t count, void* stream) {
  auto* r = static_cast<EmuRank*>(ctx);
  Emulated& e = *r->e;
  if (cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) != cudaSuccess) return 1;
  (*e.bufs)[r->rank] = buf;
  e.bar->arrive_and_wait();
  for (int g = 0; g < e.P; ++g)
    if (g != r->rank &&
        cudaMemcpy(buf + g * count, (*e.bufs)[g] + g * count, count * sizeof(double), cudaMemcpyDeviceToDevice) !=
            cudaSuccess)
      return 1;
  e.bar->arrive_and_wait();  // nobody overwrites its slice before every peer copied it
  return 0;
}

std::vector<double> random_x(int64_t n, int nvec) {
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  std::vector<double> x(size_t(n) * nvec);
  for (double& v : x) v = u(g);
  return x;
}

}  // namespace

int main(int argc, char** argv) {
  Args a;
  for (int i = 1; i < argc; ++i) {
    std::string k = argv[i];
    auto next = [&] { return i + 1 < argc ? std::atoi(argv[++i]) : 0; };
    if (k == "--dim") a.dim = next();
    else if (k == "--n") a.n = next();
    else if (k == "--order") a.order = next();
    else if (k == "--gpus") a.gpus = next();
    else if (k == "--steps") a.steps = next();
    else if (k == "--warmup") a.warmup = next();
    else if (k == "--nvec") a.nvec = next();
    else if (k == "--emulate") a.emulate = next();
    else if (k == "--owned") a.owned = true;
    else if (k == "--check") a.check = true;
    else {
      std::fprintf(stderr, "unknown argument %s\n", k.c_str());
      return 2;
    }
  }
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  const bool emu = a.emulate > 0;
  const int P = emu ? a.emulate : (a.gpus > 0 ? a.gpus : ndev);
  if (P < 1 || (P & (P - 1)) || (!emu && P > ndev)) {
    std::fprintf(stderr, "need a power-of-two rank count <= visible GPUs (got %d of %d)\n", P, ndev);
    return 2;
  }
  const h2b_build_config cfg{a.dim, a.n, 64, a.order, 2.0, a.dim == 2 ? 0.1 : 0.2, 0.25, 1};
  const std::vector<double> xh = random_x(a.n, a.nvec);

  std::vector<ncclComm_t> comms(P);
  if (!emu) {
    std::vector<int> devs(P);
    for (int g = 0; g < P; ++g) devs[g] = g;
    NC(ncclCommInitAll(comms.data(), P, devs.data()));
  }
  std::barrier<> bar(P);
  std::vector<double*> bufs(P, nullptr);
  Emulated E{P, &bar, &bufs};

  std::vector<double> ms(P, 0.0), y0(emu || P == 1 ? size_t(a.n) * a.nvec : 0);
  std::vector<uint64_t> fp_global(P, 0);
  std::vector<std::thread> th;
  for (int g = 0; g < P; ++g) {
    th.emplace_back([&, g] {
      const int dev = emu ? 0 : g;
      CU(cudaSetDevice(dev));
      h2b_matrix* A = nullptr;
      CK(h2b_matrix_build_part(&cfg, dev, P, g, &A));
      h2b_matrix_info inf{};
      CK(h2b_matrix_info_get(A, &inf));
      fp_global[g] = inf.global_footprint_bytes;
      cudaStream_t st;
      CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      const size_t nx = size_t(a.n) * a.nvec;
      double *x = nullptr, *y = nullptr;
      CU(cudaMalloc(&x, nx * sizeof(double)));
      CU(cudaMalloc(&y, nx * sizeof(double)));
      CU(cudaMemcpy(x, xh.data(), nx * sizeof(double), cudaMemcpyHostToDevice));
      CU(cudaMemset(y, 0, nx * sizeof(double)));
      NcclRank nr{emu ? nullptr : comms[g], g};
      EmuRank er{&E, g};
      const h2b_dcomm dc = emu ? h2b_dcomm{&er, emu_allgather} : h2b_dcomm{&nr, nccl_allgather};
      const int ym = a.owned ? H2B_Y_OWNED : H2B_Y_REPLICATED;
      auto step = [&] {
        if (a.nvec == 1)
          CK(h2b_part_hmv(A, x, y, 1.0, 0.0, ym, &dc, st));
        else
          CK(h2b_part_hmv_multi(A, a.nvec, x, a.n, y, a.n, 1.0, 0.0, ym, &dc, st));
      };
      for (int i = 0; i < a.warmup; ++i) step();
      CU(cudaStreamSynchronize(st));
      bar.arrive_and_wait();
      cudaEvent_t e0, e1;
      CU(cudaEventCreate(&e0));
      CU(cudaEventCreate(&e1));
      CU(cudaEventRecord(e0, st));
      for (int i = 0; i < a.steps; ++i) step();
      CU(cudaEventRecord(e1, st));
      CU(cudaEventSynchronize(e1));
      float t = 0;
      CU(cudaEventElapsedTime(&t, e0, e1));
      ms[g] = t / a.steps;
      bar.arrive_and_wait();
      if (g == 0 && !y0.empty()) CU(cudaMemcpy(y0.data(), y, nx * sizeof(double), cudaMemcpyDeviceToHost));
      CU(cudaFree(x));
      CU(cudaFree(y));
      CU(cudaStreamDestroy(st));
      CK(h2b_matrix_destroy(A));
    });
  }
  for (auto& t : th) t.join();
  if (!emu)
    for (auto& c : comms) ncclCommDestroy(c);

  double err = -1.0;
  if (a.check && !y0.empty() && !a.owned) {  // whole matrix on GPU 0
    CU(cudaSetDevice(0));
    h2b_matrix* W = nullptr;
    CK(h2b_matrix_build(&cfg, 0, &W));
    std::vector<double> yr(size_t(a.n) * a.nvec);
    if (a.nvec == 1)
      CK(h2b_hmv(W, xh.data(), yr.data(), 1.0, 0.0, H2B_PTR_HOST, nullptr));
    else
      CK(h2b_hmv_multi(W, a.nvec, xh.data(), a.n, yr.data(), a.n, 1.0, 0.0, H2B_PTR_HOST, nullptr));
    double num = 0, den = 0;
    for (size_t i = 0; i < yr.size(); ++i) {
      num += (y0[i] - yr[i]) * (y0[i] - yr[i]);
      den += yr[i] * yr[i];
    }
    err = std::sqrt(num / den);
    CK(h2b_matrix_destroy(W));
  }
  const double t = *std::max_element(ms.begin(), ms.end());
  std::printf(
      "{\"driver\": \"examples/part_hmv_nccl.cpp\", \"comm\": \"%s\", \"ranks\": %d, \"dim\": %d, \"n\": %d, "
      "\"grid_order\": %d, \"nvec\": %d, \"y_mode\": \"%s\", \"steps\": %d, \"ms_per_step\": %.4f, "
      "\"GBs\": %.1f, \"footprint_bytes\": %llu, \"check_rel_err\": %.3e}\n",
      emu ? "emulated (host-staged, one GPU)" : "nccl", P, a.dim, a.n, a.order, a.nvec,
      a.owned ? "owned" : "replicated", a.steps, t, double(fp_global[0]) * a.nvec / (t * 1e6),
      (unsigned long long)fp_global[0], err);
  return (a.check && !(err >= 0.0 && err <= 1e-12)) ? 1 : 0;
}
