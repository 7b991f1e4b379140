// Internal types of libh2b.so: the HBM-resident H^2 matrix and its workspace.
//
// Device layout.  Everything the reference keeps in
// std::vector pools (BasisTree::leaf_pool / transfer[l], BSRLayer::values,
// LevelVectors::pool[l]; include/h2kit/h2_matrix.hpp:17-80, hmv.hpp:13-22)
// lives in a few large cudaMalloc'd pools:
//   * every matrix block is column-major with an EVEN leading dimension
//     ld = pad2(rows) (a zero row is appended when rows is odd), so every
//     column starts 16-byte aligned and the kernels can use 128-bit loads;
//   * block strides are ld * cols doubles, 64-bit offsets throughout;
//   * node vectors x^ / y^ are unpadded, level-concatenated (vec_off[l]).
// Marshaling (hmv.hpp:33-74, compression.hpp:47-64,185-209) is replaced by
// closed-form complete-binary-tree index arithmetic inside the kernels:
// children of level-local node i are 2i, 2i+1; the parent is i >> 1.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "h2b.h"
#include "nvtx3/nvToolsExt.h"

namespace h2b {

struct Error : std::runtime_error {
  h2b_status code;
  Error(h2b_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// The reference's require() (include/h2kit/defs.hpp:20-22).
inline void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(H2B_INVALID_ARGUMENT, msg);
}

#define H2B_CUDA(expr)                                                              \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      throw ::h2b::Error(e_ == cudaErrorMemoryAllocation ? H2B_OUT_OF_MEMORY        \
                                                         : H2B_CUDA_ERROR,          \
                         std::string(#expr) + ": " + cudaGetErrorString(e_));       \
  } while (0)

inline int pad2(int r) { return r + (r & 1); }

// NVTX range for the profilers (nsys / ncu --nvtx); no cost without a tool.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Largest block dimension the fast warp kernels cover (rows owned by a lane
// pair: 2 * 32 lanes) and the compression kernels accept; mat-vec blocks up
// to kMaxDimHmv take the k_hmv_big.cu kernels (two row pairs per lane).
constexpr int kMaxDim = 64;
constexpr int kMaxDimHmv = 128;
constexpr int kMaxLevels = 31;

// Device buffer (cudaMalloc / cudaFree).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t cnt) {
    release();
    if (cnt == 0) return;
    H2B_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), cnt * sizeof(T)));
    n = cnt;
  }
  void zero(cudaStream_t s) {
    if (n) H2B_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// One uniform-block BSR layer (a coupling level or the dense layer),
// bsr.hpp:13-31.  row_ptr/col_idx are level-local like the reference.
struct Layer {
  int br = 0, bc = 0, ld = 0;     // block dims, padded leading dim
  int64_t rows = 0, nb = 0;
  int64_t row0 = 0, row1 = -1;      // block rows this handle computes (-1: all)
  int max_row = 0;
  std::vector<int32_t> h_rp, h_ci;  // host copy of the structure
  int32_t* rp = nullptr;            // device (views into Matrix pools)
  int32_t* ci = nullptr;
  double* val = nullptr;
  int64_t block_stride() const { return int64_t(ld) * bc; }
};

// Work item of the fused BSR kernel: (layer << 26) | block_row.
constexpr int kLayerShift = 26;

// Per-caller mat-vec workspace: the HmvContext analogue (hmv.hpp:159-172,
// "a context is not thread-safe, concurrent hmv calls need one context
// each").  Every user of a Work holds its mutex while enqueueing and orders
// its stream after the previous user's work on the device (event `done`), so
// two streams sharing one Work serialise on the device instead of racing;
// two Works on one matrix run concurrently.
struct Work {
  int device = 0;
  const void* owner = nullptr;      // matrix the buffers were sized for
  uint64_t layout = 0;              // ... and its layout_version
  DevBuf<double> xc, yc;            // x, y in cluster order (n)
  DevBuf<double> xhat, yhat;        // x^ (column-basis ranks), y^ (row-basis ranks), level-concatenated
  DevBuf<double> xs, ys;            // device staging of host x / y
  DevBuf<double> xc16, yc16, xh16, yh16;  // 16-vector panels (k_hmv_mv.cu), lazily allocated
  DevBuf<double> xg, yg;            // partitioned mat-vec exchange buffers (x^ slices, y slices), lazily allocated
  // Fused dataflow sweeps (launch_up_fused / launch_down_fused): per-node
  // completion flags (epoch-valued, never reset) and the work tickets.
  DevBuf<uint32_t> flag;
  DevBuf<unsigned long long> ticket;  // [0] up ticket, [1] down ticket, [2] epoch (advanced on the device)
  std::mutex mu;
  cudaEvent_t done = nullptr;
  Work() = default;
  Work(const Work&) = delete;
  Work& operator=(const Work&) = delete;
  ~Work() {
    if (done) cudaEventDestroy(done);
  }
};

struct Matrix {
  int device = 0;
  cudaStream_t stream = nullptr;
  int n = 0, m = 0, q = 0, ldm = 0;
  std::vector<int> rank;            // per level (row basis == column basis)

  DevBuf<int32_t> perm;
  DevBuf<double> leaf;              // 2^q blocks, ldm x rank[q]
  DevBuf<double> transfer;          // level-concatenated, block ld = pad2(rank[l])
  std::vector<int64_t> tr_off;      // [l] offset into transfer (l >= 1)

  std::vector<Layer> cpl;           // q + 1 coupling levels
  Layer dense;
  DevBuf<double> cpl_val, dense_val;
  DevBuf<int32_t> cpl_rp, cpl_ci, dense_rp, dense_ci;

  std::vector<int64_t> vec_off;     // node-vector level offsets, size q + 2
  DevBuf<uint32_t> work;            // BSR work list (dense + coupling rows)
  int64_t nwork = 0;

  // The handle's own mat-vec workspace (the default HmvContext; h2b_context
  // handles are further ones).  layout_version changes whenever the ranks
  // (hence the x^ / y^ sizes) change, e.g. after compress().
  std::unique_ptr<Work> work0;
  uint64_t layout_version = 1;
  // Points (original order) + kernel of a device-built matrix, for
  // h2b_validate_sampled (validate.cu).
  DevBuf<double> pts_orig;
  int pts_dim = 0;
  double ell = 0.0;
  h2b_build_info info{};            // BuildInfo of the container format (h2_matrix.hpp:53-60)
  // coupling mirror map (block (col,row) of block (row,col)) for the symmetric
  // projection in compress(); structure only, built on first use
  bool mirror_ready = false;
  std::vector<char> mirror_sym;     // per level: pattern symmetric
  std::vector<char> value_sym;      // per level: blocks symmetric too (set at creation)
  std::vector<int64_t> mirror_off;
  DevBuf<int32_t> mirror;
  double* h_stage = nullptr;        // pinned host staging for host-pointer calls
  size_t h_stage_n = 0;

  // Per-phase CUDA-event timing (h2b_set_phase_timing): four events per
  // hmv call, recorded on the launching stream without host syncs; read and
  // reset by h2b_last_hmv_timing.
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;

  // Subtree partition: 2^part_s partitions, this handle owns
  // part_g.  Levels >= part_s are split by top subtree; levels < part_s (and
  // the transfers up to level part_s) are replicated.  part_s = 0: whole matrix.
  int part_s = 0, part_g = 0;
  uint64_t global_footprint = 0;    // memory_footprint of the whole matrix

  // Non-symmetric matrices (U != V, h2_matrix.hpp:69,75-78): the column basis
  // V / F lives in colb, a basis-only Matrix (n, m, q, ldm, rank, perm, leaf,
  // transfer, tr_off, and its own x^ workspace: xc, xhat, vec_off); coupling
  // blocks of level l are rank[l] x colb->rank[l].  Symmetric: colb is null.
  bool symmetric = true;
  std::unique_ptr<Matrix> colb;
  const Matrix& col_basis() const { return symmetric ? *this : *colb; }
  Matrix& col_basis() { return symmetric ? *this : *colb; }

  ~Matrix();
  int64_t nodes(int l) const { return int64_t(1) << l; }
  int64_t own_begin(int l) const { return l < part_s ? 0 : int64_t(part_g) << (l - part_s); }
  int64_t own_end(int l) const { return l < part_s ? nodes(l) : int64_t(part_g + 1) << (l - part_s); }
  int64_t own_count(int l) const { return own_end(l) - own_begin(l); }
  int64_t tr_begin(int l) const { return l <= part_s ? 0 : own_begin(l); }
  int64_t tr_count(int l) const { return l <= part_s ? nodes(l) : own_count(l); }
  int ld(int l) const { return pad2(rank[l]); }
  int64_t leaf_stride() const { return int64_t(ldm) * rank[q]; }
  int64_t tr_stride(int l) const { return int64_t(ld(l)) * rank[l - 1]; }
  uint64_t footprint() const;       // reference byte convention
  uint64_t device_bytes() const;
  double hmv_flops() const;         // reference analytic model
};

// ---- launchers (k_hmv.cu) ----
// Node vectors (xhat / yhat) are whole level-concatenated buffers laid out by
// the basis' vec_off.  x in original order (perm gather fused) unless
// cluster_order; xc receives x in cluster order.
void launch_up_leaf(const Matrix& B, const double* x, double* xc, double* xhat, cudaStream_t s,
                    bool cluster_order = false);
// parents at level l-1 in [p0, p1) (children in the transfer pool)
void launch_up_level(const Matrix& B, int l, double* xhat, cudaStream_t s, int64_t p0 = 0, int64_t p1 = -1);
// x^ level offsets from xb (the column basis' vec_off), y^ from A.
void launch_bsr(const Matrix& A, const uint32_t* work, int64_t nwork, const double* xdense,
                double* ydense, const double* xh, double* yh, cudaStream_t s, const Matrix* xb = nullptr);
// One generic BSR layer, y <- alpha L x + beta y (block_sparse_mv, bsr.hpp:50-82),
// bitwise the reference's arithmetic (phase API).
void launch_bsr_exact(const Layer& L, const double* x, double* y, double alpha, double beta, cudaStream_t s);
// children at level l in [c0, c1)
void launch_down_level(const Matrix& A, int l, double* yhat, cudaStream_t s, int64_t c0 = 0, int64_t c1 = -1);
// yc += U y^q; to_user: y[perm[t]] = alpha v + beta y[perm[t]] (original
// order); else y[t] = v with t relative to the first owned leaf (cluster-order slice).
void launch_down_leaf(const Matrix& A, const double* yhat, const double* yc, double* y, double alpha,
                      double beta, bool to_user, cudaStream_t s);
// Whole-matrix upsweep above the leaves (levels l_hi..l_lo of basis B) and
// downsweep (levels 1..q of A) as ONE persistent launch each: warps claim
// nodes deepest-first (up) / top-down (down) and wait for their children /
// parent through per-node flags (held by the Work w).
// sweep_begin: a new epoch for the flags (once per mat-vec, stream-ordered
// on s).  Up: child levels l_hi..l_lo (l_hi's x^ is input); down: levels
// 1..q (the root's y^ is input); own: this handle's node ranges (partition).
void sweep_begin(Work& w, const Matrix& A, cudaStream_t s);
void launch_up_fused(Work& w, const Matrix& B, double* xhat, cudaStream_t s, int l_hi, int l_lo, bool own);
void launch_down_fused(Work& w, const Matrix& A, double* yhat, cudaStream_t s, bool own);
void launch_gather(const int32_t* perm, const double* x, double* xc, int64_t n, cudaStream_t s);
// y[perm[t]] = alpha ys[t] + beta y[perm[t]] (t < n): the owner-row scatter of
// a cluster-order y (partitioned mat-vec).
void launch_scatter(const int32_t* perm, const double* ys, double* y, int64_t n, double alpha, double beta,
                    cudaStream_t s);

// ---- blocks of 65..128 rows / columns (k_hmv_big.cu) ----
bool big_basis(const Matrix& B);   // leaf size or some rank > kMaxDim
bool big_matrix(const Matrix& A);  // ... of the row or the column basis
void launch_up_leaf_big(const Matrix& B, const double* x, double* xc, double* xhat, cudaStream_t s,
                        bool cluster_order);
void launch_up_level_big(const Matrix& B, int l, double* xhat, cudaStream_t s, int64_t p0, int64_t p1);
void launch_down_level_big(const Matrix& A, int l, double* yhat, cudaStream_t s, int64_t c0, int64_t c1);
void launch_down_leaf_big(const Matrix& A, const double* yhat, const double* yc, double* y, double alpha,
                          double beta, bool to_user, cudaStream_t s);
void launch_bsr_big(const Matrix& A, const uint32_t* work, int64_t nwork, const double* xdense, double* ydense,
                    const double* xh, double* yh, cudaStream_t s, const Matrix* xb);

// ---- workspaces (capi.cu) ----
// (Re)size w for A's current layout; the default workspace of A.
void ensure_work(Matrix& A, Work& w);
Work& default_work(Matrix& A);
// Holds w for one call on stream s (mutex + device-order after the previous user).
struct WorkUse {
  Work& w;
  cudaStream_t s;
  WorkUse(Work& work, cudaStream_t st);
  ~WorkUse();
  WorkUse(const WorkUse&) = delete;
  WorkUse& operator=(const WorkUse&) = delete;
};

// 16-vector FP64-MMA mat-vec, device pointers (k_hmv_mv.cu).
void hmv_multi_device(Matrix& A, Work& w, const double* X, int64_t ldx, double* Y, int64_t ldy, int nv,
                      double alpha, double beta, cudaStream_t s);
// Partitioned 16-vector pass (k_hmv_mv.cu): owned leaves + levels > part_s
// into w.xh16; then (after the x^ exchange) the replicated top, owned rows,
// downsweep and leaf expansion into Y (yslice null: owned rows of Y, original
// order, alpha / beta applied) or the cluster-order vector-minor slice.
void part_mv_upsweep(Matrix& A, Work& w, const double* X, int64_t ldx, int nv, cudaStream_t s);
void part_mv_finish(Matrix& A, Work& w, double* Y, int64_t ldy, int nv, double alpha, double beta, double* yslice,
                    cudaStream_t s);
// Y[perm[t] + v ldy] = alpha yc[t * 16 + v] + beta Y[...], t < n, v < nv.
void launch_scatter_mv(const int32_t* perm, const double* yc, int64_t n, int nv, double* Y, int64_t ldy,
                       double alpha, double beta, cudaStream_t s);

// ---- x^ exchange of the partitioned mat-vec (part_hmv.cu) ----
// Doubles per partition slice (x^ entries of width `width`: 1 or 16).
int64_t part_exchange_count(const Matrix& A, int width);
// slice part_g of buf <- this partition's x^ runs at levels >= part_s
void launch_pack_xhat(const Matrix& A, int width, const double* pool, double* buf, cudaStream_t s);
// x^ runs of every other partition <- their slices of buf
void launch_unpack_xhat(const Matrix& A, int width, const double* buf, double* pool, cudaStream_t s);

// Build the fused BSR work list for the given layers (rows sorted by
// decreasing block count so the round-robin warp assignment is balanced).
std::vector<uint32_t> make_work_list(const std::vector<const Layer*>& layers);

// ---- padded <-> packed block copies (k_hmv.cu) ----
// dst (ld_dst x cols, stride sd) <- src (ld_src x cols, stride ss), rows valid.
void launch_repack(const double* src, int64_t ss, int ld_src, double* dst, int64_t sd, int ld_dst,
                   int rows, int cols, int64_t count, cudaStream_t s);

}  // namespace h2b

// The opaque handles of include/h2b.h: the device matrix itself, and a Work.
struct h2b_matrix : h2b::Matrix {};
struct h2b_context : h2b::Work {};
