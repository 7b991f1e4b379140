// C-ABI implementation (include/h2b.h): host orchestration of the device
// H^2 matrix.  The reference's call sequence (hmv.hpp:175-188) is kept phase
// for phase; marshaling, pool management and OpenMP fork/joins are replaced
// by the kernels in k_hmv.cu acting on HBM-resident pools.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "h2b_internal.hpp"

namespace h2b {

namespace {
thread_local std::string g_err;

template <class F>
h2b_status guarded(F&& f) {
  try {
    f();
    return H2B_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return H2B_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_err = e.what();
    return H2B_INTERNAL;
  }
}

int usable_devices() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int ok = 0;
  for (int d = 0; d < n; ++d) {
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d);
    if (major >= 10) ++ok;
  }
  return ok;
}

void need_device(int device) {
  const int n = usable_devices();
  if (n == 0) throw Error(H2B_NO_DEVICE, "no sm_100 CUDA device available (libh2b has no CPU fallback)");
  require(device >= 0 && device < n, "device index out of range");
  H2B_CUDA(cudaSetDevice(device));
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    H2B_CUDA(cudaSetDevice(d));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

bool resolve_device(h2b_ptr_kind kind, const void* p) {
  if (kind == H2B_PTR_DEVICE) return true;
  if (kind == H2B_PTR_HOST) return false;
  return p && is_device_ptr(p);
}

// Upload `count` column-major blocks of rows x cols stored densely
// (stride rows*cols) into a padded device pool (ld = pad2(rows)).
void upload_blocks(const double* h, double* d, int rows, int cols, int64_t count,
                   cudaStream_t s) {
  const int ld = pad2(rows);
  const size_t packed = size_t(rows) * cols * count;
  if (packed == 0) return;
  if (ld == rows) {
    H2B_CUDA(cudaMemcpyAsync(d, h, packed * sizeof(double), cudaMemcpyHostToDevice, s));
    return;
  }
  DevBuf<double> tmp;
  tmp.alloc(packed);
  H2B_CUDA(cudaMemcpyAsync(tmp.p, h, packed * sizeof(double), cudaMemcpyHostToDevice, s));
  launch_repack(tmp.p, int64_t(rows) * cols, rows, d, int64_t(ld) * cols, ld, rows, cols, count, s);
  H2B_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

// for phases.cu
h2b_status guarded_call(const std::function<void()>& f) { return guarded(f); }
void need_device_public(int device) { need_device(device); }
bool resolve_device_public(h2b_ptr_kind kind, const void* p) { return resolve_device(kind, p); }
// host -> padded device blocks, synchronous (phases.cu)
void upload_blocks_sync(const double* h, double* d, int rows, int cols, int64_t count, cudaStream_t s) {
  upload_blocks(h, d, rows, cols, count, s);
  H2B_CUDA(cudaStreamSynchronize(s));
}

// padded device blocks -> unpadded host blocks (also used by io.cu)
void download_blocks(const double* d, double* h, int rows, int cols, int64_t count,
                     cudaStream_t s) {
  const int ld = pad2(rows);
  const size_t packed = size_t(rows) * cols * count;
  if (packed == 0) return;
  if (ld == rows) {
    H2B_CUDA(cudaMemcpyAsync(h, d, packed * sizeof(double), cudaMemcpyDeviceToHost, s));
    H2B_CUDA(cudaStreamSynchronize(s));
    return;
  }
  DevBuf<double> tmp;
  tmp.alloc(packed);
  launch_repack(d, int64_t(ld) * cols, ld, tmp.p, int64_t(rows) * cols, rows, rows, cols, count, s);
  H2B_CUDA(cudaMemcpyAsync(h, tmp.p, packed * sizeof(double), cudaMemcpyDeviceToHost, s));
  H2B_CUDA(cudaStreamSynchronize(s));
}


Matrix::~Matrix() {
  if (stream) cudaStreamSynchronize(stream);
  if (h_stage) cudaFreeHost(h_stage);
  for (auto& e : ev_pool)
    if (e) cudaEventDestroy(e);
  if (stream) cudaStreamDestroy(stream);
}

uint64_t Matrix::footprint() const {
  // memory_footprint(A) (h2_matrix.hpp:90-102): unpadded entries * 8 bytes.
  // (a partition handle counts the blocks it stores)
  uint64_t e = uint64_t(dense.nb) * dense.br * dense.bc + uint64_t(own_count(q)) * m * rank[q];
  for (int l = 0; l <= q; ++l) e += uint64_t(cpl[l].nb) * cpl[l].br * cpl[l].bc;
  for (int l = 1; l <= q; ++l) e += uint64_t(tr_count(l)) * rank[l] * rank[l - 1];
  if (!symmetric) {  // the column basis counts too (h2_matrix.hpp:97-100)
    const Matrix& C = *colb;
    e += uint64_t(own_count(q)) * m * C.rank[q];
    for (int l = 1; l <= q; ++l) e += uint64_t(tr_count(l)) * C.rank[l] * C.rank[l - 1];
  }
  return e * sizeof(double);
}

uint64_t Matrix::device_bytes() const {
  uint64_t b = perm.bytes() + leaf.bytes() + transfer.bytes() + cpl_val.bytes() + dense_val.bytes() +
               cpl_rp.bytes() + cpl_ci.bytes() + dense_rp.bytes() + dense_ci.bytes() + work.bytes() +
               (colb ? colb->device_bytes() : 0);
  if (work0)
    b += work0->xc.bytes() + work0->yc.bytes() + work0->xhat.bytes() + work0->yhat.bytes() + work0->xs.bytes() +
         work0->ys.bytes() + work0->xc16.bytes() + work0->yc16.bytes() + work0->xh16.bytes() +
         work0->yh16.bytes() + work0->flag.bytes() + work0->xg.bytes() + work0->yg.bytes();
  return b;
}

// ---------------------------------------------------------------- workspaces
void ensure_work(Matrix& A, Work& w) {
  if (w.owner == &A && w.layout == A.layout_version) return;
  const Matrix& C = A.col_basis();
  const int q = A.q;
  w.device = A.device;
  w.xc.alloc(A.n);
  w.yc.alloc(A.n);
  w.xhat.alloc(std::max<int64_t>(1, C.vec_off[q + 1]));
  w.yhat.alloc(std::max<int64_t>(1, A.vec_off[q + 1]));
  w.xs.release();
  w.ys.release();
  w.xh16.release();
  w.yh16.release();
  w.xg.release();
  w.yg.release();
  if (!w.done) H2B_CUDA(cudaEventCreateWithFlags(&w.done, cudaEventDisableTiming));
  w.owner = &A;
  w.layout = A.layout_version;
}

Work& default_work(Matrix& A) {
  if (!A.work0) A.work0.reset(new Work);
  return *A.work0;
}

WorkUse::WorkUse(Work& work, cudaStream_t st) : w(work), s(st) {
  w.mu.lock();
  if (w.done) {
    const cudaError_t e = cudaStreamWaitEvent(s, w.done, 0);
    if (e != cudaSuccess) {
      w.mu.unlock();
      H2B_CUDA(e);
    }
  }
}

WorkUse::~WorkUse() {
  if (w.done) cudaEventRecord(w.done, s);
  w.mu.unlock();
}

double Matrix::hmv_flops() const {
  // flops.hpp:29-47 over the call sequence of hmv.hpp:175-188.
  double f = 2.0 * dense.br * dense.bc * double(dense.nb);
  const Matrix& C = col_basis();
  f += 2.0 * m * (rank[q] + C.rank[q]) * double(nodes(q));  // leaf gemv down (U) + up (V)
  for (int l = 1; l <= q; ++l)
    f += 2.0 * (rank[l] * rank[l - 1] + C.rank[l] * C.rank[l - 1]) * double(nodes(l));
  for (int l = 0; l <= q; ++l)
    if (cpl[l].nb) f += 2.0 * cpl[l].br * cpl[l].bc * double(cpl[l].nb);
  return f;
}

// Allocate pools and the workspace for the structure already set in A
// (n, m, q, rank, layers' host CSR).  Values are left uninitialised.
void allocate(Matrix& A) {
  const int q = A.q;
  A.ldm = pad2(A.m);
  A.perm.alloc(A.n);
  A.leaf.alloc(size_t(A.own_count(q)) * A.leaf_stride());
  A.tr_off.assign(q + 2, 0);
  int64_t t = 0;
  for (int l = 1; l <= q; ++l) {
    A.tr_off[l] = t;
    t += A.tr_count(l) * A.tr_stride(l);
  }
  A.tr_off[q + 1] = t;
  A.transfer.alloc(t);
  int64_t nv = 0, nrp = 0, nci = 0;
  for (int l = 0; l <= q; ++l) {
    Layer& L = A.cpl[l];
    L.ld = pad2(L.br);
    nv += L.nb * L.block_stride();
    nrp += L.rows + 1;
    nci += L.nb;
  }
  A.cpl_val.alloc(nv);
  A.cpl_rp.alloc(nrp);
  A.cpl_ci.alloc(nci);
  nv = nrp = nci = 0;
  for (int l = 0; l <= q; ++l) {
    Layer& L = A.cpl[l];
    L.val = A.cpl_val.p + nv;
    L.rp = A.cpl_rp.p + nrp;
    L.ci = A.cpl_ci.p + nci;
    nv += L.nb * L.block_stride();
    nrp += L.rows + 1;
    nci += L.nb;
  }
  Layer& D = A.dense;
  D.ld = pad2(D.br);
  A.dense_val.alloc(size_t(D.nb) * D.block_stride());
  A.dense_rp.alloc(D.rows + 1);
  A.dense_ci.alloc(D.nb);
  D.val = A.dense_val.p;
  D.rp = A.dense_rp.p;
  D.ci = A.dense_ci.p;

  A.vec_off.assign(q + 2, 0);
  for (int l = 0; l <= q; ++l) A.vec_off[l + 1] = A.vec_off[l] + A.nodes(l) * A.rank[l];
  ++A.layout_version;
}

// Column basis of a non-symmetric matrix: leaf / transfer pools for the
// column ranks plus the x^ side of the workspace (the upsweep runs on it).
void allocate_col(Matrix& A, const int32_t* cranks) {
  const int q = A.q;
  A.symmetric = false;
  A.colb.reset(new Matrix);
  Matrix& C = *A.colb;
  C.device = A.device;
  C.stream = nullptr;  // borrowed: A's stream is passed explicitly
  C.n = A.n;
  C.m = A.m;
  C.q = q;
  C.ldm = A.ldm;
  C.rank.assign(cranks, cranks + q + 1);
  C.perm.alloc(A.n);
  C.leaf.alloc(size_t(C.own_count(q)) * C.leaf_stride());
  C.tr_off.assign(q + 2, 0);
  int64_t t = 0;
  for (int l = 1; l <= q; ++l) {
    C.tr_off[l] = t;
    t += C.tr_count(l) * C.tr_stride(l);
  }
  C.tr_off[q + 1] = t;
  C.transfer.alloc(t);
  C.vec_off.assign(q + 2, 0);
  for (int l = 0; l <= q; ++l) C.vec_off[l + 1] = C.vec_off[l] + C.nodes(l) * C.rank[l];
  ++A.layout_version;
}

// Upload the CSR structure of every layer and build the fused work list.
// Mirror map of the coupling levels (used by the symmetric projection of
// compress()): mirror[b] = index of block (col, row) for block b = (row, col)
// when the level's block pattern is symmetric (always, for construct()), -1
// everywhere otherwise.  O(nb log k) per level: every row's (col, block)
// pairs sorted, merged with the transposed pattern built by a counting pass.
void build_mirror(Matrix& A) {
  const int q = A.q;
  std::vector<int32_t> all;
  A.mirror_sym.assign(q + 1, 0);
  A.mirror_off.assign(q + 2, 0);
  for (int l = 0; l <= q; ++l) {
    const Layer& L = A.cpl[l];
    std::vector<int32_t> mir(L.nb, -1);
    bool ok = A.part_s == 0 && L.nb > 0 && A.symmetric;  // a partition handle does not hold the mirror rows
    if (ok) {
      // transposed pattern: for row c, the blocks (r, c) in increasing r
      std::vector<int64_t> tp(L.rows + 1, 0);
      for (int64_t b = 0; b < L.nb; ++b) ++tp[L.h_ci[b] + 1];
      for (int64_t r = 0; r < L.rows; ++r) tp[r + 1] += tp[r];
      std::vector<std::pair<int32_t, int32_t>> tr(L.nb);  // (row, block)
      std::vector<int64_t> fill(tp.begin(), tp.end() - 1);
      for (int64_t r = 0; r < L.rows && ok; ++r)
        for (int32_t b = L.h_rp[r]; b < L.h_rp[r + 1]; ++b) {
          if (L.h_ci[b] == r) ok = false;
          tr[fill[L.h_ci[b]]++] = {int32_t(r), b};
        }
      std::vector<std::pair<int32_t, int32_t>> row;  // (col, block) of row c, sorted
      for (int64_t c = 0; c < L.rows && ok; ++c) {
        row.clear();
        for (int32_t b = L.h_rp[c]; b < L.h_rp[c + 1]; ++b) row.push_back({L.h_ci[b], b});
        std::sort(row.begin(), row.end());
        const int64_t t0 = tp[c], t1 = tp[c + 1];
        if (t1 - t0 != int64_t(row.size())) {
          ok = false;
          break;
        }
        // block (r, c) = tr[t] mirrors block (c, r) = row[k]
        for (int64_t t = t0, k = 0; t < t1; ++t, ++k) {
          if (tr[t].first != row[k].first) {
            ok = false;
            break;
          }
          mir[tr[t].second] = row[k].second;
        }
      }
    }
    if (!ok) std::fill(mir.begin(), mir.end(), -1);
    A.mirror_sym[l] = ok;
    A.mirror_off[l + 1] = A.mirror_off[l] + L.nb;
    all.insert(all.end(), mir.begin(), mir.end());
  }
  A.mirror.alloc(std::max<size_t>(1, all.size()));
  if (!all.empty())
    H2B_CUDA(cudaMemcpyAsync(A.mirror.p, all.data(), all.size() * sizeof(int32_t), cudaMemcpyHostToDevice, A.stream));
  A.mirror_ready = true;
}

// Value symmetry of the mirrored coupling blocks: S_(c,r) == S_(r,c)^T bit for
// bit.  The reference's "symmetric" means row basis == column basis; a
// construct() matrix (kernel evaluations) is symmetric in its blocks too, a
// user's h2b_matrix_create matrix need not be.  One pass over the coupling
// pool at creation; the symmetric projection of compress() is used only on
// levels that pass (and keeps them exactly symmetric).
__global__ void k_sym_check(const double* __restrict__ val, int64_t bstride, int ld, int k, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ ci, const int32_t* __restrict__ mirror, int64_t rows,
                            int* __restrict__ bad) {
  const int64_t r = blockIdx.x;
  if (r >= rows) return;
  for (int b = rp[r]; b < rp[r + 1]; ++b) {
    if (ci[b] <= r) continue;
    const double* S = val + int64_t(b) * bstride;
    const double* M = val + int64_t(mirror[b]) * bstride;
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
      const int j = e / k, i = e - j * k;
      if (S[i + j * ld] != M[j + i * ld]) *bad = 1;
    }
  }
}

void check_value_symmetry(Matrix& A) {
  cudaStream_t s = A.stream;
  A.value_sym.assign(A.q + 1, 0);
  DevBuf<int> bad;
  bad.alloc(A.q + 1);
  bad.zero(s);
  for (int l = 0; l <= A.q; ++l) {
    const Layer& L = A.cpl[l];
    if (!A.mirror_sym[l] || L.nb == 0) continue;
    k_sym_check<<<unsigned(L.rows), 128, 0, s>>>(L.val, L.block_stride(), L.ld, L.br, L.rp, L.ci,
                                                 A.mirror.p + A.mirror_off[l], L.rows, bad.p + l);
    H2B_CUDA(cudaGetLastError());
  }
  std::vector<int> h(A.q + 1);
  H2B_CUDA(cudaMemcpyAsync(h.data(), bad.p, (A.q + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
  H2B_CUDA(cudaStreamSynchronize(s));
  for (int l = 0; l <= A.q; ++l) A.value_sym[l] = A.mirror_sym[l] && !h[l];
}

// The BSR work list for the current block shapes (LPT order), reusing the
// device list when the row count is unchanged.
void rebuild_work_list(Matrix& A) {
  cudaStream_t s = A.stream;
  std::vector<const Layer*> layers;
  for (int l = 0; l <= A.q; ++l) layers.push_back(&A.cpl[l]);
  layers.push_back(&A.dense);
  const std::vector<uint32_t> w = make_work_list(layers);
  if (A.work.n != w.size()) A.work.alloc(w.size());
  A.nwork = int64_t(w.size());
  if (!w.empty())
    H2B_CUDA(cudaMemcpyAsync(A.work.p, w.data(), w.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  H2B_CUDA(cudaStreamSynchronize(s));
}

void upload_structure(Matrix& A) {
  cudaStream_t s = A.stream;
  build_mirror(A);
  for (int l = 0; l <= A.q; ++l) {
    Layer& L = A.cpl[l];
    L.max_row = 0;
    for (int64_t r = 0; r < L.rows; ++r) L.max_row = std::max(L.max_row, L.h_rp[r + 1] - L.h_rp[r]);
    H2B_CUDA(cudaMemcpyAsync(L.rp, L.h_rp.data(), (L.rows + 1) * sizeof(int32_t),
                             cudaMemcpyHostToDevice, s));
    if (L.nb)
      H2B_CUDA(cudaMemcpyAsync(L.ci, L.h_ci.data(), L.nb * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  }
  Layer& D = A.dense;
  D.max_row = 0;
  for (int64_t r = 0; r < D.rows; ++r) D.max_row = std::max(D.max_row, D.h_rp[r + 1] - D.h_rp[r]);
  H2B_CUDA(cudaMemcpyAsync(D.rp, D.h_rp.data(), (D.rows + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  if (D.nb) H2B_CUDA(cudaMemcpyAsync(D.ci, D.h_ci.data(), D.nb * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  std::vector<const Layer*> layers;
  for (int l = 0; l <= A.q; ++l) layers.push_back(&A.cpl[l]);
  layers.push_back(&A.dense);
  const std::vector<uint32_t> w = make_work_list(layers);
  A.nwork = int64_t(w.size());
  A.work.alloc(w.size());
  if (!w.empty())
    H2B_CUDA(cudaMemcpyAsync(A.work.p, w.data(), w.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  H2B_CUDA(cudaStreamSynchronize(s));
}

void check_shape(int n, int m, int depth, const int32_t* ranks) {
  require(depth >= 0 && depth <= kMaxLevels - 1, "depth out of range");
  require(m >= 1, "leaf size must be positive");
  require(int64_t(m) << depth == n, "n must equal m * 2^depth");
  if (m > kMaxDimHmv) throw Error(H2B_UNSUPPORTED, "leaf size > 128 not supported by the compiled kernels");
  for (int l = 0; l <= depth; ++l) {
    require(ranks[l] >= 0, "ranks must be non-negative");
    if (ranks[l] > kMaxDimHmv) throw Error(H2B_UNSUPPORTED, "rank > 128 not supported by the compiled kernels");
  }
  require(int64_t(1) << (depth + 1) < (int64_t(1) << kLayerShift), "tree too deep for the work-list encoding");
}

// cols: block columns (BSRLayer::block_cols; -1: == rows, a coupling level).
void set_layer_structure(Layer& L, int64_t rows, int br, int bc, const int32_t* rp,
                         const int32_t* ci, int64_t cols = -1) {
  if (cols < 0) cols = rows;
  L.rows = rows;
  L.br = br;
  L.bc = bc;
  L.h_rp.assign(rp, rp + rows + 1);
  require(L.h_rp[0] == 0, "row_ptr must start at 0");
  for (int64_t r = 0; r < rows; ++r) require(L.h_rp[r] <= L.h_rp[r + 1], "row_ptr must be non-decreasing");
  L.nb = L.h_rp[rows];
  L.h_ci.assign(ci, ci + L.nb);
  for (int64_t r = 0; r < rows; ++r)
    for (int32_t b = L.h_rp[r]; b < L.h_rp[r + 1]; ++b)
      require(L.h_ci[b] >= 0 && L.h_ci[b] < cols, "col_idx out of range");
}

h2b_matrix* create_from_desc(const h2b_matrix_desc& d, int device) {
  require(d.symmetric == 0 || d.symmetric == 1, "symmetric must be 0 or 1");
  require(d.perm && d.ranks && d.leaf && d.cpl_row_ptr && d.dense_row_ptr, "null pointer in descriptor");
  check_shape(d.n, d.m, d.depth, d.ranks);
  const bool sym = d.symmetric == 1;
  if (!sym) {
    require(d.col_ranks && d.col_leaf, "non-symmetric descriptor: null column basis");
    check_shape(d.n, d.m, d.depth, d.col_ranks);
    require(d.m >= 1, "leaf size must be positive");
  }
  need_device(device);
  std::unique_ptr<h2b_matrix> A(new h2b_matrix);
  A->device = device;
  H2B_CUDA(cudaStreamCreateWithFlags(&A->stream, cudaStreamNonBlocking));
  A->n = d.n;
  A->m = d.m;
  A->q = d.depth;
  A->rank.assign(d.ranks, d.ranks + d.depth + 1);
  const int q = A->q;
  A->cpl.resize(q + 1);
  const int32_t* rp = d.cpl_row_ptr;
  const int32_t* ci = d.cpl_col_idx;
  for (int l = 0; l <= q; ++l) {
    set_layer_structure(A->cpl[l], A->nodes(l), A->rank[l], sym ? A->rank[l] : d.col_ranks[l], rp, ci);
    rp += A->nodes(l) + 1;
    ci += A->cpl[l].nb;
  }
  set_layer_structure(A->dense, A->nodes(q), A->m, A->m, d.dense_row_ptr, d.dense_col_idx);
  for (int t = 0; t < d.n; ++t) require(d.perm[t] >= 0 && d.perm[t] < d.n, "perm out of range");
  allocate(*A);
  if (!sym) allocate_col(*A, d.col_ranks);
  cudaStream_t s = A->stream;
  if (!sym) {
    Matrix& C = *A->colb;
    H2B_CUDA(cudaMemcpyAsync(C.perm.p, d.perm, size_t(d.n) * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    upload_blocks(d.col_leaf, C.leaf.p, C.m, C.rank[q], C.nodes(q), s);
    const double* ct = d.col_transfer;
    for (int l = 1; l <= q; ++l) {
      upload_blocks(ct, C.transfer.p + C.tr_off[l], C.rank[l], C.rank[l - 1], C.nodes(l), s);
      ct += C.nodes(l) * C.rank[l] * C.rank[l - 1];
    }
  }
  H2B_CUDA(cudaMemcpyAsync(A->perm.p, d.perm, size_t(d.n) * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  upload_blocks(d.leaf, A->leaf.p, A->m, A->rank[q], A->nodes(q), s);
  const double* tr = d.transfer;
  for (int l = 1; l <= q; ++l) {
    upload_blocks(tr, A->transfer.p + A->tr_off[l], A->rank[l], A->rank[l - 1], A->nodes(l), s);
    tr += A->nodes(l) * A->rank[l] * A->rank[l - 1];
  }
  const double* sv = d.cpl_values;
  for (int l = 0; l <= q; ++l) {
    const Layer& L = A->cpl[l];
    upload_blocks(sv, L.val, L.br, L.bc, L.nb, s);
    sv += L.nb * L.br * L.bc;
  }
  upload_blocks(d.dense_values, A->dense.val, A->m, A->m, A->dense.nb, s);
  upload_structure(*A);
  check_value_symmetry(*A);
  return A.release();
}

// ---------------------------------------------------------------- HMV driver
cudaEvent_t* timing_slots(Matrix& A) {
  if (!A.timing) return nullptr;
  if (A.ev_used + 4 > A.ev_pool.size()) {
    const size_t old = A.ev_pool.size();
    A.ev_pool.resize(std::max<size_t>(64, 2 * old));
    for (size_t i = old; i < A.ev_pool.size(); ++i) H2B_CUDA(cudaEventCreate(&A.ev_pool[i]));
  }
  cudaEvent_t* e = A.ev_pool.data() + A.ev_used;
  A.ev_used += 4;
  return e;
}

// One mat-vec on device pointers with workspace w (held by the caller).
void hmv_device(Matrix& A, Work& w, const double* x, double* y, double alpha, double beta, cudaStream_t s) {
  NvtxRange nv("h2b hmv");
  const int q = A.q;
  cudaEvent_t* ev = timing_slots(A);
  if (ev) H2B_CUDA(cudaEventRecord(ev[0], s));
  Matrix& C = A.col_basis();  // upsweep on the column basis (hmv.hpp:182)
  sweep_begin(w, A, s);
  launch_up_leaf(C, x, w.xc.p, w.xhat.p, s);
  if (q >= 1) launch_up_fused(w, C, w.xhat.p, s, q, 1, false);  // levels q..1 in one dataflow launch
  if (ev) H2B_CUDA(cudaEventRecord(ev[1], s));
  launch_bsr(A, A.work.p, A.nwork, w.xc.p, w.yc.p, w.xhat.p, w.yhat.p, s, &C);
  if (ev) H2B_CUDA(cudaEventRecord(ev[2], s));
  if (q >= 1) launch_down_fused(w, A, w.yhat.p, s, false);
  launch_down_leaf(A, w.yhat.p, w.yc.p, y, alpha, beta, true, s);
  if (ev) H2B_CUDA(cudaEventRecord(ev[3], s));
}

void hmv_for_validation(Matrix& A, const double* x, double* y, cudaStream_t s) {
  Work& w = default_work(A);
  WorkUse u(w, s);
  ensure_work(A, w);
  hmv_device(A, w, x, y, 1.0, 0.0, s);
}

double validate_sampled_device(Matrix& A, const double* points_host, int dim, double ell,
                               double fraction, uint64_t seed);

void ensure_host_stage(Matrix& A, size_t n) {
  if (A.h_stage_n >= n) return;
  if (A.h_stage) cudaFreeHost(A.h_stage);
  A.h_stage = nullptr;
  A.h_stage_n = 0;
  H2B_CUDA(cudaMallocHost(&A.h_stage, n * sizeof(double)));
  A.h_stage_n = n;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

void copy_in(double* dst, const double* src, size_t n, cudaStream_t s) {
  H2B_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyHostToDevice, s));
}

void copy_out(double* dst, const double* src, size_t n, cudaStream_t s) {
  H2B_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost, s));
}

// hmv(A, x, y, alpha, beta, ctx) (hmv.hpp:175-188); w = nullptr: the handle's
// own workspace.
void hmv(Matrix& A, Work* wp, const double* x, double* y, double alpha, double beta, h2b_ptr_kind kind,
         cudaStream_t s) {
  require(x && y, "hmv: null vector");
  require(A.part_s == 0, "hmv: partition handles use h2b_part_upsweep / h2b_part_finish");
  DeviceGuard g(A.device);
  if (!s) s = A.stream;
  Work& w = wp ? *wp : default_work(A);
  require(w.device == A.device || w.owner == nullptr, "hmv: context belongs to another device");
  const bool async_host = kind == H2B_PTR_HOST_ASYNC;
  if (async_host)
    require(is_pinned(x) && is_pinned(y), "hmv: H2B_PTR_HOST_ASYNC needs pinned (page-locked) host vectors");
  const bool dx = !async_host && resolve_device(kind, x), dy = !async_host && resolve_device(kind, y);
  bool sync = false;
  {
    WorkUse u(w, s);
    ensure_work(A, w);
    const double* xd = x;
    double* yd = y;
    if (!dx) {
      if (!w.xs.p) w.xs.alloc(A.n);
      copy_in(w.xs.p, x, A.n, s);
      xd = w.xs.p;
    }
    if (!dy) {
      if (!w.ys.p) w.ys.alloc(A.n);
      if (beta != 0.0) copy_in(w.ys.p, y, A.n, s);
      yd = w.ys.p;
    }
    hmv_device(A, w, xd, yd, alpha, beta, s);
    if (!dy) copy_out(y, w.ys.p, A.n, s);
    sync = (!dx || !dy) && !async_host;
  }
  if (sync) H2B_CUDA(cudaStreamSynchronize(s));
}

void whole(const Matrix& A, const char* what) {
  require(A.part_s == 0, std::string(what) + ": not supported on a partition handle");
}

// Phase helpers take host or device pointers; host data goes through
// temporary device buffers.
struct Staged {
  DevBuf<double> buf;
  double* d = nullptr;
  double* host = nullptr;
  size_t n = 0;
};

const double* stage_in(Staged& st, const double* p, size_t n, bool dev, cudaStream_t s) {
  if (dev) return p;
  st.buf.alloc(std::max<size_t>(n, 1));
  if (n) H2B_CUDA(cudaMemcpyAsync(st.buf.p, p, n * sizeof(double), cudaMemcpyHostToDevice, s));
  return st.buf.p;
}

double* stage_out(Staged& st, double* p, size_t n, bool dev, bool copy_existing, cudaStream_t s) {
  if (dev) return p;
  st.buf.alloc(std::max<size_t>(n, 1));
  st.host = p;
  st.n = n;
  if (copy_existing && n)
    H2B_CUDA(cudaMemcpyAsync(st.buf.p, p, n * sizeof(double), cudaMemcpyHostToDevice, s));
  return st.buf.p;
}

void finish_out(Staged& st, cudaStream_t s) {
  if (st.host && st.n)
    H2B_CUDA(cudaMemcpyAsync(st.host, st.buf.p, st.n * sizeof(double), cudaMemcpyDeviceToHost, s));
  H2B_CUDA(cudaStreamSynchronize(s));
}

}  // namespace h2b

using namespace h2b;

// Implemented in build.cu / compress.cu.
namespace h2b {
h2b_matrix* build_matrix(const h2b_build_config& cfg, int device, int nparts, int part);
void save_matrix(const Matrix& A, const std::string& path, const h2b_build_info* info);
h2b_matrix* load_matrix(const std::string& path, int device, h2b_build_info* info_out);
uint32_t crc32_bytes(const void* p, size_t n);
void compress_matrix(Matrix& A, double eps, h2b_compress_report* rep, const h2b_comm* comm = nullptr);
void release_workspaces(int device);
void orthogonalize_matrix(Matrix& A, double* t_out, bool col);
}  // namespace h2b

extern "C" {

const char* h2b_last_error(void) { return g_err.c_str(); }
const char* h2b_version(void) { return "h2b 0.1 (sm_100a, fp64)"; }
int h2b_device_count(void) { return usable_devices(); }

h2b_status h2b_release_cached_memory(int device) {
  return guarded([&] {
    require(device >= 0 && device < usable_devices(), "invalid device");
    int prev = 0;
    H2B_CUDA(cudaGetDevice(&prev));
    H2B_CUDA(cudaSetDevice(device));
    H2B_CUDA(cudaDeviceSynchronize());
    release_workspaces(device);
    H2B_CUDA(cudaSetDevice(prev));
  });
}

h2b_status h2b_matrix_create(const h2b_matrix_desc* desc, int device, h2b_matrix** out) {
  return guarded([&] {
    require(desc && out, "null argument");
    *out = create_from_desc(*desc, device);
  });
}

h2b_status h2b_matrix_build(const h2b_build_config* cfg, int device, h2b_matrix** out) {
  return guarded([&] {
    require(cfg && out, "null argument");
    *out = build_matrix(*cfg, device, 1, 0);
  });
}

h2b_status h2b_matrix_destroy(h2b_matrix* A) {
  return guarded([&] {
    if (!A) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(A->device);
    delete A;
    cudaSetDevice(prev);
  });
}

h2b_status h2b_matrix_info_get(const h2b_matrix* Ah, h2b_matrix_info* info) {
  return guarded([&] {
    require(Ah && info, "null argument");
    const Matrix& A = *Ah;
    std::memset(info, 0, sizeof(*info));
    info->n = A.n;
    info->m = A.m;
    info->depth = A.q;
    info->symmetric = A.symmetric ? 1 : 0;
    for (int l = 0; l <= A.q; ++l) {
      info->ranks[l] = A.rank[l];
      info->col_ranks[l] = A.col_basis().rank[l];
      info->cpl_blocks[l] = A.cpl[l].nb;
      info->cpl_max_row[l] = A.cpl[l].max_row;
    }
    info->dense_blocks = A.dense.nb;
    info->dense_max_row = A.dense.max_row;
    info->footprint_bytes = A.footprint();
    info->global_footprint_bytes = A.part_s ? A.global_footprint : A.footprint();
    info->part_log2 = A.part_s;
    info->part_index = A.part_g;
    info->device_bytes = A.device_bytes();
    info->hmv_flops = A.hmv_flops();
  });
}

uint64_t h2b_matrix_footprint(const h2b_matrix* A) {
  return A ? reinterpret_cast<const Matrix*>(A)->footprint() : 0;
}

h2b_status h2b_matrix_export(const h2b_matrix* Ah, int32_t* perm, double* leaf, double* transfer,
                             int32_t* cpl_row_ptr, int32_t* cpl_col_idx, double* cpl_values,
                             int32_t* dense_row_ptr, int32_t* dense_col_idx,
                             double* dense_values) {
  return guarded([&] {
    require(Ah, "null matrix");
    const Matrix& A = *Ah;
    whole(A, "h2b_matrix_export");
    DeviceGuard g(A.device);
    cudaStream_t s = A.stream;
    const int q = A.q;
    if (perm) {
      H2B_CUDA(cudaMemcpyAsync(perm, A.perm.p, size_t(A.n) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      H2B_CUDA(cudaStreamSynchronize(s));
    }
    if (leaf) download_blocks(A.leaf.p, leaf, A.m, A.rank[q], A.nodes(q), s);
    if (transfer)
      for (int l = 1; l <= q; ++l) {
        download_blocks(A.transfer.p + A.tr_off[l], transfer, A.rank[l], A.rank[l - 1], A.nodes(l), s);
        transfer += A.nodes(l) * A.rank[l] * A.rank[l - 1];
      }
    for (int l = 0; l <= q; ++l) {
      const Layer& L = A.cpl[l];
      if (cpl_row_ptr) cpl_row_ptr = std::copy(L.h_rp.begin(), L.h_rp.end(), cpl_row_ptr);
      if (cpl_col_idx) cpl_col_idx = std::copy(L.h_ci.begin(), L.h_ci.end(), cpl_col_idx);
      if (cpl_values) {
        download_blocks(L.val, cpl_values, L.br, L.bc, L.nb, s);
        cpl_values += L.nb * L.br * L.bc;
      }
    }
    if (dense_row_ptr) std::copy(A.dense.h_rp.begin(), A.dense.h_rp.end(), dense_row_ptr);
    if (dense_col_idx) std::copy(A.dense.h_ci.begin(), A.dense.h_ci.end(), dense_col_idx);
    if (dense_values) download_blocks(A.dense.val, dense_values, A.m, A.m, A.dense.nb, s);
  });
}

h2b_status h2b_matrix_export_col(const h2b_matrix* Ah, double* col_leaf, double* col_transfer) {
  return guarded([&] {
    require(Ah, "null matrix");
    const Matrix& A = *Ah;
    require(!A.symmetric, "h2b_matrix_export_col: the matrix is symmetric (column basis == row basis)");
    DeviceGuard g(A.device);
    cudaStream_t s = A.stream;
    const Matrix& C = *A.colb;
    const int q = A.q;
    if (col_leaf) download_blocks(C.leaf.p, col_leaf, C.m, C.rank[q], C.nodes(q), s);
    if (col_transfer)
      for (int l = 1; l <= q; ++l) {
        download_blocks(C.transfer.p + C.tr_off[l], col_transfer, C.rank[l], C.rank[l - 1], C.nodes(l), s);
        col_transfer += C.nodes(l) * C.rank[l] * C.rank[l - 1];
      }
  });
}

h2b_status h2b_hmv(h2b_matrix* Ah, const double* x, double* y, double alpha, double beta,
                   h2b_ptr_kind kind, void* stream) {
  return guarded([&] {
    require(Ah, "null matrix");
    hmv(*Ah, nullptr, x, y, alpha, beta, kind, static_cast<cudaStream_t>(stream));
  });
}

h2b_status h2b_context_create(h2b_matrix* Ah, h2b_context** out) {
  return guarded([&] {
    require(Ah && out, "null argument");
    Matrix& A = *Ah;
    DeviceGuard g(A.device);
    std::unique_ptr<h2b_context> c(new h2b_context);
    c->device = A.device;
    ensure_work(A, *c);
    *out = c.release();
  });
}

h2b_status h2b_context_destroy(h2b_context* c) {
  return guarded([&] {
    if (!c) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    {
      std::lock_guard<std::mutex> lk(c->mu);
      if (c->done) cudaEventSynchronize(c->done);  // no kernel may still use the buffers
    }
    delete c;
    cudaSetDevice(prev);
  });
}

h2b_status h2b_hmv_ctx(h2b_matrix* Ah, h2b_context* ctx, const double* x, double* y, double alpha, double beta,
                       h2b_ptr_kind kind, void* stream) {
  return guarded([&] {
    require(Ah, "null matrix");
    hmv(*Ah, ctx, x, y, alpha, beta, kind, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"

struct h2b_hmv_graph {
  h2b::Matrix* A = nullptr;
  h2b::Work* w = nullptr;
  uint64_t layout = 0;
  int device = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

extern "C" {

h2b_status h2b_hmv_graph_create(h2b_matrix* Ah, h2b_context* ctx, const double* x, double* y, double alpha,
                                double beta, h2b_hmv_graph** out) {
  return guarded([&] {
    require(Ah && x && y && out, "null argument");
    Matrix& A = *Ah;
    require(A.part_s == 0, "h2b_hmv_graph_create: partition handles use h2b_part_hmv");
    DeviceGuard g(A.device);
    require(resolve_device(H2B_PTR_AUTO, x) && resolve_device(H2B_PTR_AUTO, y),
            "h2b_hmv_graph_create: x and y must be device vectors");
    Work& w = ctx ? *static_cast<Work*>(ctx) : default_work(A);
    require(w.device == A.device || w.owner == nullptr, "hmv: context belongs to another device");
    std::unique_ptr<h2b_hmv_graph> G(new h2b_hmv_graph);
    {
      // size the workspace and its sweep flags outside the capture (no
      // allocation may happen inside it), then capture with the workspace held
      WorkUse u(w, A.stream);
      ensure_work(A, w);
      sweep_begin(w, A, A.stream);
    }
    H2B_CUDA(cudaStreamSynchronize(A.stream));
    std::lock_guard<std::mutex> lk(w.mu);
    cudaStream_t cs = nullptr;
    H2B_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    const bool timing = A.timing;
    A.timing = false;
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      try {
        hmv_device(A, w, x, y, alpha, beta, cs);
      } catch (...) {
        cudaGraph_t dead = nullptr;
        cudaStreamEndCapture(cs, &dead);
        if (dead) cudaGraphDestroy(dead);
        cudaStreamDestroy(cs);
        A.timing = timing;
        throw;
      }
      e = cudaStreamEndCapture(cs, &G->graph);
    }
    A.timing = timing;
    cudaStreamDestroy(cs);
    H2B_CUDA(e);
    H2B_CUDA(cudaGraphInstantiate(&G->exec, G->graph, 0));
    G->A = &A;
    G->w = &w;
    G->layout = A.layout_version;
    G->device = A.device;
    *out = G.release();
  });
}

h2b_status h2b_hmv_graph_launch(h2b_hmv_graph* G, void* stream) {
  return guarded([&] {
    require(G && G->exec, "null graph");
    Matrix& A = *G->A;
    require(A.layout_version == G->layout,
            "h2b_hmv_graph_launch: the matrix layout changed since the capture (compress); capture a new graph");
    DeviceGuard g(G->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : A.stream;
    WorkUse u(*G->w, s);
    H2B_CUDA(cudaGraphLaunch(G->exec, s));
  });
}

h2b_status h2b_hmv_graph_destroy(h2b_hmv_graph* G) {
  return guarded([&] {
    if (!G) return;
    DeviceGuard g(G->device);
    if (G->exec) cudaGraphExecDestroy(G->exec);
    if (G->graph) cudaGraphDestroy(G->graph);
    delete G;
  });
}

h2b_status h2b_hmv_multi(h2b_matrix* Ah, int nvec, const double* X, int64_t ldx, double* Y,
                         int64_t ldy, double alpha, double beta, h2b_ptr_kind kind, void* stream) {
  return guarded([&] {
    require(Ah, "null matrix");
    Matrix& A = *Ah;
    whole(A, "h2b_hmv_multi");
    require(nvec >= 0 && ldx >= A.n && ldy >= A.n, "hmv_multi: bad leading dimension");
    require(X && Y, "hmv_multi: null vector");
    if (nvec == 0) return;
    DeviceGuard g(A.device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : A.stream;
    const bool dx = resolve_device(kind, X), dy = resolve_device(kind, Y);
    DevBuf<double> xs, ys;
    const double* xd = X;
    double* yd = Y;
    int64_t lx = ldx, ly = ldy;
    if (!dx) {
      xs.alloc(size_t(A.n) * nvec);
      H2B_CUDA(cudaMemcpy2DAsync(xs.p, A.n * sizeof(double), X, ldx * sizeof(double), A.n * sizeof(double),
                                 nvec, cudaMemcpyHostToDevice, s));
      xd = xs.p;
      lx = A.n;
    }
    if (!dy) {
      ys.alloc(size_t(A.n) * nvec);
      if (beta != 0.0)
        H2B_CUDA(cudaMemcpy2DAsync(ys.p, A.n * sizeof(double), Y, ldy * sizeof(double),
                                   A.n * sizeof(double), nvec, cudaMemcpyHostToDevice, s));
      yd = ys.p;
      ly = A.n;
    }
    {
      Work& w = default_work(A);
      WorkUse u(w, s);
      ensure_work(A, w);
      if (big_matrix(A)) {  // blocks > 64: the single-vector kernels, column by column
        for (int v = 0; v < nvec; ++v) hmv_device(A, w, xd + v * lx, yd + v * ly, alpha, beta, s);
      } else {
        for (int v0 = 0; v0 < nvec; v0 += 16)
          hmv_multi_device(A, w, xd + v0 * lx, lx, yd + v0 * ly, ly, std::min(16, nvec - v0), alpha, beta, s);
      }
    }
    if (!dy)
      H2B_CUDA(cudaMemcpy2DAsync(Y, ldy * sizeof(double), ys.p, A.n * sizeof(double), A.n * sizeof(double),
                                 nvec, cudaMemcpyDeviceToHost, s));
    // host vectors: synchronous (like h2b_hmv); device vectors: stream-ordered
    if (!dx || !dy) H2B_CUDA(cudaStreamSynchronize(s));
  });
}

h2b_status h2b_upsweep(h2b_matrix* Ah, const double* xc, double* xhat, h2b_ptr_kind kind) {
  return guarded([&] {
    require(Ah && xc && xhat, "null argument");
    Matrix& A = *Ah;
    whole(A, "h2b_upsweep");
    DeviceGuard g(A.device);
    cudaStream_t s = A.stream;
    const bool dev = resolve_device(kind, xc);
    Staged si, so;
    const double* xin = stage_in(si, xc, A.n, dev, s);
    Matrix& C = A.col_basis();  // upsweep(A.col_basis(), ...) (hmv.hpp:182)
    double* out = stage_out(so, xhat, C.vec_off[A.q + 1], resolve_device(kind, xhat), false, s);
    {
      Work& w = default_work(A);
      WorkUse u(w, s);
      ensure_work(A, w);
      launch_up_leaf(C, xin, w.xc.p, w.xhat.p, s, /*cluster_order=*/true);
      for (int l = A.q; l >= 1; --l) launch_up_level(C, l, w.xhat.p, s);
      if (C.vec_off[A.q + 1])
        H2B_CUDA(cudaMemcpyAsync(out, w.xhat.p, C.vec_off[A.q + 1] * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    finish_out(so, s);
  });
}

h2b_status h2b_tree_multiply(h2b_matrix* Ah, const double* xhat, double* yhat, h2b_ptr_kind kind) {
  return guarded([&] {
    require(Ah && xhat && yhat, "null argument");
    Matrix& A = *Ah;
    whole(A, "h2b_tree_multiply");
    DeviceGuard g(A.device);
    cudaStream_t s = A.stream;
    const Matrix& C = A.col_basis();
    const size_t nv = A.vec_off[A.q + 1], nx = C.vec_off[A.q + 1];
    Staged si, so;
    const double* xin = stage_in(si, xhat, nx, resolve_device(kind, xhat), s);
    double* out = stage_out(so, yhat, nv, resolve_device(kind, yhat), false, s);
    // coupling layers only: work items with layer index <= q
    std::vector<const Layer*> layers;
    for (int l = 0; l <= A.q; ++l) layers.push_back(&A.cpl[l]);
    const auto w = make_work_list(layers);
    DevBuf<uint32_t> dw;
    dw.alloc(w.size());
    if (!w.empty())
      H2B_CUDA(cudaMemcpyAsync(dw.p, w.data(), w.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    launch_bsr(A, dw.p, int64_t(w.size()), nullptr, nullptr, xin, out, s, &C);
    finish_out(so, s);
  });
}

// downsweep(U, yhat, y, n) (hmv.hpp:129-157): yhat is updated in place
// (y^l += E y^{l-1}), y += U y^q.
h2b_status h2b_downsweep(h2b_matrix* Ah, double* yhat, double* yc, h2b_ptr_kind kind) {
  return guarded([&] {
    require(Ah && yhat && yc, "null argument");
    Matrix& A = *Ah;
    whole(A, "h2b_downsweep");
    DeviceGuard g(A.device);
    cudaStream_t s = A.stream;
    const size_t nv = A.vec_off[A.q + 1];
    Staged sh, so;
    double* yh = stage_out(sh, yhat, nv, resolve_device(kind, yhat), true, s);
    double* out = stage_out(so, yc, A.n, resolve_device(kind, yc), true, s);
    {
      Work& w = default_work(A);
      WorkUse u(w, s);
      ensure_work(A, w);
      H2B_CUDA(cudaMemcpyAsync(w.yc.p, out, A.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
      for (int l = 1; l <= A.q; ++l) launch_down_level(A, l, yh, s);
      launch_down_leaf(A, yh, w.yc.p, out, 1.0, 0.0, false, s);
    }
    finish_out(sh, s);
    finish_out(so, s);
  });
}

h2b_status h2b_dense_mv(h2b_matrix* Ah, const double* xc, double* yc, double alpha, double beta,
                        h2b_ptr_kind kind) {
  return guarded([&] {
    require(Ah && xc && yc, "null argument");
    Matrix& A = *Ah;
    whole(A, "h2b_dense_mv");
    require(alpha == 1.0 && beta == 0.0, "h2b_dense_mv: only alpha = 1, beta = 0 (the hmv call site) is implemented");
    DeviceGuard g(A.device);
    cudaStream_t s = A.stream;
    Staged si, so;
    const double* xin = stage_in(si, xc, A.n, resolve_device(kind, xc), s);
    double* out = stage_out(so, yc, A.n, resolve_device(kind, yc), false, s);
    std::vector<const Layer*> layers(A.q + 1, nullptr);
    layers.push_back(&A.dense);
    const auto w = make_work_list(layers);
    DevBuf<uint32_t> dw;
    dw.alloc(w.size());
    if (!w.empty())
      H2B_CUDA(cudaMemcpyAsync(dw.p, w.data(), w.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    launch_bsr(A, dw.p, int64_t(w.size()), xin, out, nullptr, nullptr, s);
    finish_out(so, s);
  });
}

h2b_status h2b_compress(h2b_matrix* Ah, double eps, h2b_compress_report* report) {
  return guarded([&] {
    require(Ah, "null matrix");
    whole(*Ah, "h2b_compress");
    compress_matrix(*Ah, eps, report);
  });
}

uint32_t h2b_crc32(const void* data, uint64_t len) { return crc32_bytes(data, size_t(len)); }

h2b_status h2b_matrix_save(const h2b_matrix* Ah, const char* path, const h2b_build_info* info) {
  return guarded([&] {
    require(Ah && path, "null argument");
    DeviceGuard g(Ah->device);
    save_matrix(*Ah, path, info);
  });
}

h2b_status h2b_matrix_load(const char* path, int device, h2b_matrix** out, h2b_build_info* info) {
  return guarded([&] {
    require(path && out, "null argument");
    *out = load_matrix(path, device, info);
  });
}

h2b_status h2b_part_compress(h2b_matrix* Ah, double eps, const h2b_comm* comm, h2b_compress_report* report) {
  return guarded([&] {
    require(Ah, "null matrix");
    if (Ah->part_s > 0)
      require(comm && comm->allgather && comm->allreduce_max_i32 && comm->allreduce_sum_f64,
              "h2b_part_compress: a partition handle needs a communicator");
    compress_matrix(*Ah, eps, report, Ah->part_s > 0 ? comm : nullptr);
  });
}

// orthogonalize_basis(A.row_basis) / orthogonalize_basis(A.col_basis())
// (compression.hpp:69-126, h2_matrix.hpp:69-78); symmetric: the same tree.
h2b_status h2b_orthogonalize(h2b_matrix* Ah, double* t_out) {
  return guarded([&] {
    require(Ah, "null matrix");
    whole(*Ah, "h2b_orthogonalize");
    orthogonalize_matrix(*Ah, t_out, false);
  });
}

h2b_status h2b_orthogonalize_col(h2b_matrix* Ah, double* t_out) {
  return guarded([&] {
    require(Ah, "null matrix");
    whole(*Ah, "h2b_orthogonalize_col");
    orthogonalize_matrix(*Ah, t_out, true);
  });
}

h2b_status h2b_matrix_build_part(const h2b_build_config* cfg, int device, int nparts, int part,
                                  h2b_matrix** out) {
  return guarded([&] {
    require(cfg && out, "null argument");
    *out = build_matrix(*cfg, device, nparts, part);
  });
}

h2b_status h2b_workspace(h2b_matrix* Ah, int which, void** ptr, int64_t* count) {
  return guarded([&] {
    require(Ah && ptr && count, "null argument");
    Matrix& A = *Ah;
    DeviceGuard g(A.device);
    Work& w = default_work(A);
    {
      WorkUse u(w, A.stream);
      ensure_work(A, w);
    }
    switch (which) {
      case H2B_WS_XHAT: *ptr = w.xhat.p; *count = A.col_basis().vec_off[A.q + 1]; break;
      case H2B_WS_YHAT: *ptr = w.yhat.p; *count = A.vec_off[A.q + 1]; break;
      case H2B_WS_XC: *ptr = w.xc.p; *count = A.n; break;
      case H2B_WS_PERM: *ptr = A.perm.p; *count = A.n; break;
      default: require(false, "h2b_workspace: unknown buffer");
    }
  });
}

h2b_status h2b_part_upsweep(h2b_matrix* Ah, const double* x, void* stream) {
  return guarded([&] {
    require(Ah && x, "null argument");
    Matrix& A = *Ah;
    DeviceGuard g(A.device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : A.stream;
    Work& w = default_work(A);
    WorkUse u(w, s);
    ensure_work(A, w);
    sweep_begin(w, A, s);
    launch_up_leaf(A, x, w.xc.p, w.xhat.p, s);
    launch_gather(A.perm.p, x, w.xc.p, A.n, s);  // dense blocks read remote columns
    // this partition's levels q..s+1: one dataflow launch over its nodes
    if (A.q > A.part_s) launch_up_fused(w, A, w.xhat.p, s, A.q, A.part_s + 1, true);
  });
}

h2b_status h2b_part_finish(h2b_matrix* Ah, double* y_slice, void* stream) {
  return guarded([&] {
    require(Ah && y_slice, "null argument");
    Matrix& A = *Ah;
    DeviceGuard g(A.device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : A.stream;
    Work& w = default_work(A);
    WorkUse u(w, s);
    ensure_work(A, w);
    cudaEvent_t* ev = timing_slots(A);
    if (ev) H2B_CUDA(cudaEventRecord(ev[0], s));
    // replicated top (level s's x^ gathered from every partition)
    if (A.part_s >= 1) launch_up_fused(w, A, w.xhat.p, s, A.part_s, 1, false);
    if (ev) H2B_CUDA(cudaEventRecord(ev[1], s));
    launch_bsr(A, A.work.p, A.nwork, w.xc.p, w.yc.p, w.xhat.p, w.yhat.p, s);
    if (ev) H2B_CUDA(cudaEventRecord(ev[2], s));
    if (A.q >= 1) launch_down_fused(w, A, w.yhat.p, s, true);  // replicated top + own subtree
    launch_down_leaf(A, w.yhat.p, w.yc.p, y_slice, 1.0, 0.0, false, s);
    if (ev) H2B_CUDA(cudaEventRecord(ev[3], s));
  });
}

namespace {
// comm->allgather of nparts slices of `count` doubles in buf, stream-ordered.
void dcomm_allgather(const h2b_dcomm* comm, double* buf, int64_t count, cudaStream_t s) {
  if (comm->allgather(comm->ctx, buf, count, s) != 0) throw Error(H2B_CUDA_ERROR, "communicator: allgather failed");
}

void require_dcomm(const Matrix& A, const h2b_dcomm* comm) {
  require(A.symmetric, "partitioned mat-vec: symmetric matrices only");
  require(A.part_s == 0 || (comm && comm->allgather), "partitioned mat-vec: null communicator");
}
}  // namespace

namespace {
// One partitioned mat-vec on device vectors with workspace w (held by the caller).
void part_hmv_device(Matrix& A, Work& w, const double* x, double* y, double alpha, double beta, int y_mode,
                     const h2b_dcomm* comm, cudaStream_t s) {
  const int nparts = 1 << A.part_s;
  cudaEvent_t* ev = timing_slots(A);  // upsweep + exchange | coupling + dense | downsweep + y
  if (ev) H2B_CUDA(cudaEventRecord(ev[0], s));
  sweep_begin(w, A, s);
  launch_up_leaf(A, x, w.xc.p, w.xhat.p, s);
  if (A.part_s > 0) launch_gather(A.perm.p, x, w.xc.p, A.n, s);  // dense blocks read remote columns
  if (A.q > A.part_s) launch_up_fused(w, A, w.xhat.p, s, A.q, A.part_s + 1, true);
  if (nparts > 1) {  // one all-gather of every level >= s
    const int64_t cnt = part_exchange_count(A, 1);
    if (w.xg.n < size_t(cnt) * nparts) w.xg.alloc(size_t(cnt) * nparts);
    launch_pack_xhat(A, 1, w.xhat.p, w.xg.p, s);
    dcomm_allgather(comm, w.xg.p, cnt, s);
    launch_unpack_xhat(A, 1, w.xg.p, w.xhat.p, s);
  }
  if (A.part_s >= 1) launch_up_fused(w, A, w.xhat.p, s, A.part_s, 1, false);  // replicated top
  if (ev) H2B_CUDA(cudaEventRecord(ev[1], s));
  launch_bsr(A, A.work.p, A.nwork, w.xc.p, w.yc.p, w.xhat.p, w.yhat.p, s);
  if (ev) H2B_CUDA(cudaEventRecord(ev[2], s));
  if (A.q >= 1) launch_down_fused(w, A, w.yhat.p, s, true);
  if (y_mode == H2B_Y_OWNED || nparts == 1) {
    launch_down_leaf(A, w.yhat.p, w.yc.p, y, alpha, beta, true, s);  // owned rows, original order
  } else {
    const int64_t slice = A.n / nparts;
    if (w.yg.n < size_t(A.n)) w.yg.alloc(A.n);
    launch_down_leaf(A, w.yhat.p, w.yc.p, w.yg.p + A.part_g * slice, 1.0, 0.0, false, s);
    dcomm_allgather(comm, w.yg.p, slice, s);
    launch_scatter(A.perm.p, w.yg.p, y, A.n, alpha, beta, s);
  }
  if (ev) H2B_CUDA(cudaEventRecord(ev[3], s));
}
}  // namespace

h2b_status h2b_part_hmv(h2b_matrix* Ah, const double* x, double* y, double alpha, double beta, int y_mode,
                        const h2b_dcomm* comm, void* stream) {
  return guarded([&] {
    require(Ah && x && y, "null argument");
    require(y_mode == H2B_Y_REPLICATED || y_mode == H2B_Y_OWNED, "h2b_part_hmv: bad y_mode");
    Matrix& A = *Ah;
    require_dcomm(A, comm);
    DeviceGuard g(A.device);
    require(resolve_device(H2B_PTR_AUTO, x) && resolve_device(H2B_PTR_AUTO, y), "h2b_part_hmv: device vectors");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : A.stream;
    Work& w = default_work(A);
    WorkUse u(w, s);
    ensure_work(A, w);
    part_hmv_device(A, w, x, y, alpha, beta, y_mode, comm, s);
  });
}

h2b_status h2b_part_hmv_multi(h2b_matrix* Ah, int nvec, const double* X, int64_t ldx, double* Y, int64_t ldy,
                              double alpha, double beta, int y_mode, const h2b_dcomm* comm, void* stream) {
  return guarded([&] {
    require(Ah, "null matrix");
    require(y_mode == H2B_Y_REPLICATED || y_mode == H2B_Y_OWNED, "h2b_part_hmv_multi: bad y_mode");
    Matrix& A = *Ah;
    require_dcomm(A, comm);
    require(nvec >= 0 && ldx >= A.n && ldy >= A.n, "hmv_multi: bad leading dimension");
    require(X && Y, "hmv_multi: null vector");
    if (nvec == 0) return;
    DeviceGuard g(A.device);
    require(resolve_device(H2B_PTR_AUTO, X) && resolve_device(H2B_PTR_AUTO, Y), "h2b_part_hmv_multi: device vectors");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : A.stream;
    const int nparts = 1 << A.part_s;
    constexpr int NV = 16;
    Work& w = default_work(A);
    WorkUse u(w, s);
    ensure_work(A, w);
    if (big_matrix(A)) {  // blocks > 64: the single-vector kernels, column by column
      for (int v = 0; v < nvec; ++v) part_hmv_device(A, w, X + v * ldx, Y + v * ldy, alpha, beta, y_mode, comm, s);
      return;
    }
    for (int v0 = 0; v0 < nvec; v0 += NV) {
      const int nv = std::min(NV, nvec - v0);
      const double* Xv = X + v0 * ldx;
      double* Yv = Y + v0 * ldy;
      part_mv_upsweep(A, w, Xv, ldx, nv, s);
      if (nparts > 1) {
        const int64_t cnt = part_exchange_count(A, NV);
        if (w.xg.n < size_t(cnt) * nparts) w.xg.alloc(size_t(cnt) * nparts);
        launch_pack_xhat(A, NV, w.xh16.p, w.xg.p, s);
        dcomm_allgather(comm, w.xg.p, cnt, s);
        launch_unpack_xhat(A, NV, w.xg.p, w.xh16.p, s);
      }
      if (y_mode == H2B_Y_OWNED || nparts == 1) {
        part_mv_finish(A, w, Yv, ldy, nv, alpha, beta, nullptr, s);
      } else {
        const int64_t slice = int64_t(A.n / nparts) * NV;
        if (w.yg.n < size_t(A.n) * NV) w.yg.alloc(size_t(A.n) * NV);
        part_mv_finish(A, w, Yv, ldy, nv, alpha, beta, w.yg.p + A.part_g * slice, s);
        dcomm_allgather(comm, w.yg.p, slice, s);
        launch_scatter_mv(A.perm.p, w.yg.p, A.n, nv, Yv, ldy, alpha, beta, s);
      }
    }
  });
}

h2b_status h2b_validate_sampled(h2b_matrix* Ah, const double* points, int dim, double ell,
                                double fraction, uint64_t seed, double* err) {
  return guarded([&] {
    require(Ah && err, "null argument");
    Matrix& A = *Ah;
    whole(A, "h2b_validate_sampled");
    DeviceGuard g(A.device);
    if (!points) {
      if (dim <= 0) dim = A.pts_dim;
      if (ell <= 0) ell = A.ell;
    }
    *err = validate_sampled_device(A, points, dim, ell, fraction, seed);
  });
}

h2b_status h2b_last_hmv_timing(h2b_matrix* Ah, double* ms4) {
  return guarded([&] {
    require(Ah && ms4, "null argument");
    Matrix& A = *Ah;
    DeviceGuard g(A.device);
    for (int i = 0; i < 4; ++i) ms4[i] = 0.0;
    const size_t calls = A.ev_used / 4;
    for (size_t c = 0; c < calls; ++c) {
      cudaEvent_t* e = A.ev_pool.data() + 4 * c;
      H2B_CUDA(cudaEventSynchronize(e[3]));
      for (int i = 0; i < 3; ++i) {
        float t = 0;
        H2B_CUDA(cudaEventElapsedTime(&t, e[i], e[i + 1]));
        ms4[i] += t;
        ms4[3] += t;
      }
    }
    if (calls)
      for (int i = 0; i < 4; ++i) ms4[i] /= double(calls);
    A.ev_used = 0;
  });
}

h2b_status h2b_set_phase_timing(h2b_matrix* Ah, int on) {
  return guarded([&] {
    require(Ah, "null matrix");
    Matrix& A = *Ah;
    A.timing = on != 0;
    A.ev_used = 0;
  });
}

}  // extern "C"
