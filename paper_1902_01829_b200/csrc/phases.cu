// The reference's phase API on its component objects:
//   BasisTree<double>  (h2_matrix.hpp:17-41)  -> h2b_basis
//   MatrixTree<double> (h2_matrix.hpp:46-51)  -> h2b_mtree
//   BSRLayer<double>   (bsr.hpp:13-31)        -> h2b_layer
// and the functions that take them:
//   upsweep / downsweep (hmv.hpp:79-111,129-157), tree_multiply (:114-125),
//   block_sparse_mv (bsr.hpp:79-82), orthogonalize_basis (compression.hpp:69-126),
//   project_coupling (:130-169), generate_weight_tree (:213-256),
//   truncate_basis (:267-420).
// Each handle is a device Matrix holding only its part (a basis-only or a
// coupling-only H^2 matrix), so the same kernels run as in hmv() / compress().
// ProjectionTree / WeightTree cross the boundary as the reference's pools
// concatenated over levels (rows[l] x cols[l] per node, column-major).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "h2b_internal.hpp"

namespace h2b {

// capi.cu
void allocate(Matrix& A);
void allocate_col(Matrix& A, const int32_t* cranks);
void upload_structure(Matrix& A);
void check_value_symmetry(Matrix& A);
void set_layer_structure(Layer& L, int64_t rows, int br, int bc, const int32_t* rp, const int32_t* ci,
                         int64_t cols = -1);
void download_blocks(const double* d, double* h, int rows, int cols, int64_t count, cudaStream_t s);
void upload_blocks_sync(const double* h, double* d, int rows, int cols, int64_t count, cudaStream_t s);
h2b_status guarded_call(const std::function<void()>& f);
void need_device_public(int device);
bool resolve_device_public(h2b_ptr_kind kind, const void* p);
// compress.cu
void phase_orthogonalize(Matrix& B, double* t_dev, cudaStream_t s);
void phase_project(Matrix& S, const double* tr, const std::vector<int>& tr_rows, const std::vector<int>& tr_cols,
                   const double* tc, const std::vector<int>& tc_rows, const std::vector<int>& tc_cols, bool same,
                   cudaStream_t s);
void phase_weights(Matrix& S, Matrix& B, double* r_dev, cudaStream_t s);
void phase_truncate(Matrix& B, const double* r_dev, double eps, double* t_dev, std::vector<double>& energy,
                    cudaStream_t s);

namespace {

struct Dev {
  int prev = -1;
  explicit Dev(int d) {
    cudaGetDevice(&prev);
    H2B_CUDA(cudaSetDevice(d));
  }
  ~Dev() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Host or device array of n doubles as a device pointer (host data copied in).
struct In {
  DevBuf<double> buf;
  const double* p = nullptr;
  In(const double* src, size_t n, cudaStream_t s) {
    if (!src || n == 0 || resolve_device_public(H2B_PTR_AUTO, src)) {
      p = src;
      return;
    }
    buf.alloc(n);
    H2B_CUDA(cudaMemcpyAsync(buf.p, src, n * sizeof(double), cudaMemcpyHostToDevice, s));
    p = buf.p;
  }
};

// Output array of n doubles (host or device): device scratch when host, copied
// back by finish().  copy_in: the caller's data is input too.
struct Out {
  DevBuf<double> buf;
  double* host = nullptr;
  double* p = nullptr;
  size_t n = 0;
  Out(double* dst, size_t cnt, bool copy_in, cudaStream_t s) : n(cnt) {
    if (!dst || cnt == 0 || resolve_device_public(H2B_PTR_AUTO, dst)) {
      p = dst;
      return;
    }
    host = dst;
    buf.alloc(cnt);
    p = buf.p;
    if (copy_in) H2B_CUDA(cudaMemcpyAsync(buf.p, dst, cnt * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  void finish(cudaStream_t s) {
    if (host && n) H2B_CUDA(cudaMemcpyAsync(host, buf.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    H2B_CUDA(cudaStreamSynchronize(s));
  }
};

std::vector<int> tree_shape(const int32_t* v, int q, const char* what) {
  require(v != nullptr, std::string(what) + ": null shape");
  std::vector<int> r(v, v + q + 1);
  for (int x : r) require(x >= 0, std::string(what) + ": negative dimension");
  return r;
}

size_t tree_size(int q, const std::vector<int>& r, const std::vector<int>& c) {
  size_t t = 0;
  for (int l = 0; l <= q; ++l) t += (size_t(1) << l) * r[l] * c[l];
  return t;
}

// A basis-only Matrix: leaves + transfers, no coupling / dense blocks.
h2b_matrix* make_basis(const h2b_basis_desc& d, int device) {
  require(d.depth >= 0 && d.depth <= kMaxLevels - 1, "depth out of range");
  require(d.m >= 1, "leaf size must be positive");
  require(d.ranks && (d.leaf || d.ranks[d.depth] == 0), "null pointer in basis descriptor");
  for (int l = 0; l <= d.depth; ++l) {
    require(d.ranks[l] >= 0, "ranks must be non-negative");
    if (d.ranks[l] > kMaxDimHmv) throw Error(H2B_UNSUPPORTED, "rank > 128 not supported by the compiled kernels");
  }
  if (d.m > kMaxDimHmv) throw Error(H2B_UNSUPPORTED, "leaf size > 128 not supported by the compiled kernels");
  need_device_public(device);
  std::unique_ptr<h2b_matrix> A(new h2b_matrix);
  A->device = device;
  H2B_CUDA(cudaStreamCreateWithFlags(&A->stream, cudaStreamNonBlocking));
  A->m = d.m;
  A->q = d.depth;
  A->n = int(int64_t(d.m) << d.depth);
  A->rank.assign(d.ranks, d.ranks + d.depth + 1);
  const int q = A->q;
  A->cpl.resize(q + 1);
  for (int l = 0; l <= q; ++l) {
    std::vector<int32_t> rp(A->nodes(l) + 1, 0);
    set_layer_structure(A->cpl[l], A->nodes(l), A->rank[l], A->rank[l], rp.data(), nullptr);
  }
  std::vector<int32_t> drp(A->nodes(q) + 1, 0);
  set_layer_structure(A->dense, A->nodes(q), A->m, A->m, drp.data(), nullptr);
  allocate(*A);
  cudaStream_t s = A->stream;
  upload_blocks_sync(d.leaf, A->leaf.p, A->m, A->rank[q], A->nodes(q), s);
  const double* tr = d.transfer;
  for (int l = 1; l <= q; ++l) {
    const int64_t cnt = A->nodes(l) * int64_t(A->rank[l]) * A->rank[l - 1];
    if (cnt) require(tr != nullptr, "null transfer pool in basis descriptor");
    upload_blocks_sync(tr, A->transfer.p + A->tr_off[l], A->rank[l], A->rank[l - 1], A->nodes(l), s);
    if (cnt) tr += cnt;
  }
  H2B_CUDA(cudaStreamSynchronize(s));
  return A.release();
}

void check_layer_desc(const h2b_layer_desc& L, int64_t want_rows, int64_t want_cols) {
  require(L.block_rows >= 0 && L.block_cols >= 0 && L.brows >= 0 && L.bcols >= 0, "layer: negative dimension");
  if (want_rows >= 0) require(L.block_rows == want_rows && L.block_cols == want_cols,
                              "tree level: block_rows / block_cols must be 2^l");
  require(L.row_ptr != nullptr, "layer: null row_ptr");
  if (L.brows > kMaxDimHmv || L.bcols > kMaxDimHmv)
    throw Error(H2B_UNSUPPORTED, "block dimension > 128 not supported by the compiled kernels");
}

// A coupling-only Matrix (MatrixTree): level l holds 2^l x 2^l blocks of
// brows[l] x bcols[l]; rank = brows, the column "basis" carries bcols (its
// x^ offsets), no leaves / transfers / dense blocks.
h2b_matrix* make_mtree(int nlevels, const h2b_layer_desc* lv, int device) {
  require(nlevels >= 1 && nlevels <= kMaxLevels, "matrix tree: level count out of range");
  require(lv != nullptr, "null argument");
  const int q = nlevels - 1;
  std::vector<int32_t> br(q + 1), bc(q + 1);
  bool square = true;
  for (int l = 0; l <= q; ++l) {
    check_layer_desc(lv[l], int64_t(1) << l, int64_t(1) << l);
    br[l] = lv[l].brows;
    bc[l] = lv[l].bcols;
    square = square && br[l] == bc[l];
  }
  need_device_public(device);
  std::unique_ptr<h2b_matrix> A(new h2b_matrix);
  A->device = device;
  H2B_CUDA(cudaStreamCreateWithFlags(&A->stream, cudaStreamNonBlocking));
  A->m = 0;  // no leaves: the leaf / dense pools stay empty
  A->q = q;
  A->n = 0;
  A->rank.assign(br.begin(), br.end());
  A->cpl.resize(q + 1);
  for (int l = 0; l <= q; ++l)
    set_layer_structure(A->cpl[l], A->nodes(l), br[l], bc[l], lv[l].row_ptr, lv[l].col_idx);
  std::vector<int32_t> drp(A->nodes(q) + 1, 0);
  set_layer_structure(A->dense, A->nodes(q), 0, 0, drp.data(), nullptr);
  allocate(*A);
  if (!square) allocate_col(*A, bc.data());
  cudaStream_t s = A->stream;
  for (int l = 0; l <= q; ++l) {
    const Layer& L = A->cpl[l];
    if (L.nb) require(lv[l].values != nullptr, "layer: null values");
    upload_blocks_sync(lv[l].values, L.val, L.br, L.bc, L.nb, s);
  }
  upload_structure(*A);
  check_value_symmetry(*A);
  return A.release();
}

}  // namespace
}  // namespace h2b

using namespace h2b;

struct h2b_basis : h2b::Matrix {};
struct h2b_mtree : h2b::Matrix {};
struct h2b_layer {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t block_cols = 0;
  h2b::Layer L;
  h2b::DevBuf<double> val;
  h2b::DevBuf<int32_t> rp, ci;
  ~h2b_layer() {
    if (stream) {
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }
};

extern "C" {

// ---------------------------------------------------------------- BasisTree
h2b_status h2b_basis_create(const h2b_basis_desc* desc, int device, h2b_basis** out) {
  return guarded_call([&] {
    require(desc && out, "null argument");
    *out = reinterpret_cast<h2b_basis*>(make_basis(*desc, device));
  });
}

h2b_status h2b_basis_destroy(h2b_basis* B) {
  return guarded_call([&] {
    if (!B) return;
    Dev g(B->device);
    delete static_cast<h2b_matrix*>(static_cast<Matrix*>(B));
  });
}

h2b_status h2b_basis_shape(const h2b_basis* B, int32_t* m, int32_t* depth, int32_t* ranks) {
  return guarded_call([&] {
    require(B, "null basis");
    if (m) *m = B->m;
    if (depth) *depth = B->q;
    if (ranks) std::copy(B->rank.begin(), B->rank.end(), ranks);
  });
}

h2b_status h2b_basis_export(const h2b_basis* B, double* leaf, double* transfer) {
  return guarded_call([&] {
    require(B, "null basis");
    Dev g(B->device);
    cudaStream_t s = B->stream;
    const int q = B->q;
    if (leaf) download_blocks(B->leaf.p, leaf, B->m, B->rank[q], B->nodes(q), s);
    if (transfer)
      for (int l = 1; l <= q; ++l) {
        download_blocks(B->transfer.p + B->tr_off[l], transfer, B->rank[l], B->rank[l - 1], B->nodes(l), s);
        transfer += B->nodes(l) * B->rank[l] * B->rank[l - 1];
      }
  });
}

// upsweep(V, x, n, xhat) (hmv.hpp:79-111): x in cluster order; xhat level-concatenated.
h2b_status h2b_basis_upsweep(h2b_basis* V, const double* x, int64_t n, double* xhat, h2b_ptr_kind kind) {
  return guarded_call([&] {
    require(V && x && xhat, "null argument");
    Matrix& B = *V;
    require(int64_t(B.nodes(B.q)) * B.m == n, "upsweep: dim mismatch");
    Dev g(B.device);
    cudaStream_t s = B.stream;
    (void)kind;
    In xin(x, size_t(n), s);
    Out xo(xhat, size_t(B.vec_off[B.q + 1]), false, s);
    Work& w = default_work(B);
    {
      WorkUse u(w, s);
      ensure_work(B, w);
      launch_up_leaf(B, xin.p, w.xc.p, xo.p ? xo.p : w.xhat.p, s, /*cluster_order=*/true);
      for (int l = B.q; l >= 1; --l) launch_up_level(B, l, xo.p ? xo.p : w.xhat.p, s);
    }
    xo.finish(s);
  });
}

// downsweep(U, yhat, y, n) (hmv.hpp:129-157): yhat in/out (y^l += E y^{l-1}), y += U y^q.
h2b_status h2b_basis_downsweep(h2b_basis* U, double* yhat, double* y, int64_t n, h2b_ptr_kind kind) {
  return guarded_call([&] {
    require(U && yhat && y, "null argument");
    Matrix& B = *U;
    require(int64_t(B.nodes(B.q)) * B.m == n, "downsweep: dim mismatch");
    Dev g(B.device);
    cudaStream_t s = B.stream;
    (void)kind;
    Out yh(yhat, size_t(B.vec_off[B.q + 1]), true, s);
    Out yo(y, size_t(n), true, s);
    Work& w = default_work(B);
    {
      WorkUse u(w, s);
      ensure_work(B, w);
      H2B_CUDA(cudaMemcpyAsync(w.yc.p, yo.p, size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
      for (int l = 1; l <= B.q; ++l) launch_down_level(B, l, yh.p, s);
      launch_down_leaf(B, yh.p, w.yc.p, yo.p, 1.0, 0.0, false, s);
    }
    yh.finish(s);
    yo.finish(s);
  });
}

// orthogonalize_basis(B) (compression.hpp:69-126): B in place; t_out = T.
h2b_status h2b_orthogonalize_basis(h2b_basis* Bh, double* t_out) {
  return guarded_call([&] {
    require(Bh, "null basis");
    Matrix& B = *Bh;
    Dev g(B.device);
    cudaStream_t s = B.stream;
    const size_t nt = std::max<size_t>(1, tree_size(B.q, B.rank, B.rank));
    DevBuf<double> T;
    T.alloc(nt);
    phase_orthogonalize(B, T.p, s);
    ++B.layout_version;
    if (t_out) {
      Out to(t_out, tree_size(B.q, B.rank, B.rank), false, s);
      if (to.n) H2B_CUDA(cudaMemcpyAsync(to.p, T.p, to.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
      to.finish(s);
    }
  });
}

// truncate_basis(B, R, eps, Tout) (compression.hpp:267-420): B truncated in
// place.  r_tree: the weight tree (ranks[l]^2 per node); t_out: Tout,
// new_ranks[l] x old_ranks[l] per node (capacity: old_ranks[l]^2 per node);
// new_ranks / discarded_energy: TruncationResult (depth + 1 each, may be NULL).
h2b_status h2b_truncate_basis(h2b_basis* Bh, const double* r_tree, double eps, double* t_out, int32_t* new_ranks,
                              double* discarded_energy) {
  return guarded_call([&] {
    require(Bh && r_tree, "null argument");
    require(eps >= 0.0, "truncate_basis: eps must be non-negative");
    Matrix& B = *Bh;
    Dev g(B.device);
    cudaStream_t s = B.stream;
    const std::vector<int> old = B.rank;
    In R(r_tree, tree_size(B.q, old, old), s);
    DevBuf<double> T;
    T.alloc(std::max<size_t>(1, tree_size(B.q, old, old)));
    std::vector<double> energy;
    phase_truncate(B, R.p, eps, T.p, energy, s);
    if (t_out) {
      Out to(t_out, tree_size(B.q, B.rank, old), false, s);
      if (to.n) H2B_CUDA(cudaMemcpyAsync(to.p, T.p, to.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
      to.finish(s);
    }
    if (new_ranks) std::copy(B.rank.begin(), B.rank.end(), new_ranks);
    if (discarded_energy) std::copy(energy.begin(), energy.end(), discarded_energy);
  });
}

// ---------------------------------------------------------------- BSRLayer
h2b_status h2b_layer_create(const h2b_layer_desc* d, int device, h2b_layer** out) {
  return guarded_call([&] {
    require(d && out, "null argument");
    check_layer_desc(*d, -1, -1);
    need_device_public(device);
    std::unique_ptr<h2b_layer> H(new h2b_layer);
    H->device = device;
    H2B_CUDA(cudaStreamCreateWithFlags(&H->stream, cudaStreamNonBlocking));
    H->block_cols = d->block_cols;
    Layer& L = H->L;
    set_layer_structure(L, d->block_rows, d->brows, d->bcols, d->row_ptr, d->col_idx, d->block_cols);
    L.ld = pad2(L.br);
    H->val.alloc(std::max<int64_t>(1, L.nb * L.block_stride()));
    H->rp.alloc(L.rows + 1);
    H->ci.alloc(std::max<int64_t>(1, L.nb));
    L.val = H->val.p;
    L.rp = H->rp.p;
    L.ci = H->ci.p;
    cudaStream_t s = H->stream;
    H2B_CUDA(cudaMemcpyAsync(L.rp, L.h_rp.data(), (L.rows + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    if (L.nb) {
      require(d->values != nullptr, "layer: null values");
      H2B_CUDA(cudaMemcpyAsync(L.ci, L.h_ci.data(), L.nb * sizeof(int32_t), cudaMemcpyHostToDevice, s));
      upload_blocks_sync(d->values, L.val, L.br, L.bc, L.nb, s);
    }
    H2B_CUDA(cudaStreamSynchronize(s));
    *out = H.release();
  });
}

h2b_status h2b_layer_destroy(h2b_layer* H) {
  return guarded_call([&] {
    if (!H) return;
    Dev g(H->device);
    delete H;
  });
}

// block_sparse_mv(L, x, y, alpha, beta) (bsr.hpp:79-82); beta == 0 never reads y.
h2b_status h2b_block_sparse_mv(h2b_layer* H, const double* x, double* y, double alpha, double beta,
                               h2b_ptr_kind kind) {
  return guarded_call([&] {
    require(H && x && y, "null argument");
    Dev g(H->device);
    cudaStream_t s = H->stream;
    (void)kind;
    const Layer& L = H->L;
    In xin(x, size_t(H->block_cols) * L.bc, s);
    Out yo(y, size_t(L.rows) * L.br, beta != 0.0, s);
    launch_bsr_exact(L, xin.p, yo.p, alpha, beta, s);
    yo.finish(s);
  });
}

// ---------------------------------------------------------------- MatrixTree
h2b_status h2b_mtree_create(int32_t nlevels, const h2b_layer_desc* levels, int device, h2b_mtree** out) {
  return guarded_call([&] {
    require(out, "null argument");
    *out = reinterpret_cast<h2b_mtree*>(make_mtree(nlevels, levels, device));
  });
}

h2b_status h2b_mtree_destroy(h2b_mtree* S) {
  return guarded_call([&] {
    if (!S) return;
    Dev g(S->device);
    delete static_cast<h2b_matrix*>(static_cast<Matrix*>(S));
  });
}

// Block shapes and counts per level (they change with project_coupling).
h2b_status h2b_mtree_shape(const h2b_mtree* S, int32_t* brows, int32_t* bcols, int64_t* nblocks) {
  return guarded_call([&] {
    require(S, "null matrix tree");
    for (int l = 0; l <= S->q; ++l) {
      if (brows) brows[l] = S->cpl[l].br;
      if (bcols) bcols[l] = S->cpl[l].bc;
      if (nblocks) nblocks[l] = S->cpl[l].nb;
    }
  });
}

// The block values of every level, concatenated (BSRLayer::values per level).
h2b_status h2b_mtree_export(const h2b_mtree* S, double* values) {
  return guarded_call([&] {
    require(S && values, "null argument");
    Dev g(S->device);
    for (int l = 0; l <= S->q; ++l) {
      const Layer& L = S->cpl[l];
      download_blocks(L.val, values, L.br, L.bc, L.nb, S->stream);
      values += L.nb * L.br * L.bc;
    }
  });
}

// tree_multiply(S, xhat, yhat) (hmv.hpp:114-125): per level block_sparse_mv(L,
// x^l, y^l, 1, 0) in the reference's arithmetic; empty levels give y^l = 0.
// xhat: 2^l bcols[l] per level, yhat: 2^l brows[l] per level, concatenated.
h2b_status h2b_mtree_multiply(h2b_mtree* Sh, const double* xhat, double* yhat, h2b_ptr_kind kind) {
  return guarded_call([&] {
    require(Sh && xhat && yhat, "null argument");
    Matrix& S = *Sh;
    Dev g(S.device);
    cudaStream_t s = S.stream;
    (void)kind;
    const Matrix& C = S.col_basis();
    In xin(xhat, size_t(C.vec_off[S.q + 1]), s);
    Out yo(yhat, size_t(S.vec_off[S.q + 1]), false, s);
    for (int l = 0; l <= S.q; ++l) {
      const Layer& L = S.cpl[l];
      double* yl = yo.p + S.vec_off[l];
      const int64_t ny = S.vec_off[l + 1] - S.vec_off[l];
      if (L.nb == 0) {
        if (ny) H2B_CUDA(cudaMemsetAsync(yl, 0, ny * sizeof(double), s));
        continue;
      }
      launch_bsr_exact(L, xin.p + C.vec_off[l], yl, 1.0, 0.0, s);
    }
    yo.finish(s);
  });
}

// project_coupling(Trow, Tcol, S) (compression.hpp:130-169): S <- T_row S T_col^T
// per level, blocks resized to trow_rows[l] x tcol_rows[l].  Trees: level-
// concatenated, rows[l] x cols[l] per node; tcol == NULL: Tcol is Trow (the
// reference's symmetric call, project_coupling(T, T, S)).
h2b_status h2b_project_coupling(const double* trow, const int32_t* trow_rows, const int32_t* trow_cols,
                                const double* tcol, const int32_t* tcol_rows, const int32_t* tcol_cols,
                                h2b_mtree* Sh) {
  return guarded_call([&] {
    require(Sh && trow, "null argument");
    Matrix& S = *Sh;
    const int q = S.q;
    const std::vector<int> rr = tree_shape(trow_rows, q, "project_coupling"),
                           rc = tree_shape(trow_cols, q, "project_coupling");
    const bool same = tcol == nullptr || tcol == trow;
    const std::vector<int> cr = same ? rr : tree_shape(tcol_rows, q, "project_coupling"),
                           cc = same ? rc : tree_shape(tcol_cols, q, "project_coupling");
    Dev g(S.device);
    cudaStream_t s = S.stream;
    In Tr(trow, tree_size(q, rr, rc), s);
    In Tc(same ? nullptr : tcol, same ? 0 : tree_size(q, cr, cc), s);
    phase_project(S, Tr.p, rr, rc, same ? Tr.p : Tc.p, cr, cc, same, s);
    // node-vector layout follows the new block shapes
    S.rank = rr;
    for (int l = 0; l <= q; ++l) S.rank[l] = S.cpl[l].br;
    S.vec_off.assign(q + 2, 0);
    for (int l = 0; l <= q; ++l) S.vec_off[l + 1] = S.vec_off[l] + S.nodes(l) * S.rank[l];
    bool square = true;
    for (int l = 0; l <= q; ++l) square = square && S.cpl[l].br == S.cpl[l].bc;
    std::vector<int32_t> bc(q + 1);
    for (int l = 0; l <= q; ++l) bc[l] = S.cpl[l].bc;
    if (square) {
      S.symmetric = true;
      S.colb.reset();
    } else {
      allocate_col(S, bc.data());
    }
    ++S.layout_version;
    upload_structure(S);
    check_value_symmetry(S);
  });
}

// generate_weight_tree(B, S) (compression.hpp:213-256): r_out gets R (ranks[l]^2
// per node, level-concatenated; R^0 = 0).  B must be orthogonal.
h2b_status h2b_generate_weight_tree(h2b_basis* Bh, h2b_mtree* Sh, double* r_out) {
  return guarded_call([&] {
    require(Bh && Sh && r_out, "null argument");
    Matrix& B = *Bh;
    Matrix& S = *Sh;
    require(B.device == S.device, "generate_weight_tree: basis and matrix tree on different devices");
    Dev g(B.device);
    cudaStream_t s = B.stream;
    const size_t nr = tree_size(B.q, B.rank, B.rank);
    DevBuf<double> R;
    R.alloc(std::max<size_t>(1, nr));
    H2B_CUDA(cudaStreamSynchronize(S.stream));
    phase_weights(S, B, R.p, s);
    Out ro(r_out, nr, false, s);
    if (nr) H2B_CUDA(cudaMemcpyAsync(ro.p, R.p, nr * sizeof(double), cudaMemcpyDeviceToDevice, s));
    ro.finish(s);
  });
}

}  // extern "C"
