// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Thin C-ABI wrapper around the UNMODIFIED reference library (h2kit, compiled
// from /root/reference/proj/src/*.cpp by oracle/Makefile into
// oracle/_ref/libh2ref.so).  It lets the Python tests and bench.py's
// cpu_baseline / --impl reference arm drive the reference's own public API:
//   construct<double>()        /root/reference/proj/include/h2kit/construction.hpp:179-200
//   hmv()                      /root/reference/proj/include/h2kit/hmv.hpp:175-194
//   upsweep/tree_multiply/downsweep  hmv.hpp:79-157
//   compress()                 /root/reference/proj/include/h2kit/compression.hpp:466-551
//   orthogonalize_basis/project_coupling/generate_weight_tree/truncate_basis
//                              compression.hpp:69-420
//   memory_footprint()         /root/reference/proj/include/h2kit/h2_matrix.hpp:90-102
//   flops::counter()           /root/reference/proj/include/h2kit/flops.hpp:22-25
// Matrices cross the boundary in the flat "export" layout shared with the
// product C-ABI (include/h2b.h): perm, ranks, leaf pool, level-concatenated
// transfers, level-concatenated coupling CSR + values, dense CSR + values.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "h2kit/compression.hpp"
#include "h2kit/construction.hpp"
#include "h2kit/hmv.hpp"
#include "h2kit/io.hpp"
#include "h2kit/validate.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace h2kit;
using Mat = H2Matrix<double>;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int ref_max_threads() { return max_threads(); }

int ref_points(int dim, int n, double pert, uint64_t seed, double* out) {
  return guarded([&] {
    const PointSet ps = generate_perturbed_grid(dim, n, pert, seed);
    std::memcpy(out, ps.coords.data(), ps.coords.size() * sizeof(double));
  });
}

int ref_random_vector(int n, uint64_t seed, double* out) {
  return guarded([&] {
    const auto v = random_vector<double>(n, seed);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}

int ref_construct(int dim, int n, int leaf, int order, double eta, double ell,
                  double pert, uint64_t seed, void** out) {
  return guarded([&] {
    const PointSet ps = generate_perturbed_grid(dim, n, pert, seed);
    KernelSpec spec;
    spec.correlation_length = ell;
    ConstructionConfig cfg;
    cfg.leaf_size = leaf;
    cfg.grid_order = order;
    cfg.eta = eta;
    Mat* A = new Mat(construct<double>(ps, spec, cfg));
    A->info.dim = dim;
    A->info.seed = seed;
    A->info.perturbation = pert;
    A->info.ell = ell;
    A->info.eta = eta;
    A->info.grid_order = order;
    *out = A;
  });
}

void ref_destroy(void* h) { delete static_cast<Mat*>(h); }

void* ref_clone(void* h) { return new Mat(*static_cast<Mat*>(h)); }

// Shape query: out[0]=n, out[1]=m, out[2]=depth, out[3]=symmetric.
void ref_shape(void* h, int* out) {
  const Mat& A = *static_cast<Mat*>(h);
  out[0] = A.n;
  out[1] = A.m;
  out[2] = A.depth();
  out[3] = A.symmetric ? 1 : 0;
}

// ranks[depth+1], cpl_blocks[depth+1], cpl_brows/bcols[depth+1], dense blocks.
void ref_layout(void* h, int* ranks, int64_t* cpl_blocks, int* cpl_brows,
                int* cpl_bcols, int64_t* dense_blocks) {
  const Mat& A = *static_cast<Mat*>(h);
  const int q = A.depth();
  for (int l = 0; l <= q; ++l) {
    ranks[l] = A.row_basis.ranks[l];
    cpl_blocks[l] = A.coupling.levels[l].num_blocks();
    cpl_brows[l] = A.coupling.levels[l].brows;
    cpl_bcols[l] = A.coupling.levels[l].bcols;
  }
  *dense_blocks = A.dense.num_blocks();
}

void ref_export(void* h, int32_t* perm, double* leaf, double* transfer,
                int32_t* cpl_row_ptr, int32_t* cpl_col_idx, double* cpl_values,
                int32_t* dense_row_ptr, int32_t* dense_col_idx, double* dense_values) {
  const Mat& A = *static_cast<Mat*>(h);
  const int q = A.depth();
  std::memcpy(perm, A.perm.data(), A.perm.size() * sizeof(int32_t));
  std::memcpy(leaf, A.row_basis.leaf_pool.data(),
              A.row_basis.leaf_pool.size() * sizeof(double));
  for (int l = 1; l <= q; ++l) {
    const auto& t = A.row_basis.transfer[l];
    std::memcpy(transfer, t.data(), t.size() * sizeof(double));
    transfer += t.size();
  }
  for (int l = 0; l <= q; ++l) {
    const auto& L = A.coupling.levels[l];
    if (L.row_ptr.empty()) {
      for (int r = 0; r <= L.block_rows; ++r) *cpl_row_ptr++ = 0;
    } else {
      std::memcpy(cpl_row_ptr, L.row_ptr.data(), L.row_ptr.size() * sizeof(int32_t));
      cpl_row_ptr += L.row_ptr.size();
    }
    std::memcpy(cpl_col_idx, L.col_idx.data(), L.col_idx.size() * sizeof(int32_t));
    cpl_col_idx += L.col_idx.size();
    std::memcpy(cpl_values, L.values.data(), L.values.size() * sizeof(double));
    cpl_values += L.values.size();
  }
  std::memcpy(dense_row_ptr, A.dense.row_ptr.data(), A.dense.row_ptr.size() * sizeof(int32_t));
  std::memcpy(dense_col_idx, A.dense.col_idx.data(), A.dense.col_idx.size() * sizeof(int32_t));
  std::memcpy(dense_values, A.dense.values.data(), A.dense.values.size() * sizeof(double));
}

// Build a symmetric reference H2Matrix from the flat export layout.
int ref_import(int n, int m, int depth, const int32_t* ranks, const int32_t* perm,
               const double* leaf, const double* transfer, const int32_t* cpl_row_ptr,
               const int32_t* cpl_col_idx, const double* cpl_values,
               const int32_t* dense_row_ptr, const int32_t* dense_col_idx,
               const double* dense_values, void** out) {
  return guarded([&] {
    Mat* A = new Mat;
    A->n = n;
    A->m = m;
    A->symmetric = true;
    A->perm.assign(perm, perm + n);
    BasisTree<double>& B = A->row_basis;
    B.flat = make_complete_binary_tree(depth);
    B.leaf_dim = m;
    B.ranks.assign(ranks, ranks + depth + 1);
    const size_t nleaves = size_t(1) << depth;
    B.leaf_pool.assign(leaf, leaf + nleaves * m * ranks[depth]);
    B.transfer.assign(depth + 1, {});
    for (int l = 1; l <= depth; ++l) {
      const size_t sz = (size_t(1) << l) * ranks[l] * ranks[l - 1];
      B.transfer[l].assign(transfer, transfer + sz);
      transfer += sz;
    }
    A->coupling.levels.assign(depth + 1, {});
    for (int l = 0; l <= depth; ++l) {
      BSRLayer<double>& L = A->coupling.levels[l];
      L.block_rows = L.block_cols = index_t(1) << l;
      L.brows = L.bcols = ranks[l];
      L.row_ptr.assign(cpl_row_ptr, cpl_row_ptr + L.block_rows + 1);
      cpl_row_ptr += L.block_rows + 1;
      const size_t nb = L.row_ptr.back();
      L.col_idx.assign(cpl_col_idx, cpl_col_idx + nb);
      cpl_col_idx += nb;
      const size_t nv = nb * ranks[l] * ranks[l];
      L.values.assign(cpl_values, cpl_values + nv);
      cpl_values += nv;
    }
    BSRLayer<double>& D = A->dense;
    D.block_rows = D.block_cols = index_t(nleaves);
    D.brows = D.bcols = m;
    D.row_ptr.assign(dense_row_ptr, dense_row_ptr + nleaves + 1);
    const size_t nbd = D.row_ptr.back();
    D.col_idx.assign(dense_col_idx, dense_col_idx + nbd);
    D.values.assign(dense_values, dense_values + nbd * m * m);
    *out = A;
  });
}

// Non-symmetric variant: the column basis V / F (col_basis_store,
// h2_matrix.hpp:69) and coupling blocks of ranks[l] x col_ranks[l].
int ref_import_ns(int n, int m, int depth, const int32_t* ranks, const int32_t* col_ranks,
                  const int32_t* perm, const double* leaf, const double* transfer,
                  const double* col_leaf, const double* col_transfer, const int32_t* cpl_row_ptr,
                  const int32_t* cpl_col_idx, const double* cpl_values, const int32_t* dense_row_ptr,
                  const int32_t* dense_col_idx, const double* dense_values, void** out) {
  return guarded([&] {
    Mat* A = new Mat;
    A->n = n;
    A->m = m;
    A->symmetric = false;
    A->perm.assign(perm, perm + n);
    const size_t nleaves = size_t(1) << depth;
    auto basis = [&](BasisTree<double>& B, const int32_t* rk, const double* lf, const double* tr) {
      B.flat = make_complete_binary_tree(depth);
      B.leaf_dim = m;
      B.ranks.assign(rk, rk + depth + 1);
      B.leaf_pool.assign(lf, lf + nleaves * m * rk[depth]);
      B.transfer.assign(depth + 1, {});
      for (int l = 1; l <= depth; ++l) {
        const size_t sz = (size_t(1) << l) * rk[l] * rk[l - 1];
        B.transfer[l].assign(tr, tr + sz);
        tr += sz;
      }
    };
    basis(A->row_basis, ranks, leaf, transfer);
    A->col_basis_store.emplace();
    basis(*A->col_basis_store, col_ranks, col_leaf, col_transfer);
    A->coupling.levels.assign(depth + 1, {});
    for (int l = 0; l <= depth; ++l) {
      BSRLayer<double>& L = A->coupling.levels[l];
      L.block_rows = L.block_cols = index_t(1) << l;
      L.brows = ranks[l];
      L.bcols = col_ranks[l];
      L.row_ptr.assign(cpl_row_ptr, cpl_row_ptr + L.block_rows + 1);
      cpl_row_ptr += L.block_rows + 1;
      const size_t nb = L.row_ptr.back();
      L.col_idx.assign(cpl_col_idx, cpl_col_idx + nb);
      cpl_col_idx += nb;
      const size_t nv = nb * ranks[l] * col_ranks[l];
      L.values.assign(cpl_values, cpl_values + nv);
      cpl_values += nv;
    }
    BSRLayer<double>& D = A->dense;
    D.block_rows = D.block_cols = index_t(nleaves);
    D.brows = D.bcols = m;
    D.row_ptr.assign(dense_row_ptr, dense_row_ptr + nleaves + 1);
    const size_t nbd = D.row_ptr.back();
    D.col_idx.assign(dense_col_idx, dense_col_idx + nbd);
    D.values.assign(dense_values, dense_values + nbd * m * m);
    *out = A;
  });
}

// Column basis ranks (== row ranks when symmetric) and pools (non-symmetric).
void ref_col_ranks(void* h, int* out) {
  const Mat& A = *static_cast<Mat*>(h);
  for (int l = 0; l <= A.depth(); ++l) out[l] = A.col_basis().ranks[l];
}
void ref_export_col(void* h, double* col_leaf, double* col_transfer) {
  const Mat& A = *static_cast<Mat*>(h);
  const auto& B = A.col_basis();
  std::memcpy(col_leaf, B.leaf_pool.data(), B.leaf_pool.size() * sizeof(double));
  for (int l = 1; l <= A.depth(); ++l) {
    std::memcpy(col_transfer, B.transfer[l].data(), B.transfer[l].size() * sizeof(double));
    col_transfer += B.transfer[l].size();
  }
}

uint64_t ref_footprint(void* h) { return memory_footprint(*static_cast<Mat*>(h)).total(); }

void ref_flops_reset() { flops::reset(); }
double ref_flops_total() { return flops::counter().total(); }

int ref_hmv(void* h, const double* x, double* y, double alpha, double beta) {
  return guarded([&] { hmv(*static_cast<Mat*>(h), x, y, alpha, beta); });
}

// Repeated multiplies with one context (the CLI matvec loop, h2kit.cpp:111-113).
int ref_hmv_reps(void* h, const double* x, double* y, int reps) {
  return guarded([&] {
    const Mat& A = *static_cast<Mat*>(h);
    HmvContext<double> ctx(A);
    for (int r = 0; r < reps; ++r) hmv(A, x, y, 1.0, 0.0, ctx);
  });
}

// Phase-level oracle: x in cluster order -> xhat (level-concatenated),
// yhat = S xhat, and the downsweep of a given yhat added into yc.
int ref_upsweep(void* h, const double* xc, double* xhat_out) {
  return guarded([&] {
    const Mat& A = *static_cast<Mat*>(h);
    LevelVectors<double> xh;
    xh.resize(A.col_basis());
    upsweep(A.col_basis(), xc, A.n, xh);
    for (auto& p : xh.pool) {
      std::memcpy(xhat_out, p.data(), p.size() * sizeof(double));
      xhat_out += p.size();
    }
  });
}

int ref_tree_multiply(void* h, const double* xhat_in, double* yhat_out) {
  return guarded([&] {
    const Mat& A = *static_cast<Mat*>(h);
    LevelVectors<double> xh, yh;
    xh.resize(A.col_basis());
    yh.resize(A.row_basis);
    for (auto& p : xh.pool) {
      std::memcpy(p.data(), xhat_in, p.size() * sizeof(double));
      xhat_in += p.size();
    }
    tree_multiply(A.coupling, xh, yh);
    for (auto& p : yh.pool) {
      std::memcpy(yhat_out, p.data(), p.size() * sizeof(double));
      yhat_out += p.size();
    }
  });
}

int ref_downsweep(void* h, const double* yhat_in, double* yc_inout) {
  return guarded([&] {
    const Mat& A = *static_cast<Mat*>(h);
    LevelVectors<double> yh;
    yh.resize(A.row_basis);
    for (auto& p : yh.pool) {
      std::memcpy(p.data(), yhat_in, p.size() * sizeof(double));
      yhat_in += p.size();
    }
    downsweep(A.row_basis, yh, yc_inout, A.n);
  });
}

int ref_dense_mv(void* h, const double* xc, double* yc, double alpha, double beta) {
  return guarded([&] {
    block_sparse_mv(static_cast<Mat*>(h)->dense, xc, yc, alpha, beta);
  });
}

// report[0..] = frobenius_error, frobenius_norm, bytes_before, bytes_after,
// t_orth, t_proj1, t_weights, t_trunc, t_proj2 (ms),
// f_orth, f_proj1, f_weights, f_trunc, f_proj2 (model flops).
int ref_compress(void* h, double eps, double* report) {
  return guarded([&] {
    const CompressionReport r = compress(*static_cast<Mat*>(h), eps);
    const double v[] = {r.frobenius_error,       r.frobenius_norm,
                        double(r.bytes_before),  double(r.bytes_after),
                        r.time_orthogonalize_ms, r.time_project_orth_ms,
                        r.time_weights_ms,       r.time_truncate_ms,
                        r.time_project_trunc_ms, r.flops_orthogonalize,
                        r.flops_project_orth,    r.flops_weights,
                        r.flops_truncate,        r.flops_project_trunc};
    std::memcpy(report, v, sizeof(v));
  });
}

// Orthogonalize in place; writes the projection tree T (level-concatenated,
// k_l x k_l per node) to t_out.
int ref_orthogonalize(void* h, double* t_out) {
  return guarded([&] {
    Mat& A = *static_cast<Mat*>(h);
    const ProjectionTree<double> T = orthogonalize_basis(A.row_basis);
    for (auto& p : T.pool) {
      std::memcpy(t_out, p.data(), p.size() * sizeof(double));
      t_out += p.size();
    }
  });
}

// The same on the column basis (h2_matrix.hpp:75-78; the row basis itself
// when symmetric); T: col_ranks[l]^2 per node.
int ref_orthogonalize_col(void* h, double* t_out) {
  return guarded([&] {
    Mat& A = *static_cast<Mat*>(h);
    const ProjectionTree<double> T = orthogonalize_basis(A.col_basis());
    for (auto& p : T.pool) {
      std::memcpy(t_out, p.data(), p.size() * sizeof(double));
      t_out += p.size();
    }
  });
}

// Orthogonalize + project (in place), then the weight tree R (level-
// concatenated, k_l x k_l per node).
int ref_orth_project_weights(void* h, double* r_out) {
  return guarded([&] {
    Mat& A = *static_cast<Mat*>(h);
    const ProjectionTree<double> T = orthogonalize_basis(A.row_basis);
    project_coupling(T, T, A.coupling);
    const WeightTree<double> R = generate_weight_tree(A.row_basis, A.coupling);
    for (auto& p : R.pool) {
      std::memcpy(r_out, p.data(), p.size() * sizeof(double));
      r_out += p.size();
    }
  });
}

// Dense O(n^2) expansion in original order (test oracle, n <= 8192).
int ref_expand_dense(void* h, double* out) {
  return guarded([&] {
    const auto D = expand_to_dense(*static_cast<Mat*>(h));
    std::memcpy(out, D.data(), D.size() * sizeof(double));
  });
}

int ref_validate_sampled(void* h, double fraction, uint64_t seed, double* err) {
  return guarded([&] {
    const Mat& A = *static_cast<Mat*>(h);
    const PointSet ps =
        generate_perturbed_grid(A.info.dim, A.n, A.info.perturbation, A.info.seed);
    KernelSpec spec;
    spec.correlation_length = A.info.ell;
    *err = validate_sampled(A, ps, spec, fraction, seed);
  });
}

// h2kit::save / h2kit::load (io.hpp:183-282) and crc32 (crc32.cpp:6-20).
int ref_save(void* h, const char* path) {
  return guarded([&] { save(*static_cast<Mat*>(h), std::string(path)); });
}

int ref_load(const char* path, void** out) {
  return guarded([&] { *out = new Mat(load<double>(std::string(path))); });
}

uint32_t ref_crc32(const void* data, uint64_t len) { return crc32(data, size_t(len)); }

}  // extern "C"
