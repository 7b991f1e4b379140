// h2kit_b200_bind.hpp — the H2KIT_USE_B200 binding.
//
// Explicit specializations of the reference's hot-path function templates
// for T = double that forward to the B200 library (include/h2kit_b200.hpp ->
// libh2b.so).  A translation unit that sees this header before its first use
// of these templates runs them on the B200 with no other source change:
//
//   g++ ... -DH2KIT_USE_B200 -include h2kit_b200_bind.hpp  (or #include it first)
//
// Specialized (reference declarations):
//   hmv<double> x2              include/h2kit/hmv.hpp:175-188, 190-194
//   upsweep / tree_multiply / downsweep   hmv.hpp:79-157
//   block_sparse_mv<double>     bsr.hpp:79-82
//   compress<double>            compression.hpp:466-551
//   orthogonalize_basis / project_coupling / generate_weight_tree /
//   truncate_basis              compression.hpp:69-420
// Everything else (construction, I/O, validation, the serial:: engine) stays
// the reference's own code; validate_sampled / validate_dense call hmv and so
// run their mat-vecs on the device too.
#pragma once

#include "h2kit_b200.hpp"

namespace h2kit {

template <>
inline void hmv<double>(const H2Matrix<double>& A, const double* x, double* y, double alpha, double beta,
                        HmvContext<double>& ctx) {
  h2kit_b200::hmv(A, x, y, alpha, beta, ctx);
}

template <>
inline void hmv<double>(const H2Matrix<double>& A, const double* x, double* y, double alpha, double beta) {
  h2kit_b200::hmv(A, x, y, alpha, beta);
}

template <>
inline void upsweep<double>(const BasisTree<double>& V, const double* x, index_t n, LevelVectors<double>& xhat) {
  h2kit_b200::upsweep(V, x, n, xhat);
}

template <>
inline void tree_multiply<double>(const MatrixTree<double>& S, const LevelVectors<double>& xhat,
                                  LevelVectors<double>& yhat) {
  h2kit_b200::tree_multiply(S, xhat, yhat);
}

template <>
inline void downsweep<double>(const BasisTree<double>& U, LevelVectors<double>& yhat, double* y, index_t n) {
  h2kit_b200::downsweep(U, yhat, y, n);
}

template <>
inline void block_sparse_mv<double>(const BSRLayer<double>& L, const double* x, double* y, double alpha,
                                    double beta) {
  h2kit_b200::block_sparse_mv(L, x, y, alpha, beta);
}

template <>
inline CompressionReport compress<double>(H2Matrix<double>& A, double eps) {
  return h2kit_b200::compress(A, eps);
}

template <>
inline ProjectionTree<double> orthogonalize_basis<double>(BasisTree<double>& B) {
  return h2kit_b200::orthogonalize_basis(B);
}

template <>
inline void project_coupling<double>(const ProjectionTree<double>& Trow, const ProjectionTree<double>& Tcol,
                                     MatrixTree<double>& S) {
  h2kit_b200::project_coupling(Trow, Tcol, S);
}

template <>
inline WeightTree<double> generate_weight_tree<double>(const BasisTree<double>& B, const MatrixTree<double>& S) {
  return h2kit_b200::generate_weight_tree(B, S);
}

template <>
inline TruncationResult truncate_basis<double>(BasisTree<double>& B, const WeightTree<double>& R, double eps,
                                              ProjectionTree<double>& Tout) {
  return h2kit_b200::truncate_basis(B, R, eps, Tout);
}

}  // namespace h2kit
