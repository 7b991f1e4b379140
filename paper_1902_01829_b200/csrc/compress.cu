// Algebraic recompression on the device (compression.hpp:466-551).
#include "h2b_internal.hpp"

namespace h2b {

void compress_matrix(Matrix& A, double eps, h2b_compress_report* rep) {
  (void)A; (void)eps; (void)rep;
  throw Error(H2B_UNSUPPORTED, "compress: not implemented yet");
}

void orthogonalize_matrix(Matrix& A, double* t_out) {
  (void)A; (void)t_out;
  throw Error(H2B_UNSUPPORTED, "orthogonalize: not implemented yet");
}

}  // namespace h2b
