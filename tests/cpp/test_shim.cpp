// C++ parity suite for the drop-in shim include/h2kit_b200.hpp, written like
// the reference's own doctest suites (test_hmv.cpp, test_compression.cpp):
// the reference h2kit (compiled from /root/reference into oracle/_ref) is the
// oracle; every compute call under test goes through libh2b.so.
// Exit status 0 = all checks passed; prints one line per case.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "h2kit/compression.hpp"
#include "h2kit/construction.hpp"
#include "h2kit/validate.hpp"
#include "h2kit_b200.hpp"

using namespace h2kit;

namespace {
int failures = 0, checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++checks;                                                              \
    if (!(cond)) {                                                         \
      ++failures;                                                          \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                      \
  } while (0)

H2Matrix<double> kernel_matrix(int dim, index_t n, int order) {
  const PointSet ps = generate_perturbed_grid(dim, n, 0.25, 1);
  KernelSpec spec;
  spec.correlation_length = dim == 2 ? 0.1 : 0.2;
  ConstructionConfig cfg;
  cfg.grid_order = order;
  return construct<double>(ps, spec, cfg);
}

double rel(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num / den);
}

std::vector<double> rnd(index_t n, unsigned seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> d(0.0, 1.0);
  std::vector<double> v(n);
  for (auto& e : v) e = d(rng);
  return v;
}

void run(const char* name, void (*fn)()) {
  const int f0 = failures;
  fn();
  std::printf("[%s] %s\n", failures == f0 ? "PASS" : "FAIL", name);
}

void hmv_matches_reference() {
  for (auto [dim, n, order] : {std::tuple{2, 1024, 8}, std::tuple{2, 4096, 6}, std::tuple{3, 4096, 4}}) {
    const H2Matrix<double> A = kernel_matrix(dim, n, order);
    HmvContext<double> ctx(A);
    const auto x = rnd(n, 17);
    std::vector<double> y(n), yr(n);
    h2kit_b200::hmv(A, x.data(), y.data(), 1.0, 0.0, ctx);
    h2kit::hmv(A, x.data(), yr.data());
    CHECK(rel(y, yr) <= 1e-12);
  }
}

void alpha_beta() {  // test_hmv.cpp:91-101
  const index_t n = 256;
  const H2Matrix<double> A = kernel_matrix(2, n, 8);
  std::vector<double> x(n, 1.0), base(n, 0.0), y(n);
  h2kit_b200::hmv(A, x.data(), base.data());
  for (index_t i = 0; i < n; ++i) y[i] = double(i);
  h2kit_b200::hmv(A, x.data(), y.data(), 2.0, 3.0);
  for (index_t i = 0; i < n; ++i) CHECK(std::abs(y[i] - (2.0 * base[i] + 3.0 * i)) <= 1e-13 * std::abs(y[i]));
}

void phases_match_reference() {
  const index_t n = 4096;
  const H2Matrix<double> A = kernel_matrix(2, n, 8);
  const auto xc = rnd(n, 5);
  LevelVectors<double> xr, xg, yr, yg;
  xr.resize(A.row_basis);
  h2kit::upsweep(A.row_basis, xc.data(), n, xr);
  h2kit_b200::upsweep(A, xc.data(), xg);
  for (int l = 0; l <= A.depth(); ++l)
    if (!xr.pool[l].empty()) CHECK(rel(xg.pool[l], xr.pool[l]) <= 1e-12);
  yr.resize(A.row_basis);
  h2kit::tree_multiply(A.coupling, xr, yr);
  h2kit_b200::tree_multiply(A, xr, yg);
  for (int l = 0; l <= A.depth(); ++l)
    if (!yr.pool[l].empty() && A.coupling.levels[l].num_blocks()) CHECK(rel(yg.pool[l], yr.pool[l]) <= 1e-12);
  std::vector<double> ycr(xc), ycg(xc);
  h2kit::downsweep(A.row_basis, yr, ycr.data(), n);
  h2kit_b200::downsweep(A, yg, ycg.data());
  CHECK(rel(ycg, ycr) <= 1e-12);
}

void compress_matches_reference() {
  for (auto [dim, n, order, eps] : {std::tuple{2, 4096, 8, 1e-7}, std::tuple{3, 4096, 4, 1e-6}}) {
    H2Matrix<double> Ar = kernel_matrix(dim, n, order);
    H2Matrix<double> Ag = Ar;
    const auto x = rnd(n, 3);
    std::vector<double> y0(n), yr(n), yg(n), yg_cpu(n);
    h2kit::hmv(Ar, x.data(), y0.data());
    const CompressionReport rr = h2kit::compress(Ar, eps);
    const CompressionReport rg = h2kit_b200::compress(Ag, eps);
    for (size_t l = 0; l < rr.new_ranks.size(); ++l) CHECK(std::abs(rr.new_ranks[l] - rg.new_ranks[l]) <= 1);
    CHECK(rg.frobenius_error >= 0.5 * rr.frobenius_error && rg.frobenius_error <= 2.0 * rr.frobenius_error);
    CHECK(rg.bytes_after == memory_footprint(Ag).total());  // host object refreshed
    h2kit::hmv(Ar, x.data(), yr.data());
    h2kit_b200::hmv(Ag, x.data(), yg.data());
    h2kit::hmv(Ag, x.data(), yg_cpu.data());  // the refreshed host object, on the CPU
    CHECK(rel(yg, yr) <= 10 * eps);
    CHECK(rel(yg, y0) <= 10 * eps);
    CHECK(rel(yg_cpu, yg) <= 1e-12);
  }
}

void orthogonalize_orthonormal() {  // acceptance c3 (leaf V^T V = I)
  H2Matrix<double> A = kernel_matrix(2, 4096, 8);
  h2kit_b200::orthogonalize_basis(A);
  const int m = A.row_basis.leaf_dim, k = A.row_basis.ranks[A.depth()];
  double worst = 0;
  for (index_t i = 0; i < A.row_basis.flat.level_size(A.depth()); ++i) {
    const double* V = A.row_basis.leaf(i);
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) {
        double d = 0;
        for (int r = 0; r < m; ++r) d += V[r + a * m] * V[r + b * m];
        worst = std::max(worst, std::abs(d - (a == b ? 1.0 : 0.0)));
      }
  }
  CHECK(worst <= 1e-12);
}

// A non-symmetric matrix (col_basis_store, h2_matrix.hpp:69): V = U D with a
// positive diagonal D_l per level, F_c = D_l^-1 E_c D_{l-1}, S' = S D_l^-1 --
// the same operator, evaluated by the reference and through the shim.
H2Matrix<double> scaled_nonsym(const H2Matrix<double>& A) {
  H2Matrix<double> B = A;
  B.symmetric = false;
  B.col_basis_store = A.row_basis;
  BasisTree<double>& V = *B.col_basis_store;
  const int q = A.depth();
  std::vector<std::vector<double>> d(q + 1);
  for (int l = 0; l <= q; ++l)
    for (int j = 0; j < A.row_basis.ranks[l]; ++j) d[l].push_back(0.5 + 0.01 * ((7 * j + 3 * l) % 50));
  const int m = A.m, kq = A.row_basis.ranks[q];
  for (size_t i = 0; i < V.leaf_pool.size(); ++i) V.leaf_pool[i] *= d[q][(i / m) % kq];
  for (int l = 1; l <= q; ++l) {
    const int kc = A.row_basis.ranks[l], kp = A.row_basis.ranks[l - 1];
    for (size_t e = 0; e < V.transfer[l].size(); ++e) {
      const size_t i = e % kc, j = (e / kc) % kp;
      V.transfer[l][e] *= d[l - 1][j] / d[l][i];
    }
  }
  for (int l = 0; l <= q; ++l) {
    auto& L = B.coupling.levels[l];
    const int k = L.brows;
    for (size_t e = 0; e < L.values.size(); ++e) L.values[e] /= d[l][(e / k) % k];
  }
  return B;
}

void nonsymmetric_hmv() {
  H2Matrix<double> A = kernel_matrix(2, 4096, 4);
  H2Matrix<double> B = scaled_nonsym(A);
  const index_t n = A.n;
  std::vector<double> x(n), yr(n), yb(n), yg(n);
  for (index_t i = 0; i < n; ++i) x[i] = std::sin(0.37 * i) + 1.0;
  h2kit::hmv(A, x.data(), yr.data());
  h2kit::hmv(B, x.data(), yb.data());
  h2kit_b200::hmv(B, x.data(), yg.data());
  CHECK(rel(yb, yr) <= 1e-13);
  CHECK(rel(yg, yb) <= 1e-12);
  // compress through the shim: the host object (both bases) is refreshed and
  // matches the reference's own compress of the same matrix
  H2Matrix<double> Bref = B;
  const auto rr = h2kit::compress(Bref, 1e-7);
  const auto rg = h2kit_b200::compress(B, 1e-7);
  for (size_t l = 0; l < rr.new_ranks.size(); ++l) CHECK(rg.new_ranks[l] == rr.new_ranks[l]);
  for (size_t l = 0; l < rr.new_ranks.size(); ++l)
    CHECK(B.col_basis_store->ranks[l] == Bref.col_basis_store->ranks[l]);
  CHECK(rg.bytes_after == memory_footprint(B).total());
  std::vector<double> y1(n), y2(n);
  h2kit::hmv(B, x.data(), y1.data());      // the refreshed host object, on the CPU
  h2kit::hmv(Bref, x.data(), y2.data());
  CHECK(rel(y1, yr) <= 1e-6);
  CHECK(rel(y1, y2) <= 1e-6);
}

// orthogonalize_basis on each basis of a non-symmetric matrix (compression.hpp:
// 69-126): the shim's row / column entry points against the reference's.
std::vector<double> flat(const ProjectionTree<double>& T) {
  std::vector<double> v;
  for (const auto& p : T.pool) v.insert(v.end(), p.begin(), p.end());
  return v;
}
void nonsymmetric_orthogonalize() {
  H2Matrix<double> B = scaled_nonsym(kernel_matrix(2, 4096, 4));
  H2Matrix<double> R = B;
  const auto tr_row = flat(h2kit::orthogonalize_basis(R.row_basis));
  const auto tr_col = flat(h2kit::orthogonalize_basis(R.col_basis()));
  const auto tg_row = h2kit_b200::orthogonalize_basis(B);
  const auto tg_col = h2kit_b200::orthogonalize_col_basis(B);
  CHECK(rel(tg_row, tr_row) <= 1e-11);
  CHECK(rel(tg_col, tr_col) <= 1e-11);
  CHECK(rel(B.row_basis.leaf_pool, R.row_basis.leaf_pool) <= 1e-11);
  CHECK(rel(B.col_basis().leaf_pool, R.col_basis().leaf_pool) <= 1e-11);
  for (int l = 1; l <= B.depth(); ++l) {
    CHECK(rel(B.row_basis.transfer[l], R.row_basis.transfer[l]) <= 1e-11);
    CHECK(rel(B.col_basis().transfer[l], R.col_basis().transfer[l]) <= 1e-11);
  }
}

void errors_are_invalid_argument() {
  H2Matrix<double> A = kernel_matrix(2, 1024, 8);
  bool threw = false;
  try {
    h2kit_b200::compress(A, -1.0);
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()).find("eps must be non-negative") != std::string::npos;
  }
  CHECK(threw);
}
}  // namespace

int main() {
  if (h2b_device_count() == 0) {
    std::printf("no device\n");
    return 77;
  }
  run("hmv matches the reference", hmv_matches_reference);
  run("hmv alpha/beta semantics", alpha_beta);
  run("phases match the reference", phases_match_reference);
  run("compress matches the reference", compress_matches_reference);
  run("orthogonalize gives orthonormal leaves", orthogonalize_orthonormal);
  run("non-symmetric hmv and compress match the reference", nonsymmetric_hmv);
  run("non-symmetric orthogonalize (row and column bases) matches the reference", nonsymmetric_orthogonalize);
  run("invalid arguments throw std::invalid_argument", errors_are_invalid_argument);
  std::printf("%d checks, %d failures\n", checks, failures);
  return failures ? 1 : 0;
}
