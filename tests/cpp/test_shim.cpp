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
  if (a.size() != b.size()) return 1e300;
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return den > 0 ? std::sqrt(num / den) : std::sqrt(num);  // (zero reference: absolute)
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

// The reference's phase API on its own component types, shim
// against reference, phase by phase on the same inputs.
std::vector<double> flatv(const LevelVectors<double>& v) {
  std::vector<double> f;
  for (const auto& p : v.pool) f.insert(f.end(), p.begin(), p.end());
  return f;
}
// per-node R^T R (level l, k x k blocks), concatenated
std::vector<double> gram(const std::vector<double>& pool, index_t nodes, int rows, int cols) {
  std::vector<double> g(size_t(nodes) * cols * cols, 0.0);
  for (index_t b = 0; b < nodes; ++b) {
    const double* R = pool.data() + size_t(b) * rows * cols;
    for (int j = 0; j < cols; ++j)
      for (int i = 0; i < cols; ++i) {
        double acc = 0;
        for (int s = 0; s < rows; ++s) acc += R[s + size_t(i) * rows] * R[s + size_t(j) * rows];
        g[size_t(b) * cols * cols + i + size_t(j) * cols] = acc;
      }
  }
  return g;
}

void component_phases_match_reference() {
  for (auto [dim, n, order, eps] : {std::tuple{2, 4096, 8, 1e-7}, std::tuple{3, 4096, 4, 1e-6}}) {
    H2Matrix<double> G = kernel_matrix(dim, n, order);
    H2Matrix<double> R = G;
    const int q = G.depth();
    const auto xc = rnd(n, 5);
    // upsweep / tree_multiply / downsweep (hmv.hpp:79-157)
    LevelVectors<double> xg, xr, yg, yr;
    xg.resize(G.row_basis);
    xr.resize(R.row_basis);
    h2kit_b200::upsweep(G.row_basis, xc.data(), n, xg);
    h2kit::upsweep(R.row_basis, xc.data(), n, xr);
    CHECK(rel(flatv(xg), flatv(xr)) <= 1e-13);
    yg.resize(G.row_basis);
    yr.resize(R.row_basis);
    h2kit_b200::tree_multiply(G.coupling, xr, yg);
    h2kit::tree_multiply(R.coupling, xr, yr);
    CHECK(flatv(yg) == flatv(yr));  // block_sparse_mv in the reference's exact arithmetic
    std::vector<double> ycg = rnd(n, 6), ycr = ycg;
    h2kit_b200::downsweep(G.row_basis, yg, ycg.data(), n);
    h2kit::downsweep(R.row_basis, yr, ycr.data(), n);
    CHECK(rel(ycg, ycr) <= 1e-13);
    CHECK(rel(flatv(yg), flatv(yr)) <= 1e-13);  // y^ updated in place like the reference
    // block_sparse_mv (bsr.hpp:79-82) with alpha / beta: bitwise
    std::vector<double> dg = rnd(n, 7), dr = dg;
    h2kit_b200::block_sparse_mv(G.dense, xc.data(), dg.data(), 2.0, 0.5);
    h2kit::block_sparse_mv(R.dense, xc.data(), dr.data(), 2.0, 0.5);
    CHECK(dg == dr);
    // orthogonalize_basis (compression.hpp:69-126)
    const ProjectionTree<double> Tg = h2kit_b200::orthogonalize_basis(G.row_basis);
    const ProjectionTree<double> Tr = h2kit::orthogonalize_basis(R.row_basis);
    CHECK(rel(flat(Tg), flat(Tr)) <= 1e-11);
    CHECK(Tg.rows == Tr.rows && Tg.cols == Tr.cols);
    CHECK(rel(G.row_basis.leaf_pool, R.row_basis.leaf_pool) <= 1e-11);
    // project_coupling (:130-169), square T
    h2kit_b200::project_coupling(Tg, Tg, G.coupling);
    h2kit::project_coupling(Tr, Tr, R.coupling);
    for (int l = 0; l <= q; ++l)
      if (!R.coupling.levels[l].empty()) CHECK(rel(G.coupling.levels[l].values, R.coupling.levels[l].values) <= 1e-11);
    // generate_weight_tree (:213-256): R^T R per node (the c6 Gram identity),
    // and R itself (both take diag(R) >= 0, linalg.hpp:100-113)
    const WeightTree<double> Wg = h2kit_b200::generate_weight_tree(G.row_basis, G.coupling);
    const WeightTree<double> Wr = h2kit::generate_weight_tree(R.row_basis, R.coupling);
    CHECK(Wg.dim == Wr.dim);
    for (int l = 1; l <= q; ++l) {
      const int k = Wr.dim[l];
      if (k == 0) continue;
      CHECK(rel(gram(Wg.pool[l], index_t(1) << l, k, k), gram(Wr.pool[l], index_t(1) << l, k, k)) <= 1e-11);
      CHECK(rel(Wg.pool[l], Wr.pool[l]) <= 1e-9);
    }
    // truncate_basis (:267-420): ranks identical, energies, and Tout up to the
    // singular vectors' signs (T^T T per node)
    ProjectionTree<double> Ug, Ur;
    const TruncationResult tg = h2kit_b200::truncate_basis(G.row_basis, Wg, eps, Ug);
    const TruncationResult tr = h2kit::truncate_basis(R.row_basis, Wr, eps, Ur);
    CHECK(tg.new_ranks == tr.new_ranks);
    CHECK(G.row_basis.ranks == R.row_basis.ranks);
    double eg = 0, er = 0;
    for (int l = 0; l <= q; ++l) {
      eg += tg.discarded_energy[l];
      er += tr.discarded_energy[l];
      CHECK(std::abs(tg.discarded_energy[l] - tr.discarded_energy[l]) <= 1e-9 * er + 1e-30);
    }
    CHECK(std::abs(eg - er) <= 1e-9 * er);
    CHECK(Ug.rows == Ur.rows && Ug.cols == Ur.cols);
    for (int l = 0; l <= q; ++l) {
      if (Ur.rows[l] == 0) continue;
      CHECK(rel(gram(Ug.pool[l], index_t(1) << l, Ur.rows[l], Ur.cols[l]),
                gram(Ur.pool[l], index_t(1) << l, Ur.rows[l], Ur.cols[l])) <= 1e-8);
    }
    // project with the rectangular T, then the compressed operators agree
    h2kit_b200::project_coupling(Ug, Ug, G.coupling);
    h2kit::project_coupling(Ur, Ur, R.coupling);
    for (int l = 0; l <= q; ++l) {
      CHECK(G.coupling.levels[l].brows == R.coupling.levels[l].brows);
      CHECK(G.coupling.levels[l].bcols == R.coupling.levels[l].bcols);
    }
    const auto x = rnd(n, 8);
    std::vector<double> y1(n), y2(n);
    h2kit::hmv(G, x.data(), y1.data());  // the refreshed host objects, on the CPU
    h2kit::hmv(R, x.data(), y2.data());
    CHECK(rel(y1, y2) <= 10 * eps);
  }
}

// A 1-level, 1x1-block tree (test_compression.cpp:126-147): T_row = 2,
// T_col = 3 turn S = 5 into 30; a rectangular projection grows the blocks.
void scalar_and_growing_projection() {
  BSRLayer<double> L;
  L.block_rows = L.block_cols = 1;
  L.brows = L.bcols = 1;
  L.row_ptr = {0, 1};
  L.col_idx = {0};
  L.values = {5.0};
  MatrixTree<double> S;
  S.levels.push_back(L);
  ProjectionTree<double> Tr, Tc;
  Tr.pool = {{2.0}};
  Tr.rows = {1};
  Tr.cols = {1};
  Tc.pool = {{3.0}};
  Tc.rows = {1};
  Tc.cols = {1};
  h2kit_b200::project_coupling(Tr, Tc, S);
  CHECK(S.levels[0].values.size() == 1 && std::abs(S.levels[0].values[0] - 30.0) <= 1e-15);
  ProjectionTree<double> G2;  // 2 x 1: the block grows to 2 x 2
  G2.pool = {{1.0, -1.0}};
  G2.rows = {2};
  G2.cols = {1};
  MatrixTree<double> S2 = S, S3 = S;
  h2kit_b200::project_coupling(G2, G2, S2);
  h2kit::project_coupling(G2, G2, S3);
  CHECK(S2.levels[0].brows == 2 && S2.levels[0].bcols == 2);
  CHECK(S2.levels[0].values == S3.levels[0].values);
}

// A host-side edit of an entry the default fingerprint does not sample:
// invalidate(A) (or H2KIT_B200_STRICT=1, checked by the Python runner) makes
// the next call see it.
void mutation_then_invalidate() {
  H2Matrix<double> A = kernel_matrix(2, 2048, 8);
  std::vector<double> x(A.n, 1.0), y0(A.n), y1(A.n), yr(A.n);
  h2kit_b200::hmv(A, x.data(), y0.data());
  auto& v = A.coupling.levels[A.depth()].values;
  v[v.size() / 2 + 3] += 1.0;  // off the sampling grid
  h2kit_b200::invalidate(A);
  h2kit_b200::hmv(A, x.data(), y1.data());
  h2kit::hmv(A, x.data(), yr.data());
  CHECK(rel(y1, yr) <= 1e-12);
  CHECK(rel(y1, y0) > 0.0);
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
  run("component phase API (BasisTree / MatrixTree / BSRLayer) matches the reference", component_phases_match_reference);
  run("scalar and growing projections", scalar_and_growing_projection);
  run("host-side mutation + invalidate is seen by the next call", mutation_then_invalidate);
  run("invalid arguments throw std::invalid_argument", errors_are_invalid_argument);
  std::printf("%d checks, %d failures\n", checks, failures);
  return failures ? 1 : 0;
}
