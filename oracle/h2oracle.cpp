// ============================================================================
// TEST INFRASTRUCTURE ONLY — the CPU oracle for the H^2 hot path.
//
// This file is a from-scratch restatement (flat arrays, scalar loops, no
// OpenMP) of the reference h2kit algorithms the B200 path replaces.  It is
// compiled to oracle/liboracle.so and is loaded ONLY by tests/, by
// __graft_entry__.smoke() (as the checker) and by bench.py's cpu_baseline leg.
// The product library (paper_1902_01829_b200/libh2b.so) never links it.
//
// Parity pinning: tests/test_oracle.py checks every function here against
//   (1) the real reference compiled from /root/reference (oracle/_ref), and
//   (2) the committed golden vectors in tests/golden/ and the reference's own
//       known-answer tests (test_batch.cpp:152-161, 215-226; test_bsr.cpp:38-57;
//       test_compression.cpp:126-147; test_hmv.cpp:36-72).
// All floating-point expressions keep the reference's operation order so
// that, compiled with the reference's flags, results are bit-identical.
//
// Each routine cites the reference location (relative to
// /root/reference/proj/) whose behaviour it restates.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

void check(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}

// ----------------------------------------------------------------------------
// Analytic flop model (include/h2kit/flops.hpp:29-47).
struct Flops {
  double total = 0;
  void gemm(double cnt, int m, int n, int k) { total += 2.0 * m * n * k * cnt; }
  void gemv(double cnt, int m, int n) { total += 2.0 * m * n * cnt; }
  void qr(double cnt, int r, int c) { total += 2.0 * c * c * (r - c / 3.0) * cnt; }
  void svd(double cnt, int r, int c) {
    const int s = std::min(r, c);
    total += (2.0 * s * s * (std::max(r, c) - s / 3.0) + 60.0 * s * s * s) * cnt;
  }
  void spmv(double blocks, int br, int bc) { total += 2.0 * br * bc * blocks; }
};
thread_local Flops g_flops;

// ----------------------------------------------------------------------------
// Flat H^2 matrix (symmetric: one basis).  Level-local node i of level l has
// children 2i, 2i+1 (flat_tree.cpp:18-41).
struct Csr {
  int rows = 0, br = 0, bc = 0;  // block rows, block dims
  std::vector<int32_t> ptr, col;
  std::vector<double> val;
  int64_t nblocks() const { return ptr.empty() ? 0 : ptr.back(); }
  const double* blk(int64_t b) const { return val.data() + b * int64_t(br) * bc; }
  double* blk(int64_t b) { return val.data() + b * int64_t(br) * bc; }
};

struct OMat {
  int n = 0, m = 0, q = 0;
  std::vector<int32_t> perm;
  std::vector<int> rank;                 // per level
  std::vector<double> leaf;              // 2^q blocks of m x rank[q]
  std::vector<std::vector<double>> tr;   // tr[l]: 2^l blocks of rank[l] x rank[l-1]
  std::vector<Csr> cpl;                  // per level
  Csr dense;
  int64_t nodes(int l) const { return int64_t(1) << l; }
};

// ---------------------------------------------------------------- geometry
// generate_perturbed_grid (src/geometry.cpp:36-93).
std::vector<int64_t> grid_sides(int dim, int64_t n) {
  const int64_t side = std::llround(std::pow(double(n), 1.0 / dim));
  int64_t prod = 1;
  for (int a = 0; a < dim; ++a) prod *= side;
  if (prod == n) return std::vector<int64_t>(dim, side);
  check(n > 0 && (n & (n - 1)) == 0,
        "generate_perturbed_grid: n must be a perfect dim-th power or a power of two");
  int e = 0;
  while ((int64_t(1) << e) < n) ++e;
  std::vector<int64_t> s(dim);
  for (int a = 0; a < dim; ++a) s[a] = int64_t(1) << (e / dim + (a < e % dim ? 1 : 0));
  return s;
}

std::vector<double> make_points(int dim, int n, double pert, uint64_t seed) {
  check(dim == 2 || dim == 3, "generate_perturbed_grid: dim must be 2 or 3");
  check(n > 0, "generate_perturbed_grid: n must be positive");
  check(pert >= 0 && pert < 0.5, "generate_perturbed_grid: perturbation must be in [0, 0.5)");
  const auto sides = grid_sides(dim, n);
  double step[3] = {0, 0, 0};
  for (int a = 0; a < dim; ++a) step[a] = sides[a] > 1 ? 1.0 / double(sides[a] - 1) : 1.0;
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<double> jit(-1.0, 1.0);
  std::vector<double> pts(size_t(n) * dim);
  int64_t cnt[3] = {0, 0, 0};
  for (int64_t p = 0; p < n; ++p) {
    for (int a = 0; a < dim; ++a) {
      const double base = sides[a] > 1 ? double(cnt[a]) * step[a] : 0.5;
      const double v = base + pert * step[a] * jit(gen);
      pts[p * dim + a] = std::clamp(v, 0.0, 1.0);
    }
    for (int a = 0; a < dim; ++a) {  // first axis fastest
      if (++cnt[a] < sides[a]) break;
      cnt[a] = 0;
    }
  }
  return pts;
}

struct Box {
  double lo[3], hi[3];
};

double diam(const Box& b, int dim) {
  double s = 0;
  for (int a = 0; a < dim; ++a) {
    const double w = b.hi[a] - b.lo[a];
    s += w * w;
  }
  return std::sqrt(s);
}

double gap(const Box& x, const Box& y, int dim) {
  double s = 0;
  for (int a = 0; a < dim; ++a) {
    const double g = std::max({0.0, x.lo[a] - y.hi[a], y.lo[a] - x.hi[a]});
    s += g * g;
  }
  return std::sqrt(s);
}

// Cluster tree: DFS, split the widest axis at the exact median, ties by
// index (src/geometry.cpp:116-169).  boxes[l][i] = tight box of node (l,i).
struct Clusters {
  int q = 0;
  std::vector<int32_t> order;              // cluster position -> point id
  std::vector<std::vector<Box>> boxes;     // per level
};

Clusters cluster(const std::vector<double>& pts, int dim, int n, int leaf) {
  check(leaf > 0, "build_cluster_tree: leaf_size must be positive");
  const int64_t nl = n / leaf;
  check(nl * leaf == n, "build_cluster_tree: n must be leaf_size * 2^q");
  int q = 0;
  while ((int64_t(1) << q) < nl) ++q;
  check((int64_t(1) << q) == nl, "build_cluster_tree: n must be leaf_size * 2^q");
  Clusters C;
  C.q = q;
  C.order.resize(n);
  std::iota(C.order.begin(), C.order.end(), 0);
  C.boxes.resize(q + 1);
  for (int l = 0; l <= q; ++l) C.boxes[l].resize(size_t(1) << l);
  const double* X = pts.data();
  // explicit stack instead of recursion; visiting order does not affect the
  // result because subranges are disjoint, but keep pre-order anyway.
  struct Item { int l; int64_t i, s, e; };
  std::vector<Item> st{{0, 0, 0, n}};
  while (!st.empty()) {
    const Item it = st.back();
    st.pop_back();
    int32_t* ids = C.order.data() + it.s;
    const int64_t cnt = it.e - it.s;
    Box& b = C.boxes[it.l][it.i];
    for (int a = 0; a < dim; ++a) {
      b.lo[a] = 1e300;
      b.hi[a] = -1e300;
    }
    for (int a = dim; a < 3; ++a) b.lo[a] = b.hi[a] = 0;
    for (int64_t t = 0; t < cnt; ++t)
      for (int a = 0; a < dim; ++a) {
        const double c = X[int64_t(ids[t]) * dim + a];
        b.lo[a] = std::min(b.lo[a], c);
        b.hi[a] = std::max(b.hi[a], c);
      }
    if (it.l == q) continue;
    int ax = 0;
    double w = -1;
    for (int a = 0; a < dim; ++a)
      if (b.hi[a] - b.lo[a] > w) {
        w = b.hi[a] - b.lo[a];
        ax = a;
      }
    const int64_t half = cnt / 2;
    std::nth_element(ids, ids + half, ids + cnt, [=](int32_t u, int32_t v) {
      const double cu = X[int64_t(u) * dim + ax], cv = X[int64_t(v) * dim + ax];
      return cu < cv || (cu == cv && u < v);
    });
    st.push_back({it.l + 1, 2 * it.i + 1, it.s + half, it.e});
    st.push_back({it.l + 1, 2 * it.i, it.s, it.s + half});
  }
  return C;
}

// ---------------------------------------------------------------- Chebyshev
// src/chebyshev.cpp:21-98.
std::vector<double> cheb_pts(int order) {
  std::vector<double> t(order);
  for (int i = 0; i < order; ++i) t[i] = -std::cos(M_PI * (2.0 * i + 1.0) / (2.0 * order));
  if (order == 1) t[0] = 0.0;
  return t;
}

void widen(const Box& b, int a, double& lo, double& hi) {
  lo = b.lo[a];
  hi = b.hi[a];
  if (hi - lo < 1e-8) {
    const double mid = 0.5 * (lo + hi);
    lo = mid - 0.5 * 1e-8;
    hi = mid + 0.5 * 1e-8;
  }
}

// order^dim nodes, point-major, first axis fastest.
std::vector<double> cheb_nodes(const Box& b, int dim, int order) {
  const auto t = cheb_pts(order);
  double ax[3][64];
  for (int a = 0; a < dim; ++a) {
    double lo, hi;
    widen(b, a, lo, hi);
    for (int i = 0; i < order; ++i) ax[a][i] = 0.5 * (lo + hi) + 0.5 * (hi - lo) * t[i];
  }
  int k = 1;
  for (int a = 0; a < dim; ++a) k *= order;
  std::vector<double> out(size_t(k) * dim);
  int idx[3] = {0, 0, 0};
  for (int g = 0; g < k; ++g) {
    for (int a = 0; a < dim; ++a) out[size_t(g) * dim + a] = ax[a][idx[a]];
    for (int a = 0; a < dim; ++a) {
      if (++idx[a] < order) break;
      idx[a] = 0;
    }
  }
  return out;
}

void lagrange1(double lo, double hi, int order, double x, double* out) {
  const auto t = cheb_pts(order);
  const double xr = (2.0 * x - (lo + hi)) / (hi - lo);
  for (int j = 0; j < order; ++j)
    if (xr == t[j]) {
      for (int i = 0; i < order; ++i) out[i] = i == j ? 1.0 : 0.0;
      return;
    }
  double den = 0;
  double term[64];
  for (int j = 0; j < order; ++j) {
    double w = std::sin(M_PI * (2.0 * j + 1.0) / (2.0 * order));
    if (j % 2 == 0) w = -w;
    term[j] = w / (xr - t[j]);
    den += term[j];
  }
  for (int j = 0; j < order; ++j) out[j] = term[j] / den;
}

void lagrangeN(const Box& b, int dim, int order, const double* x, double* out) {
  double per[3][64];
  for (int a = 0; a < dim; ++a) {
    double lo, hi;
    widen(b, a, lo, hi);
    lagrange1(lo, hi, order, x[a], per[a]);
  }
  int k = 1;
  for (int a = 0; a < dim; ++a) k *= order;
  int idx[3] = {0, 0, 0};
  for (int g = 0; g < k; ++g) {
    double v = 1.0;
    for (int a = 0; a < dim; ++a) v *= per[a][idx[a]];
    out[g] = v;
    for (int a = 0; a < dim; ++a) {
      if (++idx[a] < order) break;
      idx[a] = 0;
    }
  }
}

double kern(const double* x, const double* y, int dim, double ell) {
  double d2 = 0;
  for (int a = 0; a < dim; ++a) {
    const double d = x[a] - y[a];
    d2 += d * d;
  }
  return std::exp(-std::sqrt(d2) / ell);  // include/h2kit/kernels.hpp:11-22
}

// ---------------------------------------------------------------- partition
// Dual traversal (src/construction.cpp:7-36): root pair never admissible,
// admissible if max(diam) <= eta * dist, dense at the leaf level.
struct Part {
  std::vector<std::vector<std::pair<int32_t, int32_t>>> far;
  std::vector<std::pair<int32_t, int32_t>> near;
};

void dual(const Clusters& C, int dim, double eta, int l, int32_t i, int32_t j, Part& P) {
  const Box& bi = C.boxes[l][i];
  const Box& bj = C.boxes[l][j];
  if (l != 0 && std::max(diam(bi, dim), diam(bj, dim)) <= eta * gap(bi, bj, dim)) {
    P.far[l].emplace_back(i, j);
    return;
  }
  if (l == C.q) {
    P.near.emplace_back(i, j);
    return;
  }
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) dual(C, dim, eta, l + 1, 2 * i + a, 2 * j + b, P);
}

Csr csr_of(std::vector<std::pair<int32_t, int32_t>> pr, int rows, int br, int bc) {
  std::sort(pr.begin(), pr.end());
  Csr L;
  L.rows = rows;
  L.br = br;
  L.bc = bc;
  L.ptr.assign(rows + 1, 0);
  L.col.resize(pr.size());
  for (size_t b = 0; b < pr.size(); ++b) {
    ++L.ptr[pr[b].first + 1];
    L.col[b] = pr[b].second;
  }
  for (int r = 0; r < rows; ++r) L.ptr[r + 1] += L.ptr[r];
  L.val.assign(pr.size() * size_t(br) * bc, 0.0);
  return L;
}

// ---------------------------------------------------------------- construct
// construct<double> (include/h2kit/construction.hpp:71-200).
OMat build(int dim, int n, int leaf, int order, double eta, double ell, double pert,
           uint64_t seed) {
  check(eta > 0, "dual_traversal_partition: eta must be positive");
  check(order >= 1 && order <= 64, "order out of range");
  const auto pts = make_points(dim, n, pert, seed);
  const Clusters C = cluster(pts, dim, n, leaf);
  const int q = C.q;
  int k = 1;
  for (int a = 0; a < dim; ++a) k *= order;
  OMat A;
  A.n = n;
  A.m = leaf;
  A.q = q;
  A.perm = C.order;
  A.rank.assign(q + 1, k);
  // leaf bases: Lagrange polynomials of the leaf box at its points
  const int64_t nleaf = A.nodes(q);
  A.leaf.assign(size_t(nleaf) * leaf * k, 0.0);
  std::vector<double> row(k);
  for (int64_t i = 0; i < nleaf; ++i) {
    double* U = A.leaf.data() + i * leaf * k;
    for (int p = 0; p < leaf; ++p) {
      const int32_t pid = C.order[i * leaf + p];
      lagrangeN(C.boxes[q][i], dim, order, &pts[size_t(pid) * dim], row.data());
      for (int a = 0; a < k; ++a) U[p + size_t(a) * leaf] = row[a];
    }
  }
  // transfers: parent Lagrange polynomials at the child's Chebyshev nodes
  A.tr.assign(q + 1, {});
  for (int l = 1; l <= q; ++l) {
    A.tr[l].assign(size_t(A.nodes(l)) * k * k, 0.0);
    for (int64_t c = 0; c < A.nodes(l); ++c) {
      const auto cn = cheb_nodes(C.boxes[l][c], dim, order);
      double* E = A.tr[l].data() + c * k * k;
      for (int ac = 0; ac < k; ++ac) {
        lagrangeN(C.boxes[l - 1][c / 2], dim, order, &cn[size_t(ac) * dim], row.data());
        for (int ap = 0; ap < k; ++ap) E[ac + size_t(ap) * k] = row[ap];
      }
    }
  }
  Part P;
  P.far.resize(q + 1);
  dual(C, dim, eta, 0, 0, 0, P);
  A.cpl.resize(q + 1);
  for (int l = 0; l <= q; ++l) {
    A.cpl[l] = csr_of(P.far[l], int(A.nodes(l)), k, k);
    Csr& L = A.cpl[l];
    for (int r = 0; r < L.rows; ++r)
      for (int32_t b = L.ptr[r]; b < L.ptr[r + 1]; ++b) {
        const auto gi = cheb_nodes(C.boxes[l][r], dim, order);
        const auto gj = cheb_nodes(C.boxes[l][L.col[b]], dim, order);
        double* S = L.blk(b);
        for (int c = 0; c < k; ++c)
          for (int a = 0; a < k; ++a)
            S[a + size_t(c) * k] = kern(&gi[size_t(a) * dim], &gj[size_t(c) * dim], dim, ell);
      }
  }
  A.dense = csr_of(P.near, int(nleaf), leaf, leaf);
  Csr& D = A.dense;
  for (int r = 0; r < D.rows; ++r)
    for (int32_t b = D.ptr[r]; b < D.ptr[r + 1]; ++b) {
      double* blk = D.blk(b);
      const int32_t cb = D.col[b];
      for (int c = 0; c < leaf; ++c) {
        const int32_t pj = C.order[int64_t(cb) * leaf + c];
        for (int a = 0; a < leaf; ++a) {
          const int32_t pi = C.order[int64_t(r) * leaf + a];
          blk[a + size_t(c) * leaf] = kern(&pts[size_t(pi) * dim], &pts[size_t(pj) * dim], dim, ell);
        }
      }
    }
  return A;
}

// ---------------------------------------------------------------- small dense kernels
// Column-major; semantics of include/h2kit/linalg.hpp:18-46 (beta == 0 never reads C).
void mm(int m, int n, int k, const double* A, int lda, bool ta, const double* B, int ldb,
        bool tb, double* C, int ldc) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) {
      double s = 0;
      for (int p = 0; p < k; ++p)
        s += (ta ? A[p + size_t(i) * lda] : A[i + size_t(p) * lda]) *
             (tb ? B[j + size_t(p) * ldb] : B[p + size_t(j) * ldb]);
      C[i + size_t(j) * ldc] = 1.0 * s + 0.0;  // alpha = 1, beta = 0 at every call site
    }
}

// y = op(A) x (+ y when acc): linalg.hpp:35-46.
void mv(int m, int n, const double* A, int lda, bool ta, const double* x, double* y, bool acc) {
  const int ny = ta ? n : m, nk = ta ? m : n;
  for (int i = 0; i < ny; ++i) {
    double s = 0;
    for (int p = 0; p < nk; ++p) s += (ta ? A[p + size_t(i) * lda] : A[i + size_t(p) * lda]) * x[p];
    y[i] = 1.0 * s + (acc ? 1.0 * y[i] : 0.0);
  }
}

// Householder QR in place with beta = -sign(alpha)||x|| (linalg.hpp:48-75).
void house(int r, int c, double* A, int lda, double* tau) {
  for (int j = 0; j < c; ++j) {
    double* v = A + size_t(j) * lda;
    double nx = 0;
    for (int i = j; i < r; ++i) nx += v[i] * v[i];
    nx = std::sqrt(nx);
    if (nx == 0.0) {
      tau[j] = 0;
      continue;
    }
    const double al = v[j];
    const double be = al >= 0.0 ? -nx : nx;
    tau[j] = (be - al) / be;
    const double sc = 1.0 / (al - be);
    for (int i = j + 1; i < r; ++i) v[i] *= sc;
    v[j] = be;
    for (int kk = j + 1; kk < c; ++kk) {
      double* w = A + size_t(kk) * lda;
      double d = w[j];
      for (int i = j + 1; i < r; ++i) d += v[i] * w[i];
      d *= tau[j];
      w[j] -= d;
      for (int i = j + 1; i < r; ++i) w[i] -= v[i] * d;
    }
  }
}

// R with non-negative diagonal; flips[] marks negated rows (linalg.hpp:100-113).
void take_r(int c, const double* A, int lda, double* R, int ldr, std::vector<char>& flips) {
  flips.assign(c, 0);
  for (int j = 0; j < c; ++j) flips[j] = A[j + size_t(j) * lda] < 0.0;
  for (int j = 0; j < c; ++j)
    for (int i = 0; i < c; ++i) {
      const double v = i <= j ? A[i + size_t(j) * lda] : 0.0;
      R[i + size_t(j) * ldr] = flips[i] ? -v : v;
    }
}

// Thin QR: Q overwrites A (linalg.hpp:77-131).
void qr_thin(int r, int c, double* A, int lda, double* R, int ldr) {
  std::vector<double> tau(c), Q(size_t(r) * c);
  std::vector<char> fl;
  house(r, c, A, lda, tau.data());
  for (int j = 0; j < c; ++j) {
    std::fill(Q.begin() + size_t(j) * r, Q.begin() + size_t(j + 1) * r, 0.0);
    Q[j + size_t(j) * r] = 1.0;
  }
  for (int j = c - 1; j >= 0; --j) {
    if (tau[j] == 0.0) continue;
    const double* v = A + size_t(j) * lda;
    for (int kk = j; kk < c; ++kk) {
      double* w = Q.data() + size_t(kk) * r;
      double d = w[j];
      for (int i = j + 1; i < r; ++i) d += v[i] * w[i];
      d *= tau[j];
      w[j] -= d;
      for (int i = j + 1; i < r; ++i) w[i] -= v[i] * d;
    }
  }
  take_r(c, A, lda, R, ldr, fl);
  for (int j = 0; j < c; ++j) {
    const double s = fl[j] ? -1.0 : 1.0;
    for (int i = 0; i < r; ++i) A[i + size_t(j) * lda] = s * Q[i + size_t(j) * r];
  }
}

void qr_r(int r, int c, double* A, int lda, double* R, int ldr) {
  std::vector<double> tau(c);
  std::vector<char> fl;
  house(r, c, A, lda, tau.data());
  take_r(c, A, lda, R, ldr, fl);
}

// Cyclic one-sided Jacobi (linalg.hpp:142-176).
void jacobi(int r, int c, double* G, int ldg) {
  const double tol = std::numeric_limits<double>::epsilon() * 16.0;
  for (int sw = 0; sw < 60; ++sw) {
    bool any = false;
    for (int p = 0; p + 1 < c; ++p)
      for (int qq = p + 1; qq < c; ++qq) {
        double* gp = G + size_t(p) * ldg;
        double* gq = G + size_t(qq) * ldg;
        double a = 0, b = 0, d = 0;
        for (int i = 0; i < r; ++i) {
          a += gp[i] * gp[i];
          b += gq[i] * gq[i];
          d += gp[i] * gq[i];
        }
        if (std::abs(d) <= tol * std::sqrt(a * b) || d == 0.0) continue;
        any = true;
        const double z = (b - a) / (2.0 * d);
        const double t = (z >= 0.0 ? 1.0 : -1.0) / (std::abs(z) + std::sqrt(1.0 + z * z));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = cs * t;
        for (int i = 0; i < r; ++i) {
          const double u = gp[i], w = gq[i];
          gp[i] = cs * u - sn * w;
          gq[i] = sn * u + cs * w;
        }
      }
    if (!any) break;
  }
}

// Left singular vectors + sigmas, any shape (linalg.hpp:178-232).
void svd_left(int r, int c, const double* A, int lda, double* U, int ldu, double* sig) {
  const int s = std::min(r, c);
  std::vector<double> G;
  int gr, gc;
  if (r >= c) {
    gr = r;
    gc = c;
    G.resize(size_t(r) * c);
    for (int j = 0; j < c; ++j)
      std::copy(A + size_t(j) * lda, A + size_t(j) * lda + r, G.begin() + size_t(j) * r);
  } else {
    std::vector<double> At(size_t(c) * r), R(size_t(r) * r);
    for (int j = 0; j < r; ++j)
      for (int i = 0; i < c; ++i) At[i + size_t(j) * c] = A[j + size_t(i) * lda];
    qr_r(c, r, At.data(), c, R.data(), r);
    gr = gc = r;
    G.resize(size_t(r) * r);
    for (int j = 0; j < r; ++j)
      for (int i = 0; i < r; ++i) G[i + size_t(j) * r] = R[j + size_t(i) * r];
  }
  jacobi(gr, gc, G.data(), gr);
  std::vector<double> nrm(gc);
  for (int j = 0; j < gc; ++j) {
    double t = 0;
    for (int i = 0; i < gr; ++i) t += G[i + size_t(j) * gr] * G[i + size_t(j) * gr];
    nrm[j] = std::sqrt(t);
  }
  std::vector<int> ord(gc);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return nrm[a] > nrm[b]; });
  for (int j = 0; j < s; ++j) {
    const int src = ord[j];
    sig[j] = nrm[src];
    double* u = U + size_t(j) * ldu;
    const double* g = G.data() + size_t(src) * gr;
    if (nrm[src] > 0.0) {
      const double inv = 1.0 / nrm[src];
      for (int i = 0; i < gr; ++i) u[i] = g[i] * inv;
    } else {
      std::fill(u, u + gr, 0.0);
    }
  }
}

// Batched truncated SVD over contiguous entries (batch.hpp:107-140): the
// leading s columns of each W_i become left singular vectors.
void svd_batch(int64_t cnt, int r, int c, double* W, int64_t stride, double eps,
               std::vector<int>& ranks, std::vector<double>& sig) {
  check(eps >= 0.0, "svd_truncated_batched: eps must be non-negative");
  const int s = std::min(r, c);
  ranks.assign(cnt, 0);
  sig.assign(size_t(cnt) * s, 0.0);
  g_flops.svd(double(cnt), r, c);
  for (int64_t i = 0; i < cnt; ++i)
    for (int64_t e = 0; e < int64_t(r) * c; ++e)
      if (!std::isfinite(W[i * stride + e]))
        throw std::invalid_argument("svd_truncated_batched: non-finite input");
  std::vector<double> U(size_t(r) * s);
  for (int64_t i = 0; i < cnt; ++i) {
    double* w = W + i * stride;
    double* sg = sig.data() + i * s;
    svd_left(r, c, w, r, U.data(), r, sg);
    int rk = 0;
    for (int j = 0; j < s; ++j)
      if (sg[0] > 0.0 && sg[j] >= eps * sg[0]) ++rk;
    ranks[i] = rk;
    for (int j = 0; j < s; ++j) std::copy(U.begin() + size_t(j) * r, U.begin() + size_t(j + 1) * r, w + size_t(j) * r);
  }
}

// ---------------------------------------------------------------- HMV
// include/h2kit/bsr.hpp:50-82: y_r = beta*y_r (beta==0 -> 0), then blocks in
// col order, columns in order: y += col * (alpha * x_j).
void bsr_mv(const Csr& L, const double* x, double* y, double alpha, double beta) {
  g_flops.spmv(double(L.nblocks()), L.br, L.bc);
  for (int r = 0; r < L.rows; ++r) {
    double* yr = y + size_t(r) * L.br;
    for (int i = 0; i < L.br; ++i) yr[i] = beta == 0.0 ? 0.0 : beta * yr[i];
    for (int32_t b = L.ptr[r]; b < L.ptr[r + 1]; ++b) {
      const double* S = L.blk(b);
      const double* xc = x + size_t(L.col[b]) * L.bc;
      for (int j = 0; j < L.bc; ++j) {
        const double xv = alpha * xc[j];
        for (int i = 0; i < L.br; ++i) yr[i] += S[i + size_t(j) * L.br] * xv;
      }
    }
  }
}

// level-concatenated node vectors: offset of level l
std::vector<int64_t> vec_offsets(const OMat& A) {
  std::vector<int64_t> off(A.q + 2, 0);
  for (int l = 0; l <= A.q; ++l) off[l + 1] = off[l] + A.nodes(l) * A.rank[l];
  return off;
}

// hmv.hpp:79-111
void upsweep(const OMat& A, const double* xc, double* xh) {
  const auto off = vec_offsets(A);
  const int q = A.q, m = A.m, kq = A.rank[q];
  check(A.nodes(q) * m == A.n, "upsweep: dim mismatch");
  g_flops.gemv(double(A.nodes(q)), m, kq);
  for (int64_t i = 0; i < A.nodes(q); ++i)
    mv(m, kq, A.leaf.data() + i * m * kq, m, true, xc + i * m, xh + off[q] + i * kq, false);
  for (int l = q; l >= 1; --l) {
    const int kc = A.rank[l], kp = A.rank[l - 1];
    for (int slot = 0; slot < 2; ++slot) {
      g_flops.gemv(double(A.nodes(l - 1)), kc, kp);
      for (int64_t p = 0; p < A.nodes(l - 1); ++p) {
        const int64_t c = 2 * p + slot;
        mv(kc, kp, A.tr[l].data() + c * kc * kp, kc, true, xh + off[l] + c * kc,
           xh + off[l - 1] + p * kp, slot == 1);
      }
    }
  }
}

// hmv.hpp:114-125
void tree_mult(const OMat& A, const double* xh, double* yh) {
  const auto off = vec_offsets(A);
  for (int l = 0; l <= A.q; ++l) {
    if (A.cpl[l].nblocks() == 0) {
      std::fill(yh + off[l], yh + off[l + 1], 0.0);
      continue;
    }
    bsr_mv(A.cpl[l], xh + off[l], yh + off[l], 1.0, 0.0);
  }
}

// hmv.hpp:129-157
void downsweep(const OMat& A, double* yh, double* yc) {
  const auto off = vec_offsets(A);
  const int q = A.q, m = A.m, kq = A.rank[q];
  check(A.nodes(q) * m == A.n, "downsweep: dim mismatch");
  for (int l = 1; l <= q; ++l) {
    const int kc = A.rank[l], kp = A.rank[l - 1];
    g_flops.gemv(double(A.nodes(l)), kc, kp);
    for (int64_t c = 0; c < A.nodes(l); ++c)
      mv(kc, kp, A.tr[l].data() + c * kc * kp, kc, false, yh + off[l - 1] + (c / 2) * kp,
         yh + off[l] + c * kc, true);
  }
  g_flops.gemv(double(A.nodes(q)), m, kq);
  for (int64_t i = 0; i < A.nodes(q); ++i)
    mv(m, kq, A.leaf.data() + i * m * kq, m, false, yh + off[q] + i * kq, yc + i * m, true);
}

// hmv.hpp:175-188
void hmv(const OMat& A, const double* x, double* y, double alpha, double beta) {
  const auto off = vec_offsets(A);
  std::vector<double> xc(A.n), yc(A.n), xh(off.back()), yh(off.back());
  for (int t = 0; t < A.n; ++t) xc[t] = x[A.perm[t]];
  bsr_mv(A.dense, xc.data(), yc.data(), 1.0, 0.0);
  upsweep(A, xc.data(), xh.data());
  tree_mult(A, xh.data(), yh.data());
  downsweep(A, yh.data(), yc.data());
  for (int t = 0; t < A.n; ++t) {
    double& o = y[A.perm[t]];
    o = alpha * yc[t] + (beta == 0.0 ? 0.0 : beta * o);
  }
}

// ---------------------------------------------------------------- compression
// Projection tree: per level, rows[l] x cols[l] per node.
struct Proj {
  std::vector<std::vector<double>> T;
  std::vector<int> rows, cols;
};

// orthogonalize_basis (compression.hpp:69-126)
Proj orthogonalize(OMat& A) {
  const int q = A.q, m = A.m, kq = A.rank[q];
  Proj P;
  P.rows = P.cols = A.rank;
  P.T.resize(q + 1);
  for (int l = 0; l <= q; ++l) P.T[l].assign(size_t(A.nodes(l)) * A.rank[l] * A.rank[l], 0.0);
  check(m >= kq, "orthogonalize_basis: leaf_dim must be >= leaf rank");
  g_flops.qr(double(A.nodes(q)), m, kq);
  for (int64_t i = 0; i < A.nodes(q); ++i)
    qr_thin(m, kq, A.leaf.data() + i * m * kq, m, P.T[q].data() + i * kq * kq, kq);
  for (int l = q; l >= 1; --l) {
    const int kc = A.rank[l], kp = A.rank[l - 1];
    const int64_t np = A.nodes(l - 1);
    std::vector<double> Z(size_t(np) * 2 * kc * kp, 0.0);
    g_flops.gemm(double(A.nodes(l)), kc, kp, kc);
    for (int64_t c = 0; c < A.nodes(l); ++c)
      mm(kc, kp, kc, P.T[l].data() + c * kc * kc, kc, false, A.tr[l].data() + c * kc * kp, kc,
         false, Z.data() + (c / 2) * 2 * kc * kp + (c % 2) * kc, 2 * kc);
    check(2 * kc >= kp, "qr_batched: requires rows >= cols");
    g_flops.qr(double(np), 2 * kc, kp);
    for (int64_t p = 0; p < np; ++p)
      qr_thin(2 * kc, kp, Z.data() + p * 2 * kc * kp, 2 * kc, P.T[l - 1].data() + p * kp * kp, kp);
    for (int64_t c = 0; c < A.nodes(l); ++c) {
      const double* src = Z.data() + (c / 2) * 2 * kc * kp + (c % 2) * kc;
      double* dst = A.tr[l].data() + c * kc * kp;
      for (int j = 0; j < kp; ++j)
        for (int i = 0; i < kc; ++i) dst[i + size_t(j) * kc] = src[i + size_t(j) * 2 * kc];
    }
  }
  return P;
}

// project_coupling (compression.hpp:130-169), symmetric: Trow == Tcol.
void project(const Proj& P, OMat& A) {
  for (int l = 0; l <= A.q; ++l) {
    Csr& L = A.cpl[l];
    if (L.nblocks() == 0) {
      L.br = P.rows[l];
      L.bc = P.rows[l];
      continue;
    }
    check(P.cols[l] == L.br && P.cols[l] == L.bc, "project_coupling: dim mismatch");
    const int rn = P.rows[l], cn = P.rows[l], ro = L.br, co = L.bc;
    const int64_t nb = L.nblocks();
    std::vector<double> ts(size_t(nb) * rn * co), out(size_t(nb) * rn * cn);
    g_flops.gemm(double(nb), rn, co, ro);
    g_flops.gemm(double(nb), rn, cn, co);
    for (int r = 0; r < L.rows; ++r)
      for (int32_t b = L.ptr[r]; b < L.ptr[r + 1]; ++b) {
        double* t = ts.data() + int64_t(b) * rn * co;
        mm(rn, co, ro, P.T[l].data() + int64_t(r) * rn * ro, rn, false, L.blk(b), ro, false, t, rn);
        mm(rn, cn, co, t, rn, false, P.T[l].data() + int64_t(L.col[b]) * cn * co, cn, true,
           out.data() + int64_t(b) * rn * cn, rn);
      }
    L.val = std::move(out);
    L.br = rn;
    L.bc = cn;
  }
}

// generate_weight_tree (compression.hpp:184-256): stack padded to
// ld = k_p + b_max * k_c rows, R-only QR.
std::vector<std::vector<double>> weights(const OMat& A) {
  const int q = A.q;
  std::vector<std::vector<double>> R(q + 1);
  R[0].assign(size_t(A.rank[0]) * A.rank[0], 0.0);
  for (int l = 1; l <= q; ++l) {
    const int kc = A.rank[l], kp = A.rank[l - 1];
    const int64_t nl = A.nodes(l);
    R[l].assign(size_t(nl) * kc * kc, 0.0);
    const Csr& L = A.cpl[l];
    int bmax = 0;
    for (int r = 0; r < L.rows; ++r) bmax = std::max(bmax, L.ptr[r + 1] - L.ptr[r]);
    const int ld = kp + bmax * kc;
    std::vector<double> st(size_t(nl) * ld * kc, 0.0);
    g_flops.gemm(double(nl), kp, kc, kp);
    for (int64_t r = 0; r < nl; ++r)
      mm(kp, kc, kp, R[l - 1].data() + (r / 2) * kp * kp, kp, false, A.tr[l].data() + r * kc * kp,
         kc, true, st.data() + r * ld * kc, ld);
    for (int64_t r = 0; r < nl; ++r)
      for (int32_t b = L.ptr[r]; b < L.ptr[r + 1]; ++b) {
        const double* S = L.blk(b);
        double* d = st.data() + r * ld * kc + kp + int64_t(b - L.ptr[r]) * kc;
        for (int j = 0; j < kc; ++j)
          for (int i = 0; i < kc; ++i) d[j + size_t(i) * ld] = S[i + size_t(j) * kc];
      }
    check(ld >= kc, "qr_r_only_batched: requires rows >= cols");
    g_flops.qr(double(nl), ld, kc);
    for (int64_t r = 0; r < nl; ++r) qr_r(ld, kc, st.data() + r * ld * kc, ld, R[l].data() + r * kc * kc, kc);
  }
  return R;
}

// truncate_basis (compression.hpp:267-420).  Returns discarded energy.
double truncate(OMat& A, const std::vector<std::vector<double>>& R, double eps, Proj& Pt) {
  check(eps >= 0.0, "truncate_basis: eps must be non-negative");
  const int q = A.q, m = A.m;
  const std::vector<int> old = A.rank;
  std::vector<int> nr(q + 1, 0);
  std::vector<double> lev_e(q + 1, 0.0);  // TruncationResult::discarded_energy
  Pt.T.assign(q + 1, {});
  Pt.rows.assign(q + 1, 0);
  Pt.cols = old;
  std::vector<int> rk;
  std::vector<double> sg;
  {
    const int kq = old[q];
    const int64_t nlf = A.nodes(q);
    std::vector<double> W(size_t(nlf) * m * kq);
    g_flops.gemm(double(nlf), m, kq, kq);
    for (int64_t i = 0; i < nlf; ++i)
      mm(m, kq, kq, A.leaf.data() + i * m * kq, m, false, R[q].data() + i * kq * kq, kq, true,
         W.data() + i * m * kq, m);
    svd_batch(nlf, m, kq, W.data(), int64_t(m) * kq, eps, rk, sg);
    const int s = std::min(m, kq);
    const int kt = std::min(*std::max_element(rk.begin(), rk.end()), s);
    nr[q] = kt;
    for (int64_t i = 0; i < nlf; ++i)
      for (int j = kt; j < s; ++j) lev_e[q] += sg[size_t(i) * s + j] * sg[size_t(i) * s + j];
    Pt.rows[q] = kt;
    Pt.T[q].assign(size_t(nlf) * kt * kq, 0.0);
    g_flops.gemm(double(nlf), kt, kq, m);
    for (int64_t i = 0; i < nlf; ++i)
      mm(kt, kq, m, W.data() + i * m * kq, m, true, A.leaf.data() + i * m * kq, m, false,
         Pt.T[q].data() + i * kt * kq, kt);
    std::vector<double> nl(size_t(nlf) * m * kt);
    for (int64_t i = 0; i < nlf; ++i)
      std::copy(W.begin() + i * m * kq, W.begin() + i * m * kq + int64_t(m) * kt, nl.begin() + i * m * kt);
    A.leaf = std::move(nl);
  }
  for (int l = q; l >= 1; --l) {
    const int kt_c = nr[l], kc = old[l], kp = old[l - 1];
    const int64_t np = A.nodes(l - 1);
    const int zr = 2 * kt_c;
    std::vector<double> Z(size_t(np) * zr * kp, 0.0);
    g_flops.gemm(double(A.nodes(l)), kt_c, kp, kc);
    for (int64_t c = 0; c < A.nodes(l); ++c)
      mm(kt_c, kp, kc, Pt.T[l].data() + c * kt_c * kc, kt_c, false, A.tr[l].data() + c * kc * kp, kc,
         false, Z.data() + (c / 2) * zr * kp + (c % 2) * kt_c, zr);
    std::vector<double> W(size_t(np) * zr * kp, 0.0);
    g_flops.gemm(double(np), zr, kp, kp);
    for (int64_t p = 0; p < np; ++p)
      mm(zr, kp, kp, Z.data() + p * zr * kp, zr, false, R[l - 1].data() + p * kp * kp, kp, true,
         W.data() + p * zr * kp, zr);
    svd_batch(np, zr, kp, W.data(), int64_t(zr) * kp, eps, rk, sg);
    const int s = std::min(zr, kp);
    const int kt_p = std::min(*std::max_element(rk.begin(), rk.end()), s);
    nr[l - 1] = kt_p;
    for (int64_t p = 0; p < np; ++p)
      for (int j = kt_p; j < s; ++j) lev_e[l - 1] += sg[size_t(p) * s + j] * sg[size_t(p) * s + j];
    Pt.rows[l - 1] = kt_p;
    Pt.T[l - 1].assign(size_t(np) * kt_p * kp, 0.0);
    g_flops.gemm(double(np), kt_p, kp, zr);
    for (int64_t p = 0; p < np; ++p)
      mm(kt_p, kp, zr, W.data() + p * zr * kp, zr, true, Z.data() + p * zr * kp, zr, false,
         Pt.T[l - 1].data() + p * kt_p * kp, kt_p);
    std::vector<double> E(size_t(A.nodes(l)) * kt_c * kt_p, 0.0);
    for (int64_t c = 0; c < A.nodes(l); ++c) {
      const double* src = W.data() + (c / 2) * zr * kp + (c % 2) * kt_c;
      double* dst = E.data() + c * kt_c * kt_p;
      for (int j = 0; j < kt_p; ++j)
        for (int i = 0; i < kt_c; ++i) dst[i + size_t(j) * kt_c] = src[i + size_t(j) * zr];
    }
    A.tr[l] = std::move(E);
  }
  A.rank = nr;
  double energy = 0;  // compress() sums the levels in order (compression.hpp:531-532)
  for (double e : lev_e) energy += e;
  return energy;
}

uint64_t footprint(const OMat& A) {
  uint64_t e = A.dense.val.size() + A.leaf.size();
  for (const auto& L : A.cpl) e += L.val.size();
  for (int l = 1; l <= A.q; ++l) e += A.tr[l].size();
  return e * sizeof(double);
}

double frob2(const OMat& A) {
  double s = 0;
  for (const auto& L : A.cpl)
    for (double v : L.val) s += v * v;
  for (double v : A.dense.val) s += v * v;
  return s;
}

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

std::vector<int64_t> concat_offsets(const OMat& A) {
  std::vector<int64_t> o(A.q + 2, 0);
  for (int l = 0; l <= A.q; ++l) o[l + 1] = o[l] + A.nodes(l) * int64_t(A.rank[l]) * A.rank[l];
  return o;
}

}  // namespace

// ============================================================================
// C-ABI (same flat layout and argument meaning as oracle/ref_capi.cpp).
extern "C" {

const char* h2o_last_error() { return g_err.c_str(); }

int h2o_points(int dim, int n, double pert, uint64_t seed, double* out) {
  return guarded([&] {
    const auto p = make_points(dim, n, pert, seed);
    std::memcpy(out, p.data(), p.size() * sizeof(double));
  });
}

int h2o_random_vector(int n, uint64_t seed, double* out) {
  // validate.hpp:13-20
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  for (int i = 0; i < n; ++i) out[i] = u(gen);
  return 0;
}

// Cluster order + per-level boxes (lo/hi, 3 doubles each, level-concatenated).
int h2o_cluster(int dim, int n, int leaf, double pert, uint64_t seed, int32_t* order,
                double* boxes_lo, double* boxes_hi) {
  return guarded([&] {
    const auto pts = make_points(dim, n, pert, seed);
    const Clusters C = cluster(pts, dim, n, leaf);
    std::memcpy(order, C.order.data(), C.order.size() * sizeof(int32_t));
    int64_t o = 0;
    for (int l = 0; l <= C.q; ++l)
      for (const Box& b : C.boxes[l]) {
        for (int a = 0; a < 3; ++a) {
          boxes_lo[o * 3 + a] = b.lo[a];
          boxes_hi[o * 3 + a] = b.hi[a];
        }
        ++o;
      }
  });
}

int h2o_construct(int dim, int n, int leaf, int order, double eta, double ell, double pert,
                  uint64_t seed, void** out) {
  return guarded([&] { *out = new OMat(build(dim, n, leaf, order, eta, ell, pert, seed)); });
}

void h2o_destroy(void* h) { delete static_cast<OMat*>(h); }
void* h2o_clone(void* h) { return new OMat(*static_cast<OMat*>(h)); }

void h2o_shape(void* h, int* out) {
  const OMat& A = *static_cast<OMat*>(h);
  out[0] = A.n;
  out[1] = A.m;
  out[2] = A.q;
  out[3] = 1;
}

void h2o_layout(void* h, int* ranks, int64_t* cpl_blocks, int* brows, int* bcols,
                int64_t* dense_blocks) {
  const OMat& A = *static_cast<OMat*>(h);
  for (int l = 0; l <= A.q; ++l) {
    ranks[l] = A.rank[l];
    cpl_blocks[l] = A.cpl[l].nblocks();
    brows[l] = A.cpl[l].br;
    bcols[l] = A.cpl[l].bc;
  }
  *dense_blocks = A.dense.nblocks();
}

void h2o_export(void* h, int32_t* perm, double* leaf, double* transfer, int32_t* rp,
                int32_t* ci, double* sv, int32_t* drp, int32_t* dci, double* dv) {
  const OMat& A = *static_cast<OMat*>(h);
  std::copy(A.perm.begin(), A.perm.end(), perm);
  std::copy(A.leaf.begin(), A.leaf.end(), leaf);
  for (int l = 1; l <= A.q; ++l) transfer = std::copy(A.tr[l].begin(), A.tr[l].end(), transfer);
  for (const Csr& L : A.cpl) {
    rp = std::copy(L.ptr.begin(), L.ptr.end(), rp);
    ci = std::copy(L.col.begin(), L.col.end(), ci);
    sv = std::copy(L.val.begin(), L.val.end(), sv);
  }
  std::copy(A.dense.ptr.begin(), A.dense.ptr.end(), drp);
  std::copy(A.dense.col.begin(), A.dense.col.end(), dci);
  std::copy(A.dense.val.begin(), A.dense.val.end(), dv);
}

int h2o_import(int n, int m, int depth, const int32_t* ranks, const int32_t* perm,
               const double* leaf, const double* transfer, const int32_t* rp,
               const int32_t* ci, const double* sv, const int32_t* drp, const int32_t* dci,
               const double* dv, void** out) {
  return guarded([&] {
    check(n == (m << depth), "import: n must equal m * 2^depth");
    OMat* A = new OMat;
    A->n = n;
    A->m = m;
    A->q = depth;
    A->perm.assign(perm, perm + n);
    A->rank.assign(ranks, ranks + depth + 1);
    const int64_t nlf = A->nodes(depth);
    A->leaf.assign(leaf, leaf + nlf * m * ranks[depth]);
    A->tr.assign(depth + 1, {});
    for (int l = 1; l <= depth; ++l) {
      const int64_t sz = A->nodes(l) * ranks[l] * ranks[l - 1];
      A->tr[l].assign(transfer, transfer + sz);
      transfer += sz;
    }
    A->cpl.resize(depth + 1);
    for (int l = 0; l <= depth; ++l) {
      Csr& L = A->cpl[l];
      L.rows = int(A->nodes(l));
      L.br = L.bc = ranks[l];
      L.ptr.assign(rp, rp + L.rows + 1);
      rp += L.rows + 1;
      const int64_t nb = L.ptr.back();
      L.col.assign(ci, ci + nb);
      ci += nb;
      L.val.assign(sv, sv + nb * ranks[l] * ranks[l]);
      sv += nb * ranks[l] * ranks[l];
    }
    Csr& D = A->dense;
    D.rows = int(nlf);
    D.br = D.bc = m;
    D.ptr.assign(drp, drp + nlf + 1);
    D.col.assign(dci, dci + D.ptr.back());
    D.val.assign(dv, dv + int64_t(D.ptr.back()) * m * m);
    *out = A;
  });
}

uint64_t h2o_footprint(void* h) { return footprint(*static_cast<OMat*>(h)); }

void h2o_flops_reset() { g_flops = Flops{}; }
double h2o_flops_total() { return g_flops.total; }

int h2o_hmv(void* h, const double* x, double* y, double alpha, double beta) {
  return guarded([&] { hmv(*static_cast<OMat*>(h), x, y, alpha, beta); });
}

int h2o_upsweep(void* h, const double* xc, double* xh) {
  return guarded([&] { upsweep(*static_cast<OMat*>(h), xc, xh); });
}

int h2o_tree_multiply(void* h, const double* xh, double* yh) {
  return guarded([&] { tree_mult(*static_cast<OMat*>(h), xh, yh); });
}

int h2o_downsweep(void* h, const double* yh_in, double* yc) {
  return guarded([&] {
    const OMat& A = *static_cast<OMat*>(h);
    const auto off = vec_offsets(A);
    std::vector<double> yh(yh_in, yh_in + off.back());
    downsweep(A, yh.data(), yc);
  });
}

int h2o_dense_mv(void* h, const double* xc, double* yc, double alpha, double beta) {
  return guarded([&] { bsr_mv(static_cast<OMat*>(h)->dense, xc, yc, alpha, beta); });
}

// Same report layout as ref_compress; times are 0 (the oracle is not timed
// per phase), flops follow the reference's analytic model.
int h2o_compress(void* h, double eps, double* report) {
  return guarded([&] {
    OMat& A = *static_cast<OMat*>(h);
    const uint64_t before = footprint(A);
    double f[5];
    double f0 = g_flops.total;
    Proj To = orthogonalize(A);
    f[0] = g_flops.total - f0;
    f0 = g_flops.total;
    project(To, A);
    f[1] = g_flops.total - f0;
    const double nrm = std::sqrt(frob2(A));
    f0 = g_flops.total;
    const auto R = weights(A);
    f[2] = g_flops.total - f0;
    f0 = g_flops.total;
    Proj Tt;
    const double energy = truncate(A, R, eps, Tt);
    f[3] = g_flops.total - f0;
    f0 = g_flops.total;
    project(Tt, A);
    f[4] = g_flops.total - f0;
    const double v[] = {nrm > 0 ? std::sqrt(energy) / nrm : 0.0, nrm, double(before),
                        double(footprint(A)), 0, 0, 0, 0, 0, f[0], f[1], f[2], f[3], f[4]};
    std::memcpy(report, v, sizeof(v));
  });
}

int h2o_orthogonalize(void* h, double* t_out) {
  return guarded([&] {
    const Proj P = orthogonalize(*static_cast<OMat*>(h));
    for (const auto& t : P.T) t_out = std::copy(t.begin(), t.end(), t_out);
  });
}

int h2o_orth_project_weights(void* h, double* r_out) {
  return guarded([&] {
    OMat& A = *static_cast<OMat*>(h);
    const Proj P = orthogonalize(A);
    project(P, A);
    const auto R = weights(A);
    for (const auto& r : R) r_out = std::copy(r.begin(), r.end(), r_out);
  });
}

// Batched-kernel oracles for the reference KATs (test_batch.cpp).
int h2o_qr(int rows, int cols, double* A, double* R) {
  return guarded([&] {
    check(rows >= cols, "qr_batched: requires rows >= cols");
    qr_thin(rows, cols, A, rows, R, cols);
  });
}

int h2o_svd(int rows, int cols, double* W, double eps, int* rank, double* sig) {
  return guarded([&] {
    std::vector<int> rk;
    std::vector<double> sg;
    svd_batch(1, rows, cols, W, int64_t(rows) * cols, eps, rk, sg);
    *rank = rk[0];
    std::copy(sg.begin(), sg.end(), sig);
  });
}

}  // extern "C"
