// Ab-initio construction of the H^2 matrix directly into HBM.
//
// Host (C++): the reference's structure — perturbed grid
// (src/geometry.cpp:115-149), KD cluster tree with exact median split
// (geometry.cpp:172-225), dual-traversal block partition
// (src/construction.cpp:7-36), CSR per level (construction.hpp:45-65).
// The same libstdc++ mt19937_64 / uniform_real_distribution / nth_element
// are used, so perm and block structure are bit-identical to construct().
//
// Device: every value pool is evaluated in place by one kernel each —
// Lagrange leaf bases (construction.hpp:71-90), transfer matrices (:95-118),
// coupling blocks at Chebyshev node pairs (:122-149), dense blocks at point
// pairs (:153-175).  This file is compiled with -fmad=false so the Chebyshev
// and Lagrange arithmetic rounds exactly like the reference; kernel values
// differ from the host only through the device exp() (<= 1 ulp).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <random>
#include <vector>

#include "h2b_internal.hpp"

namespace h2b {

void allocate(Matrix& A);
void check_value_symmetry(Matrix& A);
void upload_structure(Matrix& A);

namespace {

constexpr int kMaxOrder = 16;

struct Box3 {
  double lo[3], hi[3];
};

// ---------------------------------------------------------------- host structure
std::vector<double> perturbed_grid(int dim, int64_t n, double pert, uint64_t seed) {
  require(dim == 2 || dim == 3, "generate_perturbed_grid: dim must be 2 or 3");
  require(n > 0, "generate_perturbed_grid: n must be positive");
  require(pert >= 0 && pert < 0.5, "generate_perturbed_grid: perturbation must be in [0, 0.5)");
  std::vector<int64_t> side(dim);
  const int64_t root = std::llround(std::pow(double(n), 1.0 / dim));
  int64_t prod = 1;
  for (int a = 0; a < dim; ++a) prod *= root;
  if (prod == n) {
    std::fill(side.begin(), side.end(), root);
  } else {
    require((n & (n - 1)) == 0,
            "generate_perturbed_grid: n must be a perfect dim-th power or a power of two");
    int e = 0;
    while ((int64_t(1) << e) < n) ++e;
    for (int a = 0; a < dim; ++a) side[a] = int64_t(1) << (e / dim + (a < e % dim ? 1 : 0));
  }
  double h[3] = {0, 0, 0};
  for (int a = 0; a < dim; ++a) h[a] = side[a] > 1 ? 1.0 / double(side[a] - 1) : 1.0;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> jitter(-1.0, 1.0);
  std::vector<double> X(size_t(n) * dim);
  int64_t ix[3] = {0, 0, 0};
  for (int64_t p = 0; p < n; ++p) {
    for (int a = 0; a < dim; ++a) {
      const double base = side[a] > 1 ? double(ix[a]) * h[a] : 0.5;
      X[p * dim + a] = std::clamp(base + pert * h[a] * jitter(rng), 0.0, 1.0);
    }
    for (int a = 0; a < dim && ++ix[a] == side[a]; ++a) ix[a] = 0;
  }
  return X;
}

struct Tree {
  int q = 0;
  std::vector<int32_t> perm;
  std::vector<Box3> box;           // level-concatenated: node (l, i) at (1 << l) - 1 + i
  const Box3& at(int l, int64_t i) const { return box[(int64_t(1) << l) - 1 + i]; }
};

Tree cluster_tree(const std::vector<double>& X, int dim, int64_t n, int leaf) {
  require(leaf > 0, "build_cluster_tree: leaf_size must be positive");
  const int64_t nleaf = n / leaf;
  require(nleaf * leaf == n, "build_cluster_tree: n must be leaf_size * 2^q");
  int q = 0;
  while ((int64_t(1) << q) < nleaf) ++q;
  require((int64_t(1) << q) == nleaf, "build_cluster_tree: n must be leaf_size * 2^q");
  Tree T;
  T.q = q;
  T.perm.resize(n);
  std::iota(T.perm.begin(), T.perm.end(), 0);
  T.box.resize((size_t(2) << q) - 1);
  const double* P = X.data();
  // level by level; node (l, i) covers [i * n / 2^l, (i+1) * n / 2^l)
  for (int l = 0; l <= q; ++l) {
    const int64_t cnt = n >> l;
    for (int64_t i = 0; i < (int64_t(1) << l); ++i) {
      int32_t* ids = T.perm.data() + i * cnt;
      Box3& b = T.box[(int64_t(1) << l) - 1 + i];
      for (int a = 0; a < 3; ++a) {
        b.lo[a] = a < dim ? 1e300 : 0.0;
        b.hi[a] = a < dim ? -1e300 : 0.0;
      }
      for (int64_t t = 0; t < cnt; ++t)
        for (int a = 0; a < dim; ++a) {
          const double c = P[int64_t(ids[t]) * dim + a];
          b.lo[a] = std::min(b.lo[a], c);
          b.hi[a] = std::max(b.hi[a], c);
        }
      if (l == q) continue;
      int ax = 0;
      double wmax = -1;
      for (int a = 0; a < dim; ++a)
        if (b.hi[a] - b.lo[a] > wmax) {
          wmax = b.hi[a] - b.lo[a];
          ax = a;
        }
      std::nth_element(ids, ids + cnt / 2, ids + cnt, [=](int32_t u, int32_t v) {
        const double cu = P[int64_t(u) * dim + ax], cv = P[int64_t(v) * dim + ax];
        return cu < cv || (cu == cv && u < v);
      });
    }
  }
  return T;
}

double box_diam(const Box3& b, int dim) {
  double s = 0;
  for (int a = 0; a < dim; ++a) s += (b.hi[a] - b.lo[a]) * (b.hi[a] - b.lo[a]);
  return std::sqrt(s);
}

double box_gap(const Box3& x, const Box3& y, int dim) {
  double s = 0;
  for (int a = 0; a < dim; ++a) {
    const double g = std::max({0.0, x.lo[a] - y.hi[a], y.lo[a] - x.hi[a]});
    s += g * g;
  }
  return std::sqrt(s);
}

struct Pairs {
  std::vector<std::vector<std::pair<int32_t, int32_t>>> far;
  std::vector<std::pair<int32_t, int32_t>> near;
};

void traverse(const Tree& T, int dim, double eta, int l, int32_t i, int32_t j, Pairs& P) {
  const Box3& bi = T.at(l, i);
  const Box3& bj = T.at(l, j);
  if (l > 0 && std::max(box_diam(bi, dim), box_diam(bj, dim)) <= eta * box_gap(bi, bj, dim)) {
    P.far[l].emplace_back(i, j);
    return;
  }
  if (l == T.q) {
    P.near.emplace_back(i, j);
    return;
  }
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) traverse(T, dim, eta, l + 1, 2 * i + a, 2 * j + b, P);
}

void to_csr(std::vector<std::pair<int32_t, int32_t>>& pr, int64_t rows, int dim_r, int dim_c,
            Layer& L) {
  std::sort(pr.begin(), pr.end());
  L.rows = rows;
  L.br = dim_r;
  L.bc = dim_c;
  L.h_rp.assign(rows + 1, 0);
  L.h_ci.resize(pr.size());
  for (size_t b = 0; b < pr.size(); ++b) {
    ++L.h_rp[pr[b].first + 1];
    L.h_ci[b] = pr[b].second;
  }
  for (int64_t r = 0; r < rows; ++r) L.h_rp[r + 1] += L.h_rp[r];
  L.nb = int64_t(pr.size());
}

// ---------------------------------------------------------------- device values
struct ChebTables {
  double t[kMaxOrder];  // first-kind points, increasing (chebyshev.cpp:21-28)
  double w[kMaxOrder];  // barycentric weights (-1)^(j+1) sin((2j+1)pi/2n) (chebyshev.cpp:55-75)
};

__device__ __forceinline__ void widen_axis(const Box3& b, int a, double& lo, double& hi) {
  lo = b.lo[a];
  hi = b.hi[a];
  if (hi - lo < 1e-8) {
    const double mid = 0.5 * (lo + hi);
    lo = mid - 0.5 * 1e-8;
    hi = mid + 0.5 * 1e-8;
  }
}

__device__ __forceinline__ void lagrange_axis(const ChebTables& C, int order, double lo, double hi,
                                              double x, double* out) {
  const double xr = (2.0 * x - (lo + hi)) / (hi - lo);
  for (int j = 0; j < order; ++j)
    if (xr == C.t[j]) {
      for (int i = 0; i < order; ++i) out[i] = i == j ? 1.0 : 0.0;
      return;
    }
  double den = 0.0;
  for (int j = 0; j < order; ++j) {
    out[j] = C.w[j] / (xr - C.t[j]);
    den += out[j];
  }
  for (int j = 0; j < order; ++j) out[j] = out[j] / den;
}

// Tensor Lagrange values of `box` at point x, written with stride ostride.
__device__ void lagrange_tensor_dev(const ChebTables& C, int order, int dim, const Box3& box,
                                    const double* x, double* out, int64_t ostride, int k) {
  double per[3][kMaxOrder];
  for (int a = 0; a < dim; ++a) {
    double lo, hi;
    widen_axis(box, a, lo, hi);
    lagrange_axis(C, order, lo, hi, x[a], per[a]);
  }
  int idx[3] = {0, 0, 0};
  for (int g = 0; g < k; ++g) {
    double v = 1.0;
    for (int a = 0; a < dim; ++a) v *= per[a][idx[a]];
    out[g * ostride] = v;
    for (int a = 0; a < dim; ++a) {
      if (++idx[a] < order) break;
      idx[a] = 0;
    }
  }
}

// Chebyshev node g of `box` (first axis fastest), chebyshev.cpp:30-53.
__device__ __forceinline__ void cheb_node(const ChebTables& C, int order, int dim, const Box3& b,
                                          int g, double* out) {
  for (int a = 0; a < dim; ++a) {
    double lo, hi;
    widen_axis(b, a, lo, hi);
    const int i = g % order;
    g /= order;
    out[a] = 0.5 * (lo + hi) + 0.5 * (hi - lo) * C.t[i];
  }
}

__device__ __forceinline__ double kernel_exp(const double* x, const double* y, int dim, double ell) {
  double d2 = 0.0;
  for (int a = 0; a < dim; ++a) {
    const double d = x[a] - y[a];
    d2 += d * d;
  }
  return exp(-sqrt(d2) / ell);
}

__global__ void k_leaf_basis(const ChebTables C, int order, int dim, const Box3* __restrict__ leaf_box,
                             const double* __restrict__ pts_c, int m, int ldm, int k, int64_t nleaf,
                             double* __restrict__ leaf) {
  const int64_t total = nleaf * ldm;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / ldm;
    const int p = int(e - i * ldm);
    double* out = leaf + i * int64_t(ldm) * k + p;
    if (p >= m) {
      for (int g = 0; g < k; ++g) out[int64_t(g) * ldm] = 0.0;
      continue;
    }
    lagrange_tensor_dev(C, order, dim, leaf_box[i], pts_c + (i * m + p) * dim, out, ldm, k);
  }
}

// child_box / E start at the first stored child c0 (global index c0 + c).
__global__ void k_transfer(const ChebTables C, int order, int dim, const Box3* __restrict__ child_box,
                           const Box3* __restrict__ parent_box, int k, int ldk, int64_t nchild,
                           int64_t c0, double* __restrict__ E) {
  const int64_t total = nchild * ldk;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = e / ldk;
    const int ac = int(e - c * ldk);
    double* out = E + c * int64_t(ldk) * k + ac;
    if (ac >= k) {
      for (int g = 0; g < k; ++g) out[int64_t(g) * ldk] = 0.0;
      continue;
    }
    double node[3];
    cheb_node(C, order, dim, child_box[c], ac, node);
    lagrange_tensor_dev(C, order, dim, parent_box[(c0 + c) >> 1], node, out, ldk, k);
  }
}

__global__ void k_coupling(const ChebTables C, int order, int dim, double ell,
                           const Box3* __restrict__ lvl_box, const int32_t* __restrict__ blk_row,
                           const int32_t* __restrict__ col_idx, int k, int ldk, int64_t nb,
                           double* __restrict__ S) {
  const int64_t per = int64_t(ldk) * k;
  const int64_t total = nb * per;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = e / per;
    const int64_t w = e - b * per;
    const int c = int(w / ldk);
    const int a = int(w - int64_t(c) * ldk);
    double v = 0.0;
    if (a < k) {
      double gi[3], gj[3];
      cheb_node(C, order, dim, lvl_box[blk_row[b]], a, gi);
      cheb_node(C, order, dim, lvl_box[col_idx[b]], c, gj);
      v = kernel_exp(gi, gj, dim, ell);
    }
    S[e] = v;
  }
}

__global__ void k_dense(int dim, double ell, const double* __restrict__ pts_c,
                        const int32_t* __restrict__ blk_row, const int32_t* __restrict__ col_idx,
                        int m, int ldm, int64_t nb, double* __restrict__ D) {
  const int64_t per = int64_t(ldm) * m;
  const int64_t total = nb * per;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = e / per;
    const int64_t w = e - b * per;
    const int c = int(w / ldm);
    const int a = int(w - int64_t(c) * ldm);
    double v = 0.0;
    if (a < m)
      v = kernel_exp(pts_c + (int64_t(blk_row[b]) * m + a) * dim,
                     pts_c + (int64_t(col_idx[b]) * m + c) * dim, dim, ell);
    D[e] = v;
  }
}

unsigned grid_of(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(sms) * 32)));
}

std::vector<int32_t> block_rows(const Layer& L) {
  std::vector<int32_t> r(L.nb);
  for (int64_t i = 0; i < L.rows; ++i)
    for (int32_t b = L.h_rp[i]; b < L.h_rp[i + 1]; ++b) r[b] = int32_t(i);
  return r;
}

}  // namespace

h2b_matrix* build_matrix(const h2b_build_config& cfg, int device, int nparts, int part) {
  require(cfg.dim == 2 || cfg.dim == 3, "generate_perturbed_grid: dim must be 2 or 3");
  require(cfg.grid_order >= 1, "chebyshev_points: order must be >= 1");
  require(cfg.eta > 0, "dual_traversal_partition: eta must be positive");
  require(cfg.ell > 0, "correlation length must be positive");
  if (cfg.grid_order > kMaxOrder) throw Error(H2B_UNSUPPORTED, "grid_order > 16 not supported");
  int k = 1;
  for (int a = 0; a < cfg.dim; ++a) k *= cfg.grid_order;
  if (k > kMaxDimHmv || cfg.leaf_size > kMaxDimHmv)
    throw Error(H2B_UNSUPPORTED, "rank or leaf size > 128 not supported by the compiled kernels");

  const std::vector<double> X = perturbed_grid(cfg.dim, cfg.n, cfg.perturbation, cfg.seed);
  const Tree T = cluster_tree(X, cfg.dim, cfg.n, cfg.leaf_size);
  const int q = T.q;
  require(q <= kMaxLevels - 1, "tree too deep");
  require(nparts >= 1 && (nparts & (nparts - 1)) == 0, "partition count must be a power of two");
  int ps = 0;
  while ((1 << ps) < nparts) ++ps;
  require(ps <= q, "more partitions than leaves");
  require(part >= 0 && part < nparts, "partition index out of range");
  Pairs P;
  P.far.resize(q + 1);
  traverse(T, cfg.dim, cfg.eta, 0, 0, 0, P);

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    throw Error(H2B_NO_DEVICE, "no sm_100 CUDA device available (libh2b has no CPU fallback)");
  }
  require(device >= 0 && device < ndev, "device index out of range");
  H2B_CUDA(cudaSetDevice(device));

  std::unique_ptr<h2b_matrix> A(new h2b_matrix);
  A->device = device;
  H2B_CUDA(cudaStreamCreateWithFlags(&A->stream, cudaStreamNonBlocking));
  cudaStream_t s = A->stream;
  A->n = cfg.n;
  A->m = cfg.leaf_size;
  A->q = q;
  A->rank.assign(q + 1, k);
  A->part_s = ps;
  A->part_g = part;
  {  // memory_footprint of the whole matrix (h2_matrix.hpp:90-102)
    uint64_t e = uint64_t(P.near.size()) * A->m * A->m + uint64_t(A->nodes(q)) * A->m * k;
    for (int l = 0; l <= q; ++l) e += uint64_t(P.far[l].size()) * k * k;
    for (int l = 1; l <= q; ++l) e += uint64_t(A->nodes(l)) * k * k;
    A->global_footprint = 8 * e;
  }
  // keep only the block rows this partition computes (levels >= ps split)
  auto keep = [&](std::vector<std::pair<int32_t, int32_t>>& v, int l) {
    if (ps == 0 || l < ps) return;
    const int64_t b0 = A->own_begin(l), b1 = A->own_end(l);
    v.erase(std::remove_if(v.begin(), v.end(),
                           [&](const std::pair<int32_t, int32_t>& e) { return e.first < b0 || e.first >= b1; }),
            v.end());
  };
  A->cpl.resize(q + 1);
  for (int l = 0; l <= q; ++l) {
    keep(P.far[l], l);
    to_csr(P.far[l], A->nodes(l), k, k, A->cpl[l]);
    A->cpl[l].row0 = A->own_begin(l);
    A->cpl[l].row1 = A->own_end(l);
  }
  keep(P.near, q);
  to_csr(P.near, A->nodes(q), A->m, A->m, A->dense);
  A->dense.row0 = A->own_begin(q);
  A->dense.row1 = A->own_end(q);
  P = Pairs{};
  allocate(*A);
  upload_structure(*A);
  H2B_CUDA(cudaMemcpyAsync(A->perm.p, T.perm.data(), size_t(cfg.n) * sizeof(int32_t),
                           cudaMemcpyHostToDevice, s));

  // cluster-ordered points, boxes, Chebyshev tables
  std::vector<double> pc(size_t(cfg.n) * cfg.dim);
  for (int64_t t = 0; t < cfg.n; ++t)
    for (int a = 0; a < cfg.dim; ++a) pc[t * cfg.dim + a] = X[int64_t(T.perm[t]) * cfg.dim + a];
  A->pts_orig.alloc(X.size());
  H2B_CUDA(cudaMemcpyAsync(A->pts_orig.p, X.data(), X.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  A->pts_dim = cfg.dim;
  A->ell = cfg.ell;
  A->info.dim = cfg.dim;
  A->info.seed = cfg.seed;
  A->info.perturbation = cfg.perturbation;
  A->info.ell = cfg.ell;
  A->info.eta = cfg.eta;
  A->info.grid_order = cfg.grid_order;
  DevBuf<double> dpts;
  dpts.alloc(pc.size());
  H2B_CUDA(cudaMemcpyAsync(dpts.p, pc.data(), pc.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  DevBuf<Box3> dbox;
  dbox.alloc(T.box.size());
  H2B_CUDA(cudaMemcpyAsync(dbox.p, T.box.data(), T.box.size() * sizeof(Box3), cudaMemcpyHostToDevice, s));
  ChebTables C{};
  const int order = cfg.grid_order;
  for (int i = 0; i < order; ++i) {
    C.t[i] = -std::cos(M_PI * (2.0 * i + 1.0) / (2.0 * order));
    double w = std::sin(M_PI * (2.0 * i + 1.0) / (2.0 * order));
    C.w[i] = (i % 2 == 0) ? -w : w;
  }
  if (order == 1) C.t[0] = 0.0;
  auto box_of = [&](int l) { return dbox.p + ((int64_t(1) << l) - 1); };

  const int64_t nleaf = A->own_count(q), leaf0 = A->own_begin(q);
  k_leaf_basis<<<grid_of(nleaf * A->ldm), 256, 0, s>>>(C, order, cfg.dim, box_of(q) + leaf0,
                                                       dpts.p + leaf0 * A->m * cfg.dim, A->m, A->ldm, k,
                                                       nleaf, A->leaf.p);
  H2B_CUDA(cudaGetLastError());
  for (int l = 1; l <= q; ++l) {
    const int64_t c0 = A->tr_begin(l), nc = A->tr_count(l);
    k_transfer<<<grid_of(nc * A->ld(l)), 256, 0, s>>>(C, order, cfg.dim, box_of(l) + c0, box_of(l - 1), k,
                                                      A->ld(l), nc, c0, A->transfer.p + A->tr_off[l]);
    H2B_CUDA(cudaGetLastError());
  }
  for (int l = 0; l <= q; ++l) {
    const Layer& L = A->cpl[l];
    if (!L.nb) continue;
    const auto br = block_rows(L);
    DevBuf<int32_t> dbr;
    dbr.alloc(br.size());
    H2B_CUDA(cudaMemcpyAsync(dbr.p, br.data(), br.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    k_coupling<<<grid_of(L.nb * L.block_stride()), 256, 0, s>>>(C, order, cfg.dim, cfg.ell, box_of(l),
                                                                dbr.p, L.ci, k, L.ld, L.nb, L.val);
    H2B_CUDA(cudaGetLastError());
    H2B_CUDA(cudaStreamSynchronize(s));
  }
  {
    const Layer& D = A->dense;
    const auto br = block_rows(D);
    DevBuf<int32_t> dbr;
    dbr.alloc(std::max<size_t>(1, br.size()));
    if (!br.empty())
      H2B_CUDA(cudaMemcpyAsync(dbr.p, br.data(), br.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    if (D.nb) {
      k_dense<<<grid_of(D.nb * D.block_stride()), 256, 0, s>>>(cfg.dim, cfg.ell, dpts.p, dbr.p, D.ci,
                                                               A->m, D.ld, D.nb, D.val);
      H2B_CUDA(cudaGetLastError());
    }
    H2B_CUDA(cudaStreamSynchronize(s));
  }
  check_value_symmetry(*A);
  return A.release();
}

}  // namespace h2b
