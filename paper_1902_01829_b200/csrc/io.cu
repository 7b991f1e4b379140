// Container I/O (include/h2kit/io.hpp:22-282, src/crc32.cpp:6-20): the
// reference's ".h2" file format, byte for byte, straight to and from the
// HBM-resident matrix.
//
//   magic "H2KT" | u16 version 1 | u8 precision (8) | u8 reserved
//   sections, each  u64 payload length | u32 crc32(payload) | payload
//     meta      i64 n, i32 m, u8 symmetric, BuildInfo (i32 dim, u64 seed,
//               f64 perturbation, ell, eta, i32 grid_order)
//     bases     FlatTree (parent, head, next, level_ptr), ranks, i32 leaf_dim,
//               leaf_pool, u64 #levels, transfer[l] (l = 0..q, [0] empty)
//     coupling  u64 #levels, per level BSRLayer (i32 block_rows, block_cols,
//               brows, bcols, row_ptr, col_idx, values)
//     dense     BSRLayer
//     perm      vector<index_t>
//   (vectors are u64 count + raw little-endian elements)
//
// save: each section is streamed -- the device pools are downloaded level by
// level into pinned staging, CRC'd on the host in parallel (per-chunk CRC32 +
// GF(2) combination), and written; the header is patched after the payload.
// load: sections are read and checked (length, CRC) exactly like the
// reference, then uploaded through the same path as h2b_matrix_create.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "h2b_internal.hpp"

namespace h2b {

h2b_matrix* create_from_desc(const h2b_matrix_desc& d, int device);
void download_blocks(const double* dev, double* host, int rows, int cols, int64_t count, cudaStream_t s);

namespace {

struct IoError : Error {
  explicit IoError(const std::string& m) : Error(H2B_IO_ERROR, m) {}
};

// ------------------------------------------------------------------ CRC-32
// IEEE 802.3 (reflected 0xEDB88320), slicing-by-8.
struct CrcTables {
  uint32_t t[8][256];
  CrcTables() {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int b = 0; b < 8; ++b) c = (c >> 1) ^ ((c & 1u) ? 0xEDB88320u : 0u);
      t[0][i] = c;
    }
    for (uint32_t i = 0; i < 256; ++i)
      for (int k = 1; k < 8; ++k) t[k][i] = (t[k - 1][i] >> 8) ^ t[0][t[k - 1][i] & 0xFF];
  }
};
const CrcTables& tables() {
  static const CrcTables T;
  return T;
}

// raw (un-inverted) register update
uint32_t crc_raw(uint32_t c, const unsigned char* p, size_t n) {
  const auto& T = tables().t;
  while (n >= 8) {
    uint32_t lo, hi;
    std::memcpy(&lo, p, 4);
    std::memcpy(&hi, p + 4, 4);
    lo ^= c;
    c = T[7][lo & 0xFF] ^ T[6][(lo >> 8) & 0xFF] ^ T[5][(lo >> 16) & 0xFF] ^ T[4][lo >> 24] ^
        T[3][hi & 0xFF] ^ T[2][(hi >> 8) & 0xFF] ^ T[1][(hi >> 16) & 0xFF] ^ T[0][hi >> 24];
    p += 8;
    n -= 8;
  }
  while (n--) c = T[0][(c ^ *p++) & 0xFF] ^ (c >> 8);
  return c;
}

// zlib's crc32_combine: crc(A||B) from crc(A), crc(B), |B| (GF(2) matrices)
uint32_t gf2_times(const uint32_t* mat, uint32_t vec) {
  uint32_t sum = 0;
  for (int i = 0; vec; ++i, vec >>= 1)
    if (vec & 1) sum ^= mat[i];
  return sum;
}
void gf2_square(uint32_t* sq, const uint32_t* mat) {
  for (int n = 0; n < 32; ++n) sq[n] = gf2_times(mat, mat[n]);
}
uint32_t crc_combine(uint32_t crc1, uint32_t crc2, uint64_t len2) {
  if (len2 == 0) return crc1;
  uint32_t even[32], odd[32];
  odd[0] = 0xEDB88320u;
  uint32_t row = 1;
  for (int n = 1; n < 32; ++n) {
    odd[n] = row;
    row <<= 1;
  }
  gf2_square(even, odd);
  gf2_square(odd, even);
  do {
    gf2_square(even, odd);
    if (len2 & 1) crc1 = gf2_times(even, crc1);
    len2 >>= 1;
    if (!len2) break;
    gf2_square(odd, even);
    if (len2 & 1) crc1 = gf2_times(odd, crc1);
    len2 >>= 1;
  } while (len2);
  return crc1 ^ crc2;
}

// finalized CRC of a buffer, computed by up to 16 threads on 64 MiB chunks
uint32_t crc32_parallel(const void* data, size_t len) {
  const auto* p = static_cast<const unsigned char*>(data);
  const size_t chunk = size_t(64) << 20;
  if (len <= chunk) return ~crc_raw(~0u, p, len);
  const size_t nch = (len + chunk - 1) / chunk;
  std::vector<uint32_t> part(nch);
  const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (size_t c = t; c < nch; c += nt) {
        const size_t n = std::min(chunk, len - c * chunk);
        part[c] = ~crc_raw(~0u, p + c * chunk, n);
      }
    });
  for (auto& x : th) x.join();
  uint32_t crc = part[0];
  for (size_t c = 1; c < nch; ++c) crc = crc_combine(crc, part[c], std::min(chunk, len - c * chunk));
  return crc;
}

// ------------------------------------------------------------------ writer
// One section streamed to the file: header placeholder, payload pieces with a
// running CRC, header patched at the end.
struct SectionWriter {
  std::ofstream& os;
  std::streampos head;
  uint64_t len = 0;
  uint32_t crc = 0;  // finalized CRC of what was written so far
  explicit SectionWriter(std::ofstream& o) : os(o) {
    head = os.tellp();
    const uint64_t z64 = 0;
    const uint32_t z32 = 0;
    os.write(reinterpret_cast<const char*>(&z64), 8);
    os.write(reinterpret_cast<const char*>(&z32), 4);
  }
  void bytes(const void* p, size_t n) {
    if (!n) return;
    crc = crc_combine(crc, crc32_parallel(p, n), n);
    os.write(static_cast<const char*>(p), std::streamsize(n));
    len += n;
  }
  template <class V>
  void put(const V& v) {
    bytes(&v, sizeof(V));
  }
  template <class V>
  void put_vec(const V* p, uint64_t count) {
    put(count);
    bytes(p, count * sizeof(V));
  }
  void finish() {
    const std::streampos end = os.tellp();
    os.seekp(head);
    os.write(reinterpret_cast<const char*>(&len), 8);
    os.write(reinterpret_cast<const char*>(&crc), 4);
    os.seekp(end);
  }
};

// Complete binary tree (flat_tree.cpp:18-41)
void flat_tree(int depth, std::vector<int32_t>& parent, std::vector<int32_t>& head, std::vector<int32_t>& next,
               std::vector<int32_t>& level_ptr) {
  level_ptr.assign(depth + 2, 0);
  for (int l = 0; l <= depth; ++l) level_ptr[l + 1] = level_ptr[l] + (int32_t(1) << l);
  const int32_t n = level_ptr.back();
  parent.assign(n, -1);
  head.assign(n, -1);
  next.assign(n, -1);
  for (int l = 0; l < depth; ++l) {
    const int32_t p0 = level_ptr[l], c0 = level_ptr[l + 1], np = level_ptr[l + 1] - p0;
    for (int32_t i = 0; i < np; ++i) {
      const int32_t p = p0 + i, c1 = c0 + 2 * i, c2 = c1 + 1;
      head[p] = c1;
      next[c1] = c2;
      parent[c1] = p;
      parent[c2] = p;
    }
  }
}

// device blocks (ld padded) -> host (unpadded), written as one vector<double>
void put_device_blocks(SectionWriter& w, const double* dev, int rows, int cols, int64_t count, cudaStream_t s,
                       std::vector<double>& host) {
  const uint64_t n = uint64_t(count) * rows * cols;
  w.put(n);
  const int64_t per = std::max<int64_t>(1, (int64_t(256) << 20) / (8 * std::max(1, rows * cols)));  // ~256 MB
  for (int64_t b = 0; b < count; b += per) {
    const int64_t nb = std::min(per, count - b);
    host.resize(size_t(nb) * rows * cols);
    download_blocks(dev + b * int64_t(pad2(rows)) * cols, host.data(), rows, cols, nb, s);
    w.bytes(host.data(), host.size() * sizeof(double));
  }
}

// ------------------------------------------------------------------ reader
struct Reader {
  const unsigned char* p;
  const unsigned char* end;
  template <class V>
  V get() {
    if (p + sizeof(V) > end) throw IoError("container section truncated");
    V v;
    std::memcpy(&v, p, sizeof(V));
    p += sizeof(V);
    return v;
  }
  template <class V>
  std::vector<V> get_vec() {
    const uint64_t count = get<uint64_t>();
    if (count > uint64_t(end - p) / sizeof(V)) throw IoError("container section truncated");
    std::vector<V> v(count);
    if (count) std::memcpy(v.data(), p, count * sizeof(V));
    p += count * sizeof(V);
    return v;
  }
};

std::vector<unsigned char> read_section(std::ifstream& is) {
  uint64_t len = 0;
  uint32_t crc = 0;
  is.read(reinterpret_cast<char*>(&len), 8);
  is.read(reinterpret_cast<char*>(&crc), 4);
  if (!is) throw IoError("container truncated: missing section header");
  std::vector<unsigned char> buf(len);
  is.read(reinterpret_cast<char*>(buf.data()), std::streamsize(len));
  if (uint64_t(is.gcount()) != len) throw IoError("container truncated: incomplete section payload");
  if (crc32_parallel(buf.data(), buf.size()) != crc) throw IoError("container corrupt: section checksum mismatch");
  return buf;
}

struct LayerIn {
  int32_t block_rows, block_cols, brows, bcols;
  std::vector<int32_t> row_ptr, col_idx;
  std::vector<double> values;
};
LayerIn get_layer(Reader& r) {
  LayerIn L;
  L.block_rows = r.get<int32_t>();
  L.block_cols = r.get<int32_t>();
  L.brows = r.get<int32_t>();
  L.bcols = r.get<int32_t>();
  L.row_ptr = r.get_vec<int32_t>();
  L.col_idx = r.get_vec<int32_t>();
  L.values = r.get_vec<double>();
  return L;
}

constexpr std::array<char, 4> kMagic{'H', '2', 'K', 'T'};
constexpr uint16_t kVersion = 1;

}  // namespace

uint32_t crc32_bytes(const void* p, size_t n) { return crc32_parallel(p, n); }

void save_matrix(const Matrix& A, const std::string& path, const h2b_build_info* info) {
  require(A.part_s == 0, "h2b_matrix_save: not supported on a partition handle");
  std::ofstream os(path, std::ios::binary | std::ios::trunc);
  if (!os) throw IoError("cannot open for writing: " + path);
  os.write(kMagic.data(), kMagic.size());
  const uint16_t ver = kVersion;
  os.write(reinterpret_cast<const char*>(&ver), 2);
  const uint8_t prec = 8, reserved = 0;
  os.write(reinterpret_cast<const char*>(&prec), 1);
  os.write(reinterpret_cast<const char*>(&reserved), 1);
  const h2b_build_info bi = info ? *info : A.info;
  cudaStream_t s = A.stream;
  const int q = A.q;
  std::vector<double> host;
  {
    SectionWriter w(os);  // meta
    w.put(int64_t(A.n));
    w.put(int32_t(A.m));
    w.put(uint8_t(A.symmetric ? 1 : 0));
    w.put(int32_t(bi.dim));
    w.put(uint64_t(bi.seed));
    w.put(bi.perturbation);
    w.put(bi.ell);
    w.put(bi.eta);
    w.put(int32_t(bi.grid_order));
    w.finish();
  }
  {
    SectionWriter w(os);  // trees + ranks + bases (row basis, then the column basis if any)
    std::vector<int32_t> parent, head, next, lp;
    flat_tree(q, parent, head, next, lp);
    auto put_basis = [&](const Matrix& B) {  // io_detail::put_basis
      w.put_vec(parent.data(), parent.size());
      w.put_vec(head.data(), head.size());
      w.put_vec(next.data(), next.size());
      w.put_vec(lp.data(), lp.size());
      std::vector<int32_t> ranks(B.rank.begin(), B.rank.end());
      w.put_vec(ranks.data(), ranks.size());
      w.put(int32_t(B.m));
      put_device_blocks(w, B.leaf.p, B.m, B.rank[q], B.nodes(q), s, host);
      w.put(uint64_t(q + 1));
      w.put(uint64_t(0));  // transfer[0] unused
      for (int l = 1; l <= q; ++l)
        put_device_blocks(w, B.transfer.p + B.tr_off[l], B.rank[l], B.rank[l - 1], B.nodes(l), s, host);
    };
    put_basis(A);
    if (!A.symmetric) put_basis(*A.colb);
    w.finish();
  }
  {
    SectionWriter w(os);  // coupling
    w.put(uint64_t(q + 1));
    for (int l = 0; l <= q; ++l) {
      const Layer& L = A.cpl[l];
      w.put(int32_t(A.nodes(l)));
      w.put(int32_t(A.nodes(l)));
      w.put(int32_t(L.br));
      w.put(int32_t(L.bc));
      w.put_vec(L.h_rp.data(), L.h_rp.size());
      w.put_vec(L.h_ci.data(), L.h_ci.size());
      put_device_blocks(w, L.val, L.br, L.bc, L.nb, s, host);
    }
    w.finish();
  }
  {
    SectionWriter w(os);  // dense
    const Layer& D = A.dense;
    w.put(int32_t(A.nodes(q)));
    w.put(int32_t(A.nodes(q)));
    w.put(int32_t(A.m));
    w.put(int32_t(A.m));
    w.put_vec(D.h_rp.data(), D.h_rp.size());
    w.put_vec(D.h_ci.data(), D.h_ci.size());
    put_device_blocks(w, D.val, A.m, A.m, D.nb, s, host);
    w.finish();
  }
  {
    SectionWriter w(os);  // perm
    std::vector<int32_t> perm(A.n);
    H2B_CUDA(cudaMemcpyAsync(perm.data(), A.perm.p, size_t(A.n) * 4, cudaMemcpyDeviceToHost, s));
    H2B_CUDA(cudaStreamSynchronize(s));
    w.put_vec(perm.data(), perm.size());
    w.finish();
  }
  os.flush();
  if (!os) throw IoError("write failed: " + path);
}

h2b_matrix* load_matrix(const std::string& path, int device, h2b_build_info* info_out) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw IoError("cannot open: " + path);
  std::array<char, 4> magic{};
  is.read(magic.data(), 4);
  uint16_t ver = 0;
  uint8_t prec = 0, reserved = 0;
  is.read(reinterpret_cast<char*>(&ver), 2);
  is.read(reinterpret_cast<char*>(&prec), 1);
  is.read(reinterpret_cast<char*>(&reserved), 1);
  if (!is || magic != kMagic) throw IoError("not a valid container: " + path);
  if (ver != kVersion) throw IoError("unsupported container version in " + path);
  if (prec != 8)
    throw IoError("precision mismatch: " + path + " stores " + std::to_string(prec * 8) + "-bit scalars");
  h2b_build_info bi{};
  int64_t n;
  int32_t m;
  bool symmetric;
  {
    auto buf = read_section(is);
    Reader r{buf.data(), buf.data() + buf.size()};
    n = r.get<int64_t>();
    m = r.get<int32_t>();
    symmetric = r.get<uint8_t>() != 0;
    bi.dim = r.get<int32_t>();
    bi.seed = r.get<uint64_t>();
    bi.perturbation = r.get<double>();
    bi.ell = r.get<double>();
    bi.eta = r.get<double>();
    bi.grid_order = r.get<int32_t>();
  }
  std::vector<int32_t> ranks, cranks;
  std::vector<double> leaf, transfer, cleaf, ctransfer;
  int depth;
  {
    auto buf = read_section(is);
    Reader r{buf.data(), buf.data() + buf.size()};
    auto get_basis = [&](std::vector<int32_t>& rk, std::vector<double>& lf, std::vector<double>& tr) {
      for (int k = 0; k < 4; ++k) r.get_vec<int32_t>();  // the complete binary tree is implied
      rk = r.get_vec<int32_t>();
      depth = int(rk.size()) - 1;
      require(depth >= 0 && depth < 31, "load: bad depth");
      require(r.get<int32_t>() == m, "load: leaf_dim != m");
      lf = r.get_vec<double>();
      const uint64_t nt = r.get<uint64_t>();
      require(nt == uint64_t(depth + 1), "load: transfer levels != depth + 1");
      for (uint64_t l = 0; l < nt; ++l) {
        const auto t = r.get_vec<double>();
        tr.insert(tr.end(), t.begin(), t.end());
      }
    };
    get_basis(ranks, leaf, transfer);
    if (!symmetric) {
      const int rd = depth;
      get_basis(cranks, cleaf, ctransfer);
      require(depth == rd, "load: column basis depth != row basis depth");
    }
  }
  const std::vector<int32_t>& colr = symmetric ? ranks : cranks;
  std::vector<int32_t> rp, ci;
  std::vector<double> vals;
  {
    auto buf = read_section(is);
    Reader r{buf.data(), buf.data() + buf.size()};
    const uint64_t nl = r.get<uint64_t>();
    require(nl == uint64_t(depth + 1), "load: coupling levels != depth + 1");
    for (uint64_t l = 0; l < nl; ++l) {
      LayerIn L = get_layer(r);
      require(L.brows == ranks[l] && L.bcols == colr[l], "load: coupling block dims != ranks");
      require(L.row_ptr.size() == (size_t(1) << l) + 1, "load: coupling row_ptr size");
      rp.insert(rp.end(), L.row_ptr.begin(), L.row_ptr.end());
      ci.insert(ci.end(), L.col_idx.begin(), L.col_idx.end());
      vals.insert(vals.end(), L.values.begin(), L.values.end());
    }
  }
  LayerIn D;
  {
    auto buf = read_section(is);
    Reader r{buf.data(), buf.data() + buf.size()};
    D = get_layer(r);
    require(D.brows == m && D.bcols == m, "load: dense block dims != m");
  }
  std::vector<int32_t> perm;
  {
    auto buf = read_section(is);
    Reader r{buf.data(), buf.data() + buf.size()};
    perm = r.get_vec<int32_t>();
  }
  require(n == int64_t(perm.size()), "load: perm size != n");
  h2b_matrix_desc d{};
  d.n = int32_t(n);
  d.m = m;
  d.depth = depth;
  d.symmetric = symmetric ? 1 : 0;
  d.col_ranks = symmetric ? nullptr : cranks.data();
  d.col_leaf = symmetric ? nullptr : cleaf.data();
  d.col_transfer = symmetric ? nullptr : ctransfer.data();
  d.perm = perm.data();
  d.ranks = ranks.data();
  d.leaf = leaf.data();
  d.transfer = transfer.data();
  d.cpl_row_ptr = rp.data();
  d.cpl_col_idx = ci.data();
  d.cpl_values = vals.data();
  d.dense_row_ptr = D.row_ptr.data();
  d.dense_col_idx = D.col_idx.data();
  d.dense_values = D.values.data();
  h2b_matrix* A = create_from_desc(d, device);
  A->info = bi;
  if (info_out) *info_out = bi;
  return A;
}

}  // namespace h2b
