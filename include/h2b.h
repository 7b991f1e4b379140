/*
 * h2b.h — C-ABI of the B200-native H^2-matrix hot path (libh2b.so).
 *
 * Drop-in boundary for the reference library h2kit (arXiv 1902.01829 reference,
 * /root/reference/proj).  The reference has no FFI layer of its own: its seams
 * are C++ function templates over H2Matrix<T>.  Each entry
 * point below replaces one of them; the header-only C++ shim
 * include/h2kit_b200.hpp re-exposes them under the reference's own names and
 * signatures (h2kit_b200::hmv, ::compress, ...), and INTEGRATION.md shows the
 * binding a maintainer adds.
 *
 *   h2b_hmv              <- h2kit::hmv(A, x, y, alpha, beta[, ctx])   include/h2kit/hmv.hpp:175-194
 *   h2b_hmv_multi        <- (no reference API; SPEC.md:497 non-goal) column-wise hmv
 *   h2b_upsweep          <- h2kit::upsweep(V, xc, n, xhat)            hmv.hpp:79-111
 *   h2b_tree_multiply    <- h2kit::tree_multiply(S, xhat, yhat)       hmv.hpp:114-125
 *   h2b_downsweep        <- h2kit::downsweep(U, yhat, yc, n)          hmv.hpp:129-157
 *   h2b_dense_mv         <- h2kit::block_sparse_mv(A.dense, xc, yc, alpha, beta)  bsr.hpp:79-82
 *   h2b_compress         <- h2kit::compress(A, eps)                   include/h2kit/compression.hpp:466-551
 *   h2b_orthogonalize    <- h2kit::orthogonalize_basis(A.row_basis)   compression.hpp:69-126
 *   h2b_orthogonalize_col <- h2kit::orthogonalize_basis(A.col_basis())
 *   h2b_matrix_build     <- h2kit::construct<double>(points, spec, cfg)  include/h2kit/construction.hpp:179-200
 *   h2b_matrix_create    <- (host H2Matrix<double> -> device mirror; the HmvContext analogue hmv.hpp:161-172)
 *   h2b_matrix_export    <- (device -> host H2Matrix<double> arrays, e.g. after compress)
 *   h2b_matrix_footprint <- h2kit::memory_footprint(A).total()       include/h2kit/h2_matrix.hpp:90-102
 *
 * Conventions
 *  - All scalars are FP64, all matrices column-major, index type int32
 *    (h2kit::index_t, include/h2kit/defs.hpp:15); offsets/sizes are int64.
 *  - The flat host layout ("export layout") is the reference's own pool
 *    layout concatenated over levels:
 *      perm[n]; ranks[depth+1];
 *      leaf: 2^depth blocks of m x ranks[depth]            (BasisTree::leaf_pool)
 *      transfer: for l = 1..depth, 2^l blocks of ranks[l] x ranks[l-1]  (BasisTree::transfer[l])
 *      cpl_row_ptr: for l = 0..depth, 2^l + 1 entries      (BSRLayer::row_ptr, level-local)
 *      cpl_col_idx / cpl_values: for l = 0..depth, nb_l entries / nb_l blocks of ranks[l]^2
 *      dense_row_ptr[2^depth + 1], dense_col_idx[nbd], dense_values[nbd * m * m]
 *  - Errors: every function returns an h2b_status; H2B_INVALID_ARGUMENT is
 *    the reference's std::invalid_argument (defs.hpp:20-22), with the same
 *    message text, retrievable through h2b_last_error() (thread-local).
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns H2B_NO_DEVICE.
 */
#ifndef H2B_H
#define H2B_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define H2B_API __attribute__((visibility("default")))
#else
#define H2B_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  H2B_OK = 0,
  H2B_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  H2B_CUDA_ERROR = 2,
  H2B_OUT_OF_MEMORY = 3,
  H2B_UNSUPPORTED = 4,      /* shape outside the compiled kernel envelope */
  H2B_NO_DEVICE = 5,
  H2B_INTERNAL = 6,
  H2B_IO_ERROR = 7          /* reference: h2kit::IOError (io.hpp:19-21) */
} h2b_status;

typedef enum {
  H2B_PTR_AUTO = 0,   /* detect with cudaPointerGetAttributes */
  H2B_PTR_HOST = 1,   /* host memory (pinned or pageable); copies happen inside the call */
  H2B_PTR_DEVICE = 2, /* device memory on the matrix's device */
  H2B_PTR_HOST_ASYNC = 3 /* PINNED host memory, stream-ordered: the copies are enqueued on the
                            call's stream and the call returns without synchronising; the caller
                            synchronises before reading y or rewriting x (h2b_hmv / h2b_hmv_ctx) */
} h2b_ptr_kind;

typedef struct h2b_matrix h2b_matrix;

/* Host description of an H^2 matrix in the export layout.  symmetric = 1:
 * one basis (row == column, what construct() produces).  symmetric = 0: the
 * column basis V / F (H2Matrix::col_basis_store, h2_matrix.hpp:69,75-78) is
 * given by col_ranks / col_leaf / col_transfer and coupling block (i, j) of
 * level l is ranks[l] x col_ranks[l]. */
typedef struct {
  int32_t n;          /* points; n == m * 2^depth */
  int32_t m;          /* leaf size (BasisTree::leaf_dim) */
  int32_t depth;      /* q */
  int32_t symmetric;  /* 1: column basis == row basis; 0: col_* below */
  const int32_t* perm;
  const int32_t* ranks;
  const double* leaf;
  const double* transfer;
  const int32_t* cpl_row_ptr;
  const int32_t* cpl_col_idx;
  const double* cpl_values;
  const int32_t* dense_row_ptr;
  const int32_t* dense_col_idx;
  const double* dense_values;
  const int32_t* col_ranks;     /* symmetric == 0 only (else ignored) */
  const double* col_leaf;
  const double* col_transfer;
} h2b_matrix_desc;

/* Parameters of the reference's ab-initio construction (ConstructionConfig +
 * KernelSpec + generate_perturbed_grid, construction.hpp:15-25, kernels.hpp:10-22,
 * geometry.hpp:41-45). */
typedef struct {
  int32_t dim;          /* 2 or 3 */
  int32_t n;            /* points */
  int32_t leaf_size;    /* m (64) */
  int32_t grid_order;   /* Chebyshev order per axis; rank = order^dim */
  double eta;           /* admissibility (2.0) */
  double ell;           /* correlation length of exp(-r/ell) */
  double perturbation;  /* grid jitter (0.25) */
  uint64_t seed;        /* mt19937_64 seed (1) */
} h2b_build_config;

/* BuildInfo (h2_matrix.hpp:53-60): construction parameters stored in containers. */
typedef struct {
  int32_t dim;
  uint64_t seed;
  double perturbation, ell, eta;
  int32_t grid_order;
} h2b_build_info;

/* Sizes of a matrix in the export layout. */
typedef struct {
  int32_t n, m, depth, symmetric;
  int32_t ranks[32];
  int64_t cpl_blocks[32];     /* blocks per coupling level */
  int32_t cpl_max_row[32];    /* max blocks in one block row, per level */
  int64_t dense_blocks;
  int32_t dense_max_row;
  uint64_t footprint_bytes;   /* memory_footprint(A).total(): reference byte convention */
  uint64_t device_bytes;      /* HBM actually held by the handle (pools + workspace) */
  double hmv_flops;           /* reference analytic flop model of one hmv (flops.hpp) */
  uint64_t global_footprint_bytes; /* whole matrix (== footprint_bytes unless partitioned) */
  int32_t part_log2;          /* 2^part_log2 subtree partitions (0: whole matrix) */
  int32_t part_index;         /* partition owned by this handle */
  int32_t col_ranks[32];      /* column basis ranks (== ranks when symmetric) */
} h2b_matrix_info;

/* Workspace buffers of a handle (device pointers, see h2b_workspace). */
typedef enum { H2B_WS_XHAT = 0, H2B_WS_YHAT = 1, H2B_WS_XC = 2, H2B_WS_PERM = 3 } h2b_workspace_id;

/* compress() report (CompressionReport, compression.hpp:422-441). Times are
 * device-measured (CUDA events); flops follow the reference analytic model. */
typedef struct {
  int32_t old_ranks[32];
  int32_t new_ranks[32];
  uint64_t bytes_before, bytes_after;
  double frobenius_error;
  double frobenius_norm;
  double time_orthogonalize_ms, time_project_orth_ms, time_weights_ms,
         time_truncate_ms, time_project_trunc_ms;
  double flops_orthogonalize, flops_project_orth, flops_weights,
         flops_truncate, flops_project_trunc;
} h2b_compress_report;

H2B_API const char* h2b_last_error(void);
H2B_API const char* h2b_version(void);

/* Device count visible to the library; 0 means no usable sm_100 device. */
H2B_API int h2b_device_count(void);

H2B_API h2b_status h2b_matrix_create(const h2b_matrix_desc* desc, int device, h2b_matrix** out);
H2B_API h2b_status h2b_matrix_build(const h2b_build_config* cfg, int device, h2b_matrix** out);
H2B_API h2b_status h2b_matrix_destroy(h2b_matrix* A);
H2B_API h2b_status h2b_matrix_info_get(const h2b_matrix* A, h2b_matrix_info* info);
/* Copy the device matrix into caller-allocated host arrays (export layout,
 * sizes from h2b_matrix_info_get). Any pointer may be NULL to skip it. */
H2B_API h2b_status h2b_matrix_export(const h2b_matrix* A, int32_t* perm, double* leaf, double* transfer,
                             int32_t* cpl_row_ptr, int32_t* cpl_col_idx, double* cpl_values,
                             int32_t* dense_row_ptr, int32_t* dense_col_idx, double* dense_values);
/* Column basis of a non-symmetric matrix (V leaves, F transfers; export
 * layout, sizes from col_ranks).  Symmetric matrices: H2B_INVALID_ARGUMENT. */
H2B_API h2b_status h2b_matrix_export_col(const h2b_matrix* A, double* col_leaf, double* col_transfer);
H2B_API uint64_t h2b_matrix_footprint(const h2b_matrix* A);
/* h2kit::save / h2kit::load (io.hpp:183-282): the reference's ".h2" container
 * ("H2KT" v1, FP64, CRC-32 per section), byte-compatible in both directions;
 * the pools stream straight from / into HBM.  info: BuildInfo to store (NULL:
 * the matrix's own -- set by h2b_matrix_build / h2b_matrix_load, zeros for
 * h2b_matrix_create); info_out may be NULL.  Errors: H2B_IO_ERROR with the
 * reference's messages.  Non-symmetric matrices: the column basis follows the
 * row basis in the bases section (io.hpp:194-197). */
H2B_API h2b_status h2b_matrix_save(const h2b_matrix* A, const char* path, const h2b_build_info* info);
H2B_API h2b_status h2b_matrix_load(const char* path, int device, h2b_matrix** out, h2b_build_info* info_out);
/* h2kit::crc32 (crc32.cpp:6-20, seed 0): the containers' section checksum
 * (host memory; slicing-by-8, chunk-parallel with CRC combination). */
H2B_API uint32_t h2b_crc32(const void* data, uint64_t len);

/* y <- alpha (A_D + A_LR) x + beta y, x and y in original point order.
 * beta == 0 never reads y (hmv.hpp:186). stream is a cudaStream_t (NULL =
 * the matrix's own stream). Host pointers: the call is synchronous. */
H2B_API h2b_status h2b_hmv(h2b_matrix* A, const double* x, double* y, double alpha, double beta,
                   h2b_ptr_kind kind, void* stream);
/* Per-caller workspaces: the HmvContext analogue (hmv.hpp:159-172).  The
 * reference allows concurrent hmv calls on one immutable matrix with one
 * context each; so does this library.  A context is sized lazily for the
 * matrix it is used with (and re-sized after compress changed the ranks).
 * Calls that share a context (or use none: the handle's own workspace) are
 * serialised in device order across streams, never raced. */
typedef struct h2b_context h2b_context;
H2B_API h2b_status h2b_context_create(h2b_matrix* A, h2b_context** out);
H2B_API h2b_status h2b_context_destroy(h2b_context* ctx);
/* hmv(A, x, y, alpha, beta, ctx) (hmv.hpp:175-188); ctx may be NULL. */
H2B_API h2b_status h2b_hmv_ctx(h2b_matrix* A, h2b_context* ctx, const double* x, double* y, double alpha,
                               double beta, h2b_ptr_kind kind, void* stream);

/* nvec columns, leading dimensions ldx/ldy (>= n). */
/* CUDA-graph replay of one mat-vec (for small matrices, where the launch
 * sequence costs as much as the work): y <- alpha A x + beta y on the fixed
 * DEVICE vectors x, y is captured once with the context's workspace (NULL: the
 * matrix's own) and replayed by h2b_hmv_graph_launch on any stream, stream-
 * ordered with the other users of that workspace.  A graph is tied to the
 * matrix layout it was captured for: after compress() a launch returns
 * H2B_INVALID_ARGUMENT.  Destroy graphs before their context / matrix. */
typedef struct h2b_hmv_graph h2b_hmv_graph;
H2B_API h2b_status h2b_hmv_graph_create(h2b_matrix* A, h2b_context* ctx, const double* x, double* y, double alpha,
                                        double beta, h2b_hmv_graph** out);
H2B_API h2b_status h2b_hmv_graph_launch(h2b_hmv_graph* g, void* stream);
H2B_API h2b_status h2b_hmv_graph_destroy(h2b_hmv_graph* g);
/* Y <- alpha A X + beta Y for nvec columns (column v at X + v ldx / Y + v ldy),
 * 16 columns per FP64-tensor-core pass.  Host pointers: synchronous; device
 * pointers: stream-ordered on `stream` (NULL = the matrix's own stream). */
H2B_API h2b_status h2b_hmv_multi(h2b_matrix* A, int nvec, const double* X, int64_t ldx, double* Y,
                         int64_t ldy, double alpha, double beta, h2b_ptr_kind kind, void* stream);

/* Phase entry points (device or host pointers, cluster order; node vectors
 * are level-concatenated: level l holds 2^l * ranks[l] doubles). */
H2B_API h2b_status h2b_upsweep(h2b_matrix* A, const double* xc, double* xhat, h2b_ptr_kind kind);
H2B_API h2b_status h2b_tree_multiply(h2b_matrix* A, const double* xhat, double* yhat, h2b_ptr_kind kind);
/* yhat is in/out like the reference's LevelVectors (y^l += E y^{l-1}); yc += U y^q. */
H2B_API h2b_status h2b_downsweep(h2b_matrix* A, double* yhat, double* yc, h2b_ptr_kind kind);
H2B_API h2b_status h2b_dense_mv(h2b_matrix* A, const double* xc, double* yc, double alpha, double beta,
                        h2b_ptr_kind kind);

/* Algebraic recompression in place (orthogonalize, project, weights,
 * truncate at relative eps, project).  Exclusive access required. */
/* Non-symmetric matrices (a separate column basis) are supported by every
 * entry point; h2b_orthogonalize works on the row basis, h2b_orthogonalize_col
 * on the column basis. */
H2B_API h2b_status h2b_compress(h2b_matrix* A, double eps, h2b_compress_report* report);
/* Orthogonalize only (in place); projection tree written to t_out (host,
 * level-concatenated ranks[l]^2 per node) when non-NULL. */
H2B_API h2b_status h2b_orthogonalize(h2b_matrix* A, double* t_out);
/* orthogonalize_basis(A.col_basis()) (compression.hpp:69-126, h2_matrix.hpp:75-78):
 * the column basis of a non-symmetric matrix (t_out: col_ranks[l]^2 per node);
 * on a symmetric matrix the same as h2b_orthogonalize. */
H2B_API h2b_status h2b_orthogonalize_col(h2b_matrix* A, double* t_out);
/* compress() keeps its device workspace (projection / weight trees and
 * scratch, a few GB) cached per device for the next call; this frees it. */
H2B_API h2b_status h2b_release_cached_memory(int device);

/* validate_sampled (validate.hpp:26-62) on the device: relative mat-vec error
 * against the exact kernel exp(-|p_i - p_j|/ell) on ceil(fraction n) sampled
 * rows, x = random_vector(n, seed).  points: n x dim, original order (NULL:
 * the points h2b_matrix_build generated; dim/ell <= 0 then mean "stored"). */
H2B_API h2b_status h2b_validate_sampled(h2b_matrix* A, const double* points, int dim, double ell,
                                        double fraction, uint64_t seed, double* err);

/* ---- subtree-partitioned multi-GPU mat-vec ----
 * nparts = 2^s GPUs; partition `part` owns the leaves [part n/nparts, (part+1) n/nparts)
 * in cluster order, the basis nodes and coupling/dense block rows of its top-level
 * subtree at levels >= s; levels < s (and the transfers up to level s) are
 * replicated.  One mat-vec on every rank:
 *   h2b_part_upsweep(A, x)           x: full x (original order, device)
 *   all-gather x^ at levels >= s     (caller: NCCL; the owned slice of level l is
 *                                     nodes [part 2^(l-s), (part+1) 2^(l-s)) of the
 *                                     H2B_WS_XHAT buffer, level-concatenated)
 *   h2b_part_finish(A, y_slice)      y_slice: n/nparts doubles, cluster order
 *   all-gather y_slice; y[perm[t]] = alpha y_cluster[t] + beta y[perm[t]]. */
H2B_API h2b_status h2b_matrix_build_part(const h2b_build_config* cfg, int device, int nparts,
                                         int part, h2b_matrix** out);
/* Device pointer + element count of a workspace buffer (double, PERM: int32). */
H2B_API h2b_status h2b_workspace(h2b_matrix* A, int which, void** ptr, int64_t* count);
H2B_API h2b_status h2b_part_upsweep(h2b_matrix* A, const double* x, void* stream);
H2B_API h2b_status h2b_part_finish(h2b_matrix* A, double* y_slice, void* stream);

/* ---- one-call partitioned mat-vec, driven from the host through a
 * stream-ordered device communicator (NCCL) ----
 * allgather: enqueue on `stream` the in-place all-gather of buf, which holds
 * nparts slices of `count` doubles, slice `part` this rank's; with NCCL:
 *   ncclAllGather(buf + part * count, buf, count, ncclDouble, comm, (cudaStream_t)stream)
 * Return 0 once enqueued (no host synchronisation is needed). */
typedef struct h2b_dcomm {
  void* ctx;
  int (*allgather)(void* ctx, double* buf, int64_t count, void* stream);
} h2b_dcomm;
typedef enum {
  H2B_Y_REPLICATED = 0, /* y complete on every rank (cluster-order slices all-gathered, then scattered) */
  H2B_Y_OWNED = 1       /* each rank writes only its own rows y[perm[t]], t in its cluster-order range */
} h2b_y_mode;
/* y <- alpha A x + beta y on every rank of a partitioned matrix (x: full,
 * original order, device; y device).  Per call: one x^ all-gather (every level
 * >= s packed into one buffer) and, for H2B_Y_REPLICATED, one y all-gather;
 * comm may be NULL for a single partition.  Every kernel is in libh2b.so
 * (pack / unpack, the owner-row scatter); nothing is computed on the host. */
H2B_API h2b_status h2b_part_hmv(h2b_matrix* A, const double* x, double* y, double alpha, double beta, int y_mode,
                                const h2b_dcomm* comm, void* stream);
/* nvec right-hand sides (X, Y: n x nvec column-major, device), 16 per pass on
 * the FP64 tensor cores; one x^ all-gather (and one y all-gather) per pass. */
H2B_API h2b_status h2b_part_hmv_multi(h2b_matrix* A, int nvec, const double* X, int64_t ldx, double* Y,
                                      int64_t ldy, double alpha, double beta, int y_mode, const h2b_dcomm* comm,
                                      void* stream);

/* ---- subtree-partitioned compression (compression.hpp:466-551 on 2^s GPUs) ----
 * Every rank calls h2b_part_compress on its partition handle with the same eps;
 * the library runs the phases on the rank's subtree and calls back into the
 * host communicator at fixed points (same order on every rank):
 *   allgather   in place on DEVICE memory: buf holds nparts slices of `count`
 *               doubles, slice `part` is this rank's (NCCL all-gather); used for
 *               the projection trees T of the levels >= s (orthogonalisation and
 *               truncation) -- remote column bases of the coupling blocks;
 *   allreduce_max_i32 / allreduce_sum_f64   element-wise on HOST memory: the
 *               per-level truncated rank (compression.hpp:301,375), the
 *               non-finite flag, ||A||_F^2 and the discarded energy.
 * Levels < s are computed redundantly on every rank.  Callbacks return 0 on
 * success.  The report is global (identical on every rank). */
typedef struct h2b_comm {
  void* ctx;
  int (*allgather)(void* ctx, double* buf, int64_t count);
  int (*allreduce_max_i32)(void* ctx, int32_t* v, int n);
  int (*allreduce_sum_f64)(void* ctx, double* v, int n);
} h2b_comm;
H2B_API h2b_status h2b_part_compress(h2b_matrix* A, double eps, const h2b_comm* comm,
                                     h2b_compress_report* report);

/* ---- the reference's component objects and the phase API ----
 * BasisTree<double> (h2_matrix.hpp:17-41), MatrixTree<double> (:46-51) and
 * BSRLayer<double> (bsr.hpp:13-31) as device handles, and the reference
 * functions that take them:
 *   h2b_basis_upsweep         <- upsweep(V, x, n, xhat)              hmv.hpp:79-111
 *   h2b_basis_downsweep       <- downsweep(U, yhat, y, n)            hmv.hpp:129-157
 *   h2b_mtree_multiply        <- tree_multiply(S, xhat, yhat)        hmv.hpp:114-125
 *   h2b_block_sparse_mv       <- block_sparse_mv(L, x, y, alpha, beta)  bsr.hpp:79-82
 *   h2b_orthogonalize_basis   <- orthogonalize_basis(B) -> ProjectionTree  compression.hpp:69-126
 *   h2b_project_coupling      <- project_coupling(Trow, Tcol, S)     compression.hpp:130-169
 *   h2b_generate_weight_tree  <- generate_weight_tree(B, S) -> WeightTree  compression.hpp:213-256
 *   h2b_truncate_basis        <- truncate_basis(B, R, eps, Tout) -> TruncationResult  compression.hpp:267-420
 * Trees (ProjectionTree / WeightTree) cross as the reference's per-level pools
 * concatenated over levels: rows[l] x cols[l] per node, column-major, node i
 * of level l at offset i rows[l] cols[l] within the level.  Node vectors
 * (LevelVectors) likewise.  Vectors and trees may be host or device memory. */
typedef struct h2b_basis h2b_basis;
typedef struct h2b_mtree h2b_mtree;
typedef struct h2b_layer h2b_layer;

typedef struct {
  int32_t m;                /* BasisTree::leaf_dim */
  int32_t depth;            /* q */
  const int32_t* ranks;     /* depth + 1 */
  const double* leaf;       /* 2^depth blocks of m x ranks[depth] */
  const double* transfer;   /* l = 1..depth: 2^l blocks of ranks[l] x ranks[l-1] */
} h2b_basis_desc;

typedef struct {
  int32_t block_rows, block_cols;  /* BSRLayer::block_rows / block_cols */
  int32_t brows, bcols;            /* block shape */
  const int32_t* row_ptr;          /* block_rows + 1 */
  const int32_t* col_idx;          /* row_ptr[block_rows] */
  const double* values;            /* blocks in col_idx order, column-major */
} h2b_layer_desc;

H2B_API h2b_status h2b_basis_create(const h2b_basis_desc* desc, int device, h2b_basis** out);
H2B_API h2b_status h2b_basis_destroy(h2b_basis* B);
/* leaf size, depth, ranks (depth + 1 entries); any pointer may be NULL */
H2B_API h2b_status h2b_basis_shape(const h2b_basis* B, int32_t* m, int32_t* depth, int32_t* ranks);
H2B_API h2b_status h2b_basis_export(const h2b_basis* B, double* leaf, double* transfer);
H2B_API h2b_status h2b_basis_upsweep(h2b_basis* V, const double* x, int64_t n, double* xhat, h2b_ptr_kind kind);
H2B_API h2b_status h2b_basis_downsweep(h2b_basis* U, double* yhat, double* y, int64_t n, h2b_ptr_kind kind);
/* B orthogonalized in place; t_out (may be NULL): T, ranks[l]^2 per node. */
H2B_API h2b_status h2b_orthogonalize_basis(h2b_basis* B, double* t_out);
/* B truncated in place.  r_tree: R (ranks[l]^2 per node); t_out: Tout,
 * new_ranks[l] x old ranks[l] per node (capacity old ranks[l]^2 per node);
 * new_ranks / discarded_energy: TruncationResult, depth + 1 each.  NULLs skip. */
H2B_API h2b_status h2b_truncate_basis(h2b_basis* B, const double* r_tree, double eps, double* t_out,
                                      int32_t* new_ranks, double* discarded_energy);

H2B_API h2b_status h2b_layer_create(const h2b_layer_desc* desc, int device, h2b_layer** out);
H2B_API h2b_status h2b_layer_destroy(h2b_layer* L);
/* y <- alpha L x + beta y in the reference's exact arithmetic (bitwise equal). */
H2B_API h2b_status h2b_block_sparse_mv(h2b_layer* L, const double* x, double* y, double alpha, double beta,
                                       h2b_ptr_kind kind);

/* MatrixTree: nlevels layers, level l with block_rows = block_cols = 2^l. */
H2B_API h2b_status h2b_mtree_create(int32_t nlevels, const h2b_layer_desc* levels, int device, h2b_mtree** out);
H2B_API h2b_status h2b_mtree_destroy(h2b_mtree* S);
H2B_API h2b_status h2b_mtree_shape(const h2b_mtree* S, int32_t* brows, int32_t* bcols, int64_t* nblocks);
H2B_API h2b_status h2b_mtree_export(const h2b_mtree* S, double* values);
/* xhat: 2^l bcols[l] per level; yhat: 2^l brows[l] per level. */
H2B_API h2b_status h2b_mtree_multiply(h2b_mtree* S, const double* xhat, double* yhat, h2b_ptr_kind kind);
/* tcol == NULL: the column tree is trow (project_coupling(T, T, S)). */
H2B_API h2b_status h2b_project_coupling(const double* trow, const int32_t* trow_rows, const int32_t* trow_cols,
                                        const double* tcol, const int32_t* tcol_rows, const int32_t* tcol_cols,
                                        h2b_mtree* S);
/* r_out: R, ranks[l]^2 per node (R^0 = 0). */
H2B_API h2b_status h2b_generate_weight_tree(h2b_basis* B, h2b_mtree* S, double* r_out);

/* Per-phase device time of the h2b_hmv calls made since phase timing was
 * enabled or last read, averaged per call (ms; CUDA events recorded on the
 * launching stream, no host syncs inside h2b_hmv):
 * [0]=upsweep [1]=coupling+dense BSR [2]=downsweep+scatter [3]=total.  Resets. */
H2B_API h2b_status h2b_last_hmv_timing(h2b_matrix* A, double* ms4);
/* Enable/disable per-phase event timing inside h2b_hmv (default off). */
H2B_API h2b_status h2b_set_phase_timing(h2b_matrix* A, int on);

#ifdef __cplusplus
}
#endif
#endif /* H2B_H */
