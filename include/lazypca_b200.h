/* lazypca_b200 — C ABI of the B200-native Lazy SPCA / SPCA / RP reducer.
 *
 * Drop-in boundary for the reference C++ library `lazypca` (namespace lazypca,
 * headers proj/core/include/lazypca/*.hpp, CMake target lazypca::core). Every
 * entry point below names the reference interface it replaces; the header-only
 * C++ shim include/lazypca_b200.hpp rebuilds the reference's value types and
 * exception classes on top of these calls so existing callers relink unchanged.
 *
 * Conventions
 *  - Plain pointers and sizes; no torch / CUDA types in any signature (streams
 *    are passed as void*; NCCL unique ids as 128 opaque bytes).
 *  - Matrices are described by lpca_matrix_view. Dense data may be row- or
 *    column-major, fp32 or fp64, and live on the host or on the context's device.
 *    CSC views (the reference's SparseMatrix) below 25% density stay sparse on
 *    the device (CSR and CSC gathers in the reference's summation order);
 *    denser ones are densified for the tensor-core passes.
 *  - Every call returns an lpca_status. Non-zero codes mirror the reference's
 *    exception hierarchy (proj/core/include/lazypca/error.hpp:10-58); the message
 *    and payload (index / last_gap / line) are available per thread through
 *    lpca_last_error*().
 *  - A context is bound to one device (one process per GPU). Calls on one
 *    context are serialised by the caller; separate contexts are independent.
 *  - There is no CPU fallback: if no sm_100 device is present every compute
 *    entry point fails with LPCA_ERR_CUDA.
 */
#ifndef LAZYPCA_B200_H
#define LAZYPCA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LPCA_ABI_VERSION 1

typedef enum {
  LPCA_OK = 0,
  LPCA_ERR_DIMENSION = 1,          /* lazypca::DimensionError */
  LPCA_ERR_INVALID_ARGUMENT = 2,   /* lazypca::InvalidArgumentError */
  LPCA_ERR_RANK_DEFICIENCY = 3,    /* lazypca::RankDeficiencyError(index) */
  LPCA_ERR_CONVERGENCE = 4,        /* lazypca::ConvergenceError(last_gap) */
  LPCA_ERR_PARSE = 5,              /* lazypca::ParseError(line) */
  LPCA_ERR_CUDA = 6,               /* device / driver failure (no reference analogue) */
  LPCA_ERR_NCCL = 7,               /* collective failure (no reference analogue) */
  LPCA_ERR_INTERNAL = 9
} lpca_status;

/* lazypca::ReducerMethod (proj/core/include/lazypca/reducer.hpp:12) */
typedef enum { LPCA_RP = 0, LPCA_SPCA = 1, LPCA_LAZY_SPCA = 2 } lpca_method;
/* lazypca::ProjectionKind (proj/core/include/lazypca/projection.hpp:12) */
typedef enum { LPCA_GAUSSIAN = 0, LPCA_VERY_SPARSE = 1 } lpca_projection_kind;
/* lazypca::DensityPolicy::Mode (proj/core/include/lazypca/projection.hpp:17-21) */
typedef enum { LPCA_DENSITY_AGGRESSIVE = 0, LPCA_DENSITY_CONSERVATIVE = 1, LPCA_DENSITY_EXPLICIT = 2 } lpca_density_mode;

typedef enum { LPCA_F32 = 4, LPCA_F64 = 8 } lpca_dtype;
typedef enum { LPCA_HOST = 0, LPCA_DEVICE = 1 } lpca_location;
typedef enum { LPCA_ROW_MAJOR = 0, LPCA_COL_MAJOR = 1, LPCA_CSC = 2 } lpca_layout;

/* A matrix argument. Dense: data + ld (elements between consecutive rows for
 * row-major, between consecutive columns for column-major; 0 = packed).
 * CSC (lazypca::SparseMatrix, proj/core/include/lazypca/sparse_matrix.hpp:17-49):
 * col_ptr (cols+1), row_idx (nnz), values (nnz, dtype) — host memory only. */
typedef struct {
  int32_t dtype;      /* lpca_dtype */
  int32_t layout;     /* lpca_layout */
  int32_t location;   /* lpca_location */
  int32_t reserved;
  int64_t rows, cols, ld;
  const void* data;
  const int64_t* col_ptr;
  const int64_t* row_idx;
  int64_t nnz;
} lpca_matrix_view;

/* lazypca::ReducerConfig + nested ProjectionSpec
 * (proj/core/include/lazypca/reducer.hpp:20-33, projection.hpp:36-45). */
typedef struct {
  int32_t method;          /* lpca_method */
  int32_t projection_kind; /* lpca_projection_kind */
  int64_t k;
  int64_t l;               /* 0 = same as k */
  int64_t proj_n;          /* ProjectionSpec::n, 0 = from the data */
  int64_t proj_l;          /* ProjectionSpec::l, 0 = l */
  double density;          /* ProjectionSpec::density, in (0, 1] */
  uint64_t seed;           /* ProjectionSpec::seed */
  int64_t block_rows;      /* > 0 selects the streaming variants */
  int32_t streaming;
  int32_t deterministic;   /* accepted for manifest compatibility */
  int32_t power_iters;     /* q >= 0. Builder extension, NOT in the reference
                              (SPEC.md:371): q subspace steps Z = X^T U,
                              Z <- orth(Z), U = X Z before F is formed. */
  int32_t reserved;
} lpca_config;

/* lazypca::ReducerTimings (proj/core/include/lazypca/reducer.hpp:59-66),
 * seconds, device-event timed; `power` and `transform` are extensions, and the
 * *_pass fields time the X-pass kernel alone inside its phase (sketch U = X Omega,
 * F = U^T X, Y = X V), without operand preparation or partial-sum reduction. */
typedef struct {
  double sketch, qr, f_form, svd, total;
  double power, transform, h2d, d2h;
  double sketch_pass, f_pass, transform_pass;
  double power_pass; /* the power steps' X-pass kernels (Z = X^T U and U = X Z), first 8 steps */
} lpca_timings;

typedef struct lpca_ctx lpca_ctx;
typedef struct lpca_map lpca_map; /* device-resident lazypca::ReductionMap */

/* ---- errors ------------------------------------------------------------- */
const char* lpca_last_error(void);
int64_t lpca_last_error_index(void);   /* RankDeficiencyError::index / ParseError::line, -1 if n/a */
double lpca_last_error_gap(void);      /* ConvergenceError::last_gap */
int32_t lpca_abi_version(void);

/* ---- contexts (one per GPU) --------------------------------------------- */
lpca_status lpca_ctx_create(int32_t device, lpca_ctx** out);
/* Row-sharded data parallelism over NCCL: `rank` of `world`, all ranks pass the
 * same 128-byte id from lpca_nccl_unique_id on rank 0. world == 1 needs no id;
 * world == 1 with an id makes a one-rank communicator whose exchanges still run
 * through ncclAllReduce (the NCCL path exercised on one GPU). */
lpca_status lpca_nccl_unique_id(void* out_128_bytes);
lpca_status lpca_ctx_create_dist(int32_t device, int32_t rank, int32_t world,
                                 const void* nccl_id_128, lpca_ctx** out);
/* Row-sharded data parallelism over a caller's collective instead of NCCL (e.g.
 * an MPI or gloo allreduce, or several ranks sharing one device in tests): the
 * library calls fn(user, data, count, stream) for every exchange, where data is
 * `count` fp64 values in device memory of this context's device; fn must leave
 * their sum over all ranks in place, ordered after the work already enqueued on
 * `stream` (a cudaStream_t) and before anything enqueued after it returns (a
 * synchronous implementation may synchronise the stream first). Non-zero return
 * = failure (LPCA_ERR_NCCL). Every rank issues the same sequence of calls. */
typedef int32_t (*lpca_allreduce_fn)(void* user, double* data, int64_t count, void* cuda_stream);
lpca_status lpca_ctx_create_hooked(int32_t device, int32_t rank, int32_t world, lpca_allreduce_fn fn, void* user,
                                   lpca_ctx** out);
lpca_status lpca_ctx_destroy(lpca_ctx* ctx);
/* Launch everything on this cudaStream_t (default: the context's own stream). */
lpca_status lpca_ctx_set_stream(lpca_ctx* ctx, void* cuda_stream);
lpca_status lpca_ctx_synchronize(lpca_ctx* ctx);
/* Kernel-path switch for A/B measurements: 0 = tcgen05 split-TF32 (fp32 data,
 * default), 1 = SIMT FFMA/DFMA. Both are native sm_100a code. */
lpca_status lpca_ctx_set_gemm_path(lpca_ctx* ctx, int32_t path);
/* 1 = fp64 kernels use the reference's summation order (separate multiply and
 * add, no split-K): results bitwise equal to the reference's spmm / gemm_t /
 * dense_aat; slower. Kernel-level exports always run in this mode. */
lpca_status lpca_ctx_set_exact_order(lpca_ctx* ctx, int32_t exact);
/* Number of kernels this context launched since creation (bench evidence). */
int64_t lpca_ctx_launch_count(const lpca_ctx* ctx);
/* Debugging aid, with LPCA_WS_GUARD=1 in the environment: every workspace the
 * context allocates is followed by a 1 MB pattern band; this synchronises and
 * returns how many bands were overwritten (names, space-separated, into
 * `names`), or -1 when guards are off, -2 on a CUDA error. */
int64_t lpca_debug_check_guards(lpca_ctx* ctx, char* names, int64_t capacity);
/* Debugging aid (host only, no device): the row gather's entry schedule for a
 * very sparse Omega given as column lists (cols[c * cap + i] = j | sign << 31,
 * cnt[c] entries): out receives [warp][smax / 2][32] words of two 16-bit
 * entries (word index | sign << 15; idle lanes read zero words at index
 * round_up(n, 32) + bank); warp = part * ceil(l / 32) + column group, where a
 * row's entries are split by j into *splits parts. Returns the longest warp
 * schedule (steps), or -1 if infeasible or out_capacity is short (*smax = the
 * steps the kernel unrolls, *splits = 1 or 2; both 0 on failure). */
int32_t lpca_debug_row_schedule(const int32_t* cnt, const uint32_t* cols, int32_t cap, int64_t n, int64_t l,
                                uint32_t* out, int64_t out_capacity, int32_t* smax, int32_t* splits);

/* ---- configuration ------------------------------------------------------ */
/* ReducerConfig::resolved (proj/core/src/reducer.cpp:137-161). */
lpca_status lpca_config_resolve(const lpca_config* in, int64_t data_cols, lpca_config* out);
/* density_for (proj/core/src/projection.cpp:38-50). */
lpca_status lpca_density_for(int32_t mode, int64_t k, double value, double* out);

/* ---- projection --------------------------------------------------------- */
/* regenerate / gen_gaussian / gen_very_sparse (proj/core/src/projection.cpp:71-130)
 * Writes Omega dense column-major n x l (fp64; very sparse -> entries in
 * {-1,0,+1}, unscaled) to `out` (host or device per `out_location`) and the
 * variance constant c to *scale. Generated on the device. */
lpca_status lpca_regenerate(lpca_ctx* ctx, int32_t kind, int64_t n, int64_t l, double density,
                            uint64_t seed, void* out, int32_t out_location, double* scale);

/* ---- reducers ----------------------------------------------------------- */
/* reduce (proj/core/src/reducer.cpp:337-346) and, by method,
 * reduce_rp / reduce_spca / reduce_lazy_spca (:171-234). For a distributed
 * context X is this rank's row shard; the returned map is identical on all ranks. */
lpca_status lpca_fit(lpca_ctx* ctx, const lpca_config* cfg, const lpca_matrix_view* x,
                     lpca_map** out_map, lpca_timings* timings);
/* Streaming reducers (reduce_{spca,lazy_spca}_streaming, reducer.cpp:236-335;
 * RowBlockStream::next, sparse_matrix.hpp:58-65). The callback fills *block
 * with the next row block (any supported layout, host or device) and its
 * slice index and returns 1, returns 0 at the end of the stream, or a negative
 * value to abort (LPCA_ERR_INVALID_ARGUMENT). The block's memory must stay valid
 * until the next call. Slices must arrive as 0, 1, 2, ... and every block must
 * have the projection's width. Host row-major blocks are copied on a second
 * stream while the previous block is reduced. method rp reads only the first
 * block's width; power_iters must be 0 (one pass over the data). lpca_fit with
 * block_rows > 0 runs the same reducer over row slices of X, as reduce() does. */
typedef int32_t (*lpca_next_block_fn)(void* user, lpca_matrix_view* block, int64_t* slice_index);
lpca_status lpca_fit_stream(lpca_ctx* ctx, const lpca_config* cfg, lpca_next_block_fn next, void* user,
                            lpca_map** out_map, lpca_timings* timings);
/* apply_map (proj/core/src/reducer.cpp:348-353): Y = X V, m x k.
 * y_layout row- or column-major (the reference returns column-major), ldy 0 = packed. */
lpca_status lpca_transform(lpca_ctx* ctx, const lpca_map* map, const lpca_matrix_view* x,
                           void* y, int32_t y_dtype, int32_t y_layout, int32_t y_location,
                           int64_t ldy, lpca_timings* timings);
/* fit followed by transform of the same X, uploading a host X once. */
lpca_status lpca_fit_transform(lpca_ctx* ctx, const lpca_config* cfg, const lpca_matrix_view* x,
                               lpca_map** out_map, void* y, int32_t y_dtype, int32_t y_layout,
                               int32_t y_location, int64_t ldy, lpca_timings* timings);

/* ---- maps (lazypca::ReductionMap, proj/core/include/lazypca/reducer.hpp:47-57) */
typedef struct {
  int32_t method;
  int32_t reserved;
  int64_t k, l, n;
  uint64_t seed;
  double density;
  double scale;
  int32_t has_singular_values;
  int32_t reserved2;
} lpca_map_info;
lpca_status lpca_map_info_get(const lpca_map* map, lpca_map_info* out);
/* V: n x k column-major fp64; sigma: k fp64 (only when has_singular_values). */
lpca_status lpca_map_copy_v(const lpca_map* map, double* v_out, int32_t out_location);
lpca_status lpca_map_copy_sigma(const lpca_map* map, double* sigma_out);
/* A map from host data (e.g. a loaded map file) for lpca_transform. */
lpca_status lpca_map_create(lpca_ctx* ctx, const lpca_map_info* info, const double* v_host,
                            const double* sigma_host, lpca_map** out);
lpca_status lpca_map_destroy(lpca_map* map);
/* Map files, byte-compatible with the reference's save_map / load_map
 * (reducer.cpp:355-412): a one-line JSON header, then V as a dense
 * MatrixMarket array. lpca_map_save / lpca_map_load move a device map through a
 * file; the lpca_map_file_* pair works on host arrays and needs no GPU
 * (lpca_map_file_read with v_host == NULL fills only *info). Errors: ParseError
 * (with the line) for malformed files, DimensionError for shape mismatches. */
lpca_status lpca_map_save(const lpca_map* map, const char* path);
lpca_status lpca_map_load(lpca_ctx* ctx, const char* path, lpca_map** out);
lpca_status lpca_map_file_write(const char* path, const lpca_map_info* info, const double* v_host,
                                const double* sigma_host);
lpca_status lpca_map_file_read(const char* path, lpca_map_info* info, double* v_host, int64_t v_capacity,
                               double* sigma_host);

/* ---- matrix files (proj/core/src/matrix_io.cpp, matrix_io.hpp:1-80) ----------
 * read_sparse_matrix_market / read_dense_matrix_market / read_dense_csv with the
 * reference's rules (banner checks, 1-based coordinates with duplicates summed
 * and zeros dropped into the canonical CSC, non-finite values rejected) and its
 * ParseError messages and line numbers; the write_* functions produce the
 * reference's bytes (shortest round-trip values). A parsed file is held on the
 * host: query its shape, copy it out, or view it for lpca_fit/lpca_transform. */
typedef struct lpca_matrix_file lpca_matrix_file;
lpca_status lpca_read_sparse_matrix_market(const char* path, lpca_matrix_file** out);
lpca_status lpca_read_dense_matrix_market(const char* path, lpca_matrix_file** out);
lpca_status lpca_read_dense_csv(const char* path, lpca_matrix_file** out);
/* nnz = -1 for a dense file */
lpca_status lpca_matrix_file_info(const lpca_matrix_file* f, int64_t* rows, int64_t* cols, int64_t* nnz);
/* sparse: CSC col_ptr (cols+1), row_idx, values (nnz); dense: column-major values (rows*cols) */
lpca_status lpca_matrix_file_copy(const lpca_matrix_file* f, int64_t* col_ptr, int64_t* row_idx, double* values);
lpca_status lpca_matrix_file_view(const lpca_matrix_file* f, lpca_matrix_view* out);
void lpca_matrix_file_free(lpca_matrix_file* f);
lpca_status lpca_write_sparse_matrix_market(const char* path, int64_t rows, int64_t cols, const int64_t* col_ptr,
                                            const int64_t* row_idx, const double* values);
lpca_status lpca_write_dense_matrix_market(const char* path, int64_t rows, int64_t cols, const double* colmajor);
lpca_status lpca_write_dense_csv(const char* path, int64_t rows, int64_t cols, const double* colmajor);
/* Row-block streams from files (MatrixMarketRowBlockStream / CsvRowBlockStream,
 * matrix_io.cpp:313-443): pass lpca_file_stream_next and the stream as `next` and
 * `user` to lpca_fit_stream. MatrixMarket blocks are CSC (a counting pass at
 * open, one scan per block, one block resident); CSV blocks are dense row-major
 * fp64. A parse error inside next() aborts the fit with that ParseError. */
typedef struct lpca_file_stream lpca_file_stream;
lpca_status lpca_open_matrix_market_stream(const char* path, int64_t block_rows, lpca_file_stream** out);
lpca_status lpca_open_csv_stream(const char* path, int64_t block_rows, lpca_file_stream** out);
int32_t lpca_file_stream_next(void* stream, lpca_matrix_view* block, int64_t* slice_index);
void lpca_file_stream_close(lpca_file_stream* s);

/* ---- verification metrics on the device (proj/core/src/metrics.cpp) --------
 * chordal_distance (:123-136): n x k1 and n x k2 column-major orthonormal bases;
 * InvalidArgumentError if either is not orthonormal to 1e-8 * k. */
lpca_status lpca_chordal_distance(lpca_ctx* ctx, const double* v1, int64_t n1, int64_t k1, const double* v2,
                                  int64_t n2, int64_t k2, int32_t location, double* out);
/* distance_preservation (:311-352): all row pairs when there are at most
 * max_pairs of them, else max_pairs pairs drawn like the reference (seeded
 * xoshiro256**, with replacement). Per-pair arrays (capacity max_pairs, or the
 * pair count) may be NULL; map_b may be NULL. */
lpca_status lpca_distance_preservation(lpca_ctx* ctx, const lpca_matrix_view* x, const lpca_map* map_a,
                                       const lpca_map* map_b, int64_t max_pairs, uint64_t seed, int64_t* n_pairs,
                                       int64_t* pair_i, int64_t* pair_j, double* original, double* reduced_a,
                                       double* reduced_b, double* max_violation, double* max_discrepancy);

/* Residual norms of a projection (metrics.cpp:148-308, metrics.hpp:31-50).
 * reconstruction_error: X - P X for P the projector onto range(U), U the m x l
 * sketch (column-major fp64, host or device). route LPCA_ROUTE_QR uses an
 * orthonormal basis of U (the reference's householder_qr; here shifted
 * CholeskyQR3, equal up to roundoff), LPCA_ROUTE_LAZY the Cholesky of U^T U
 * (RankDeficiencyError with the pivot index when it is not positive definite).
 * The Frobenius error uses ||X||_F^2 - ||P X||_F^2; the spectral error runs the
 * reference's power iteration (seeded start vector, relative 1e-8, abs_tol
 * 1e-14 ||X||_F, ConvergenceError after 10000 steps). With with_bound, l >= k + 2
 * and max(m, n) <= densify_limit, sigma_{k+1} of X and bound_value are attached
 * (sigma from the eigenvalues of the smaller Gram of X, not a Jacobi SVD).
 * row_space_reconstruction_error: X - X V V^T for an orthonormal V (n x k). */
typedef enum { LPCA_ROUTE_QR = 0, LPCA_ROUTE_LAZY = 1 } lpca_residual_route;
typedef struct {
  double spectral_error;
  double frobenius_error;
  int32_t has_sigma_k_plus_1;
  int32_t has_bound;
  double sigma_k_plus_1;
  double bound;
} lpca_recon_report;
lpca_status lpca_reconstruction_error(lpca_ctx* ctx, const lpca_matrix_view* x, const double* u, int64_t u_rows,
                                      int64_t u_cols, int32_t u_location, int32_t route, int64_t k, int64_t l,
                                      int32_t with_bound, int64_t densify_limit, lpca_recon_report* out);
lpca_status lpca_row_space_reconstruction_error(lpca_ctx* ctx, const lpca_matrix_view* x, const double* v,
                                                int64_t v_rows, int64_t v_cols, int32_t v_location,
                                                lpca_recon_report* out);
/* spectral_norm(SparseMatrix / DenseMatrix) (spectral_norm.cpp:23-77): the largest
 * singular value of X by the same power iteration (no abs_tol). */
lpca_status lpca_spectral_norm(lpca_ctx* ctx, const lpca_matrix_view* x, double* out);
/* bound_value (metrics.cpp:136-146): [1 + 4 sqrt(l) / (l - k - 1) sqrt(min(m, n))] sigma;
 * InvalidArgumentError unless l >= k + 2. Host arithmetic only. */
lpca_status lpca_bound_value(int64_t m, int64_t n, int64_t k, int64_t l, double sigma_k_plus_1, double* out);

/* ---- kernel-level exports (proj/core/include/lazypca/kernels.hpp:17-36,
 *      truncated_svd.hpp:24, tridiag_eigh.hpp:8). Host or device operands; fp64
 *      column-major unless stated; X views as above. ------------------------- */
/* spmm(X, W): out m x w column-major fp64 (the sketch U = X Omega / apply). */
lpca_status lpca_spmm(lpca_ctx* ctx, const lpca_matrix_view* x, const double* w, int64_t w_cols,
                      int32_t w_location, double* out, int32_t out_location);
/* gemm_t(U, X): U m x l column-major fp64, out l x n column-major fp64. */
lpca_status lpca_gemm_t(lpca_ctx* ctx, const double* u, int64_t m, int64_t l, int32_t u_location,
                        const lpca_matrix_view* x, double* out, int32_t out_location);
/* dense_aat(F): F l x n, out l x l, bitwise symmetric. */
lpca_status lpca_dense_aat(lpca_ctx* ctx, const double* f, int64_t l, int64_t n,
                           int32_t location, double* out);
/* Symmetric eigendecomposition, eigenvalues descending, eigenvectors column-major.
 * lpca_eigh replaces tridiag_eigh (tridiag_eigh.hpp:8): Householder tridiagonalisation,
 * multisection eigenvalues, inverse-iteration eigenvectors, back-transformation.
 * lpca_eigh_jacobi replaces the cross-check jacobi_eigh (jacobi.hpp:14): parallel
 * cyclic Jacobi with the reference's schedule and stopping rule. */
lpca_status lpca_eigh(lpca_ctx* ctx, const double* a, int64_t l, int32_t location, double* evals,
                      double* evecs);
lpca_status lpca_eigh_jacobi(lpca_ctx* ctx, const double* a, int64_t l, int32_t location, double* evals,
                             double* evecs);
/* Eigensolver used by the fit's l x l step: 0 = tridiagonal route (default), 1 = Jacobi. */
lpca_status lpca_ctx_set_eigensolver(lpca_ctx* ctx, int32_t method);
/* truncated_svd_via_gram(F, k): sigma (k), v (n x k), u_tilde (l x k, may be NULL). */
lpca_status lpca_truncated_svd_via_gram(lpca_ctx* ctx, const double* f, int64_t l, int64_t n,
                                        int64_t k, int32_t location, double* sigma, double* v,
                                        double* u_tilde);

/* fp32-data kernels of the fit, on the context's GEMM path (tcgen05 split-TF32
 * or SIMT FFMA); all operands device-resident.
 * sketch: out (m x w_cols, row-major fp32, ld ldo) = X W, W fp64 column-major n x w_cols.
 * gemm_t: F (l x n column-major fp64) = U^T X, U row-major fp32 m x l (ld ldu). */
lpca_status lpca_sketch_f32(lpca_ctx* ctx, const lpca_matrix_view* x, const double* w_dev,
                            int64_t w_cols, float* out_dev, int64_t ldo);
lpca_status lpca_gemm_t_f32(lpca_ctx* ctx, const float* u_dev, int64_t ldu, int64_t l,
                            const lpca_matrix_view* x, double* f_dev);

/* ---- synthetic data (BASELINE generator; not part of the reference) -------
 * X = G diag(rho^t) H + noise * E into device memory, row-major m x n, rows
 * [row0, row0 + m) of the global matrix (so any row shard can be produced on any
 * GPU). G, H, E are counter-based N(0,1) streams keyed by (seed, index). */
lpca_status lpca_synth_lowrank(lpca_ctx* ctx, int64_t row0, int64_t m, int64_t n, int64_t r,
                               double rho, double noise, uint64_t seed, int32_t dtype, void* x_dev,
                               int64_t ldx);

#ifdef __cplusplus
}
#endif
#endif /* LAZYPCA_B200_H */
