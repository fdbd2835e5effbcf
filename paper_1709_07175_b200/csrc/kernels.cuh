// Kernel launchers of lazypca_b200 (all sm_100a). Each names the reference
// routine whose semantics it implements.
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace lpca {

// ---- projection (proj/core/src/projection.cpp:71-126) --------------------
// Omega dense column-major n x l (ld >= n), fp64, exactly the reference's
// per-column xoshiro256** streams.
void launch_omega_gaussian(cudaStream_t s, index_t n, index_t l, std::uint64_t seed, double* out,
                           index_t ld);
// {-1, 0, +1} pattern of gen_very_sparse, dense column-major, unscaled.
void launch_omega_very_sparse(cudaStream_t s, index_t n, index_t l, double density,
                              std::uint64_t seed, double* out, index_t ld);

// ---- synthetic data --------------------------------------------------------
// Rows [row0, row0+m) of X = G diag(rho^t) H + noise E, row-major, dtype 4/8.
// `sigma` holds r fp64 scale factors; scratch needs (rows_per_batch*r + r*n) doubles.
void launch_synth_lowrank(cudaStream_t s, index_t row0, index_t m, index_t n, index_t r,
                          const double* sigma_dev, double noise, std::uint64_t seed, int dtype,
                          void* x, index_t ldx, double* scratch, index_t scratch_elems);

// ---- elementwise / layout helpers -----------------------------------------
// dst[c*ldd + i] = (TO) (scale * src[c*lds + i]) for i < rows, c < cols (column-major copy/convert).
void launch_convert_f64_to_f32(cudaStream_t s, const double* src, index_t lds, float* dst,
                               index_t ldd, index_t rows, index_t cols, double scale);
void launch_scale_f64(cudaStream_t s, const double* src, double* dst, index_t count, double inv);
// Split fp64 column-major W (n x w) into tf32-exact hi/lo fp32 planes [wpad][ldd]
// (rows >= w zero-filled): hi = tf32(W), lo = tf32(W - hi).
void launch_split_tf32_w(cudaStream_t s, const double* w, index_t ldw, index_t n, index_t wc,
                         index_t wpad, float* hi, float* lo, index_t ldd);
// Densify a CSC matrix (device arrays) into row-major dtype storage.
void launch_csc_to_dense(cudaStream_t s, index_t m, index_t n, const std::int64_t* col_ptr,
                         const std::int64_t* row_idx, const double* vals, int dtype, void* x,
                         index_t ldx);
// Transpose a column-major dtype matrix into row-major.
void launch_transpose(cudaStream_t s, int dtype, const void* src, index_t lds, index_t rows,
                      index_t cols, void* dst, index_t ldd);
void launch_zero(cudaStream_t s, void* p, std::size_t bytes);
// dst (fp64, packed row-major m x n) = src (fp32 row-major, ld lds), exact widening.
void launch_widen_f32(cudaStream_t s, const float* src, index_t lds, index_t m, index_t n, double* dst);

// ---- SIMT GEMMs (FFMA / DFMA) ------------------------------------------------
// out[i*ors + c*ocs] = sum_j X[i*ldx + j] * W[c*ldw + j]  (spmm, kernels.cpp:30-47)
// T = float: fp32 products, fp32 sums over 256-wide K blocks, fp64 across blocks.
// T = double, exact: mul+add in ascending j (the reference's rounding sequence).
template <typename T, typename TO>
void launch_xw_simt(cudaStream_t s, const T* x, index_t m, index_t n, index_t ldx, const T* w,
                    index_t wc, index_t ldw, TO* out, index_t ors, index_t ocs, bool exact);
// part[c][j*l + r] = sum_{i in chunk c} U[i*ldu + r] * X[i*ldx + j]  (gemm_t, kernels.cpp:70-113)
template <typename T>
void launch_utx_simt(cudaStream_t s, const T* u, index_t ldu, const T* x, index_t ldx, index_t m,
                     index_t l, index_t n, index_t chunk_rows, double* part, bool exact);
// ---- sparse X (sparse.cu): the reference's order, bitwise (kernels.cpp:30-113) --
// out (m x w, element (i, c) at i*ors + c*ocs, fp64 or fp32) = X W with X in CSR
// and W row-major n x w (ld ldw).
void launch_spmm_csr(cudaStream_t s, index_t m, const std::int64_t* row_ptr, const std::int32_t* col,
                     const double* val, const double* wt, index_t ldw, index_t w, void* out, int out_dtype,
                     index_t ors, index_t ocs);
// F (l x n column-major) (+)= U^T X with X in CSC and U row-major m x l (ld ldu), l <= 512.
// Sparse X times a {-1, 0, +1} W (very sparse Omega) from per-row bit masks of
// W (sparse.cu): bitwise the dense-W spmm_csr. masks: n * 2 * pm1_mask_words(l).
int pm1_mask_words(index_t l);
void launch_pm1_masks(cudaStream_t s, const double* w, index_t n, index_t l, index_t ldw, std::uint32_t* masks);
void launch_spmm_csr_pm1(cudaStream_t s, index_t m, const std::int64_t* row_ptr, const std::int32_t* col,
                         const double* val, const std::uint32_t* masks, index_t w, double* out, index_t ors,
                         index_t ocs);
// Device staging of a host CSC (sparse.cu): checks in the host loop's order
// (first = 4 p + code of the first failing entry, ~0 if none), 32-bit rows,
// column of each entry, fp64 values; then the CSR copy by a stable row sort.
std::size_t csc_stage_temp_bytes(index_t m, index_t nnz);
void launch_csc_check(cudaStream_t s, index_t n, index_t rows, const std::int64_t* cp, const std::int64_t* ri64,
                      const void* val, int dtype, std::int32_t* ri, std::int32_t* colof, double* cv,
                      unsigned long long* first);
void launch_csr_from_csc(cudaStream_t s, index_t m, index_t nnz, const std::int32_t* ri, const std::int32_t* colof,
                         const double* cv, std::int64_t* rp, std::int32_t* ci, double* rv, std::int64_t* cnt,
                         std::int32_t* keys_out, void* temp, std::size_t temp_bytes);
void launch_gemm_t_csc(cudaStream_t s, index_t n, const std::int64_t* col_ptr, const std::int32_t* row,
                       const double* val, const double* u, index_t ldu, index_t l, double* f, bool accumulate);
// ---- verification metrics (metrics.cu; metrics.cpp:123-136, 311-352) -------------
// C (ka x kb) = A^T B, A n x ka and B n x kb column-major fp64.
void launch_atb(cudaStream_t s, const double* a, index_t n, index_t ka, const double* b, index_t kb, double* c);
// part[0 .. residual_sq_blocks(n, ka)) = tile sums of (A - B C)^2, C kb x ka.
index_t residual_sq_blocks(index_t n, index_t ka);
void launch_residual_sq(cudaStream_t s, const double* a, index_t n, index_t ka, const double* b, index_t kb,
                        const double* c, double* part);
// Pair distances: orig from X (dense row-major dtype/ld, or CSR when rp), da/db
// from row-major Y_a / Y_b (m x k fp64; yb nullable).
void launch_pair_distances(cudaStream_t s, int dtype, const void* x, index_t ld, index_t n, const std::int64_t* rp,
                           const std::int32_t* ci, const double* rv, const double* ya, const double* yb, index_t k,
                           const std::int64_t* pi, const std::int64_t* pj, index_t pairs, double* orig, double* da,
                           double* db);
// ---- residual-norm metrics (spectral.cu; metrics.cpp:148-308) ------------------
// y (m) = X v: dense row-major dtype (x, ld) or CSR (rp, ci, rv).
void launch_matvec(cudaStream_t s, int dtype, const void* x, index_t ld, index_t m, index_t n, const std::int64_t* rp,
                   const std::int32_t* ci, const double* rv, const double* v, double* y);
// y (n) = X^T t: dense (partials in part, matvec_t_chunks(m, n) x n) or CSC.
index_t matvec_t_chunks(index_t m, index_t n);
void launch_matvec_t(cudaStream_t s, int dtype, const void* x, index_t ld, index_t m, index_t n,
                     const std::int64_t* cp, const std::int32_t* ri, const double* cv, const double* t, double* part,
                     double* y);
// out (l) = U^T t for U m x l column-major (ld ldu); part basis_t_chunks(m) x l.
index_t basis_t_chunks(index_t m);
void launch_basis_t(cudaStream_t s, const double* u, index_t ldu, index_t m, index_t l, const double* t,
                    double* part, double* out);
// y (m) = t - U sv.
void launch_basis_sub(cudaStream_t s, const double* u, index_t ldu, index_t m, index_t l, const double* sv,
                      const double* t, double* y);
// part[0 .. sumsq_blocks(rows*cols)) = partial sums of squares of a (rows x cols, ld).
index_t sumsq_blocks(index_t count);
void launch_sumsq(cudaStream_t s, int dtype, const void* a, index_t ld, index_t rows, index_t cols, double* part);
// dense row-major m x n fp64 from CSR.
void launch_csr_to_dense(cudaStream_t s, index_t m, index_t n, const std::int64_t* rp, const std::int32_t* ci,
                         const double* rv, double* out);
// out = Rinv (Rinv^T sv): (U^T U)^{-1} sv with Rinv = L^{-T} from launch_chol_inverse.
void launch_chol_solve(cudaStream_t s, const double* rinv, index_t l, const double* sv, double* tmp, double* out);
// y += x (fp64), the streaming reducers' running F and U^T U (gemm_t_add, kernels.cpp:95-113).
void launch_add_f64(cudaStream_t s, const double* x, double* y, index_t count);
// out[idx] = sum_c part[c][idx], c ascending (fixed order; no float atomics).
void launch_reduce_partials(cudaStream_t s, const double* part, index_t nparts, index_t count,
                            double* out);

// ---- tcgen05 split-TF32 GEMMs (fp32 data) -------------------------------------
// out (fp32, row-major [m][ldo]) = X (fp32 row-major) * W, with W given as tf32
// hi/lo planes [wpad][ldw]: X_hi*W_hi + X_lo*W_hi + X_hi*W_lo accumulated in TMEM.
bool tc_xw_supported(index_t n, index_t wpad);
void launch_xw_tc(cudaStream_t s, const float* x, index_t m, index_t n, index_t ldx,
                  const float* w_hi, const float* w_lo, index_t wpad, index_t ldw, float* out,
                  index_t ldo, int num_sms);
// Same, with any of: plain fp32 output (out, ldo, first wstore columns) and the
// tf32 hi/lo planes of the output (out_hi/out_lo, ld ldh, all wpad columns).
void launch_xw_tc_planes(cudaStream_t s, const float* x, index_t m, index_t n, index_t ldx,
                         const float* w_hi, const float* w_lo, index_t wpad, index_t ldw, float* out,
                         index_t ldo, index_t wstore, float* out_hi, float* out_lo, index_t ldh,
                         int num_sms);
// part[s][j*l + r] for r < l: U^T X with U given as tf32 hi/lo planes [m][ldu];
// `splits` row splits (utx_tc_splits) summed afterwards in fixed order.
bool tc_utx_supported(index_t l, index_t n);
index_t utx_tc_splits(index_t m, index_t l, index_t n, int num_sms, index_t* rows_per_split);
void launch_utx_tc_planes(cudaStream_t s, const float* u_hi, const float* u_lo, index_t ldu,
                          const float* x, index_t ldx, index_t m, index_t l, index_t n, double* part,
                          int num_sms);
void launch_utx_tc(cudaStream_t s, const float* u, index_t ldu, const float* x, index_t ldx,
                   index_t m, index_t l, index_t n, index_t chunk_rows, double* part,
                   int num_sms);
// ---- 2-SM pair passes (tc_pair.cuh) -------------------------------------------
// Both encodings of the 3-term split: tf32 hi/lo (half = false) or fp16 hi/lo of
// power-of-two scaled operands (half = true: X scaled from max|X| = *xmax_in,
// W planes per column (winv = inverse scales), U^T planes per column and
// kUScaleRows-row block (uinv[block][c])). Planes are K-major: [wpad or round_up(l,16)][ld].
// rows per block of the U^T fp16 plane scales: two 256-row X W pair items
// (done back to back by one pair), one fp16 run (8 stages of 64 rows) of the
// X^T U pass. (1024-row blocks, XᵀU runs twice as deep, measured no faster
// at configs[2]: 134.6-138.2 against 133.0-134.9 ms per step.)
constexpr index_t kUScaleRows = 512;

struct XwPairArgs {
  const float* x = nullptr;
  index_t m = 0, n = 0, ldx = 0;
  bool half = false;
  const void* w_hi = nullptr;
  const void* w_lo = nullptr;
  index_t wpad = 0, ldw = 0;
  const float* winv = nullptr;
  const uint32_t* xmax_in = nullptr;  // max|X| bits on the device, or
  float xmax_val = 0.0f;              // max|X| by value (xmax_in null)
  uint32_t* xmax_out = nullptr;       // atomicMax of the |X| bits actually read
  int* ovf = nullptr;  // per-run scales from each run's first stage; set to 1 if a later stage needed a rescan
  const int* wlo_nz = nullptr;   // fp16: 0 when every w_lo entry is zero (the a_hi w_lo MMAs are skipped)
  float* out = nullptr;          // plain fp32 row-major (first wstore columns)
  index_t ldo = 0, wstore = 0;
  float* out_hi = nullptr;       // tf32 planes of OUT^T [wpad][ldh]
  float* out_lo = nullptr;
  __half* uh = nullptr;          // fp16 planes of OUT^T [wpad][ldh] ...
  __half* ul = nullptr;
  float* uinv = nullptr;         // ... with inverse scales [ceil(m/kUScaleRows)][wpad]
  index_t ldh = 0;
  cudaEvent_t ev_pre = nullptr, ev_post = nullptr;  // recorded around the kernel launch itself
};
struct UtxPairArgs {
  bool half = false;
  const void* u_hi = nullptr;
  const void* u_lo = nullptr;
  index_t ldt = 0;
  const float* uinv = nullptr;
  const uint32_t* xmax_in = nullptr;
  const float* x = nullptr;
  index_t ldx = 0, m = 0, l = 0, n = 0;
  double* part = nullptr;  // [chunks][n][l] (utx_pair_splits)
  cudaEvent_t ev_pre = nullptr, ev_post = nullptr;
};
bool tc_pair_mode();
void launch_xw_pair(cudaStream_t s, const XwPairArgs& p, int num_sms);
index_t utx_pair_splits(index_t m, index_t n, int num_sms, index_t* rows_per_split);
void launch_utx_pair(cudaStream_t s, const UtxPairArgs& p, int num_sms);
// W (fp64 n x wc, column-major ld ldw) -> fp16 hi/lo planes [wpad][ldd] scaled per
// column by 2^(14 - floor(log2 max|W[:,c]|)); winv[c] = inverse scale (1 for padding).
// lo_nz (optional): set to 1 if any lo entry is nonzero, else 0.
void launch_split_f16_w(cudaStream_t s, const double* w, index_t ldw, index_t n, index_t wc, index_t wpad,
                        __half* hi, __half* lo, index_t ldd, float* winv, int* lo_nz = nullptr);

// Split a row-major fp32 matrix (m x ld) into tf32 hi/lo planes of the same shape.
void launch_split_tf32_rows(cudaStream_t s, const float* src, index_t m, index_t ld, float* hi,
                            float* lo);
// Transpose + split: src row-major m x cols (ld lds) -> hi/lo planes [cols][ldt]
// (element (i, c) at c * ldt + i).
void launch_split_tf32_transpose(cudaStream_t s, const float* src, index_t m, index_t cols, index_t lds,
                                 float* hi, float* lo, index_t ldt);

// ---- small fp64 kernels (the l x l step) ----------------------------------------
// G = F F^T, F l x n column-major, bitwise symmetric (dense_aat, kernels.cpp:148-172).
void launch_gram(cudaStream_t s, const double* f, index_t l, index_t n, double* g);
// Same product for the fit path: split-K DFMA tiles, chunk partials summed in a
// fixed order (deterministic, not the reference's rounding sequence).
// `part` holds gram_fast_chunks(l, n) * l * l doubles.
index_t gram_fast_chunks(index_t l, index_t n);
void launch_gram_fast(cudaStream_t s, const double* f, index_t l, index_t n, double* g, double* part);
// U^T U for tall U (m x l row-major) into chunk partials part[c][a + b*l] (full square).
template <typename T>
void launch_syrk_partials(cudaStream_t s, const T* u, index_t ldu, index_t m, index_t l,
                          index_t chunk_rows, double* part);
// Cyclic parallel Jacobi (round-robin schedule of jacobi.cpp:18-33).
// a: l x l column-major (overwritten); evals descending; evecs column-major.
// status[0] = 0 ok / 1 no convergence; gap[0] = last max off-diagonal.
void launch_jacobi_eigh(cudaStream_t s, double* a, index_t l, double* evals, double* evecs,
                        double* work, int* status, double* gap);
// Tridiagonal route (eigh.cu): a (l x l column-major, read only) -> evals
// descending, evecs column-major. `work` holds eigh_tridiag_workspace(l) bytes.
// status[0] = 0 ok / 2 asymmetric input (gap[0] = max asymmetry).
std::size_t eigh_tridiag_workspace(index_t l);
void launch_eigh_tridiag(cudaStream_t s, const double* a, index_t l, double* evals, double* evecs, void* work,
                         int* status, double* gap);
// V(j,r) = (sum_i F(i,j) Ut(i,r)) / sigma_r  (truncated_svd.cpp:52-62), then the
// canonical sign flip (truncated_svd.cpp:64-80) applied to V and Ut.
void launch_vform(cudaStream_t s, const double* f, index_t l, index_t n, const double* ut,
                  const double* evals, index_t k, double* sigma, double* v);
void launch_sign_canon(cudaStream_t s, double* v, index_t n, index_t k, double* ut, index_t l);
// Cholesky of an SPD l x l (lower L, column-major), then R^{-1} = L^{-T} (upper).
// status[0] = pivot index + 1 on failure (pivot tol 1e-14 * max diag,
// lazy_projector.cpp:12-37).
void launch_chol_inverse(cudaStream_t s, const double* g, index_t l, double* rinv, double* work,
                         int* status, double tol_rel = 1e-14);
// Very sparse Omega sketch (csrc/sparse_omega.cu): per-(K chunk, column) lists
// of Omega's nonzeros, then U = X Omega by gathers (U row-major, ld ldu <= 512,
// padding columns zeroed; max|X| into xmax when given), and U^T fp16 planes
// with per-(column, 256-row block) scales from a plain fp32 U.
index_t sparse_sketch_chunks(index_t n, int dtype);
void launch_omega_chunk_lists(cudaStream_t s, const double* omega, index_t n, index_t l, int dtype, int* counts,
                              int* ptr, std::uint32_t* ent);
template <typename T>
void launch_sparse_sketch(cudaStream_t s, const T* x, index_t m, index_t n, index_t ldx, const int* ptr,
                          const std::uint32_t* ent, index_t l, T* u, index_t ldu, std::uint32_t* xmax, int num_sms);
void launch_u_planes_f16(cudaStream_t s, const float* u, index_t m, index_t ld, index_t npad, __half* hi, __half* lo,
                         index_t ldt, float* uinv);
// Row gather for fp32 X (lanes = Omega columns, rows by 1-D bulk copies, a
// bank-conflict-free entry schedule per warp from an edge colouring):
// column lists (device), the schedule (host, packed [warp][smax/2][32] 2x16-bit
// entries; returns the steps, -1 if infeasible), the launch.
bool row_gather_feasible(index_t m, index_t n, index_t ldx, index_t l);
void launch_omega_col_lists(cudaStream_t s, const double* omega, index_t n, index_t l, int cap, int* cnt,
                            std::uint32_t* cols);
int build_row_schedule(const int* cnt, const std::uint32_t* cols, int cap, index_t n, index_t l,
                       std::vector<std::uint32_t>& packed, int* smax_out, int* splits_out);
void launch_sparse_sketch_rows(cudaStream_t s, const float* x, index_t m, index_t n, index_t ldx,
                               const std::uint32_t* sched, int steps, int smax, int splits, index_t l, float* u,
                               index_t ldu, std::uint32_t* xmax, int num_sms);
// C = op(A) op(B) + beta C, l x l column-major (op = transpose when ta / tb; b null = identity).
void launch_small_gemm(cudaStream_t s, int ta, int tb, index_t l, const double* a, const double* b, double* c,
                       double beta);
// rdiag = 1 / diag(W) (first) or rdiag *= 1 / diag(W): diag of a product of R factors.
void launch_rdiag_update(cudaStream_t s, const double* w, index_t l, double* rdiag, int first);
void launch_trace(cudaStream_t s, const double* g, index_t l, double* out);
// W = R^{-1} for an upper-triangular R, in launch_chol_inverse's layout (work: l x l).
void launch_upper_inverse(cudaStream_t s, const double* r, index_t l, double* w, double* work, int* status);
// g_ii += c * trace(g) (shifted CholeskyQR's first pass).
void launch_add_trace_shift(cudaStream_t s, double* g, index_t l, double c);
// out[0] = flag[0] != 0 (an int flag made summable over ranks).
void launch_flag_to_f64(cudaStream_t s, const int* flag, double* out);
// F <- L^{-1} F  ==  (Z R^{-1})^T for Z = F^T; rinv = L^{-T} upper, F l x n col-major.
void launch_apply_rinv_t(cudaStream_t s, const double* rinv, index_t l, double* f, index_t n,
                         double* tmp);

}  // namespace lpca
