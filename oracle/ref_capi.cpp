// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A flat C ABI over the *unmodified* reference `lazypca` core, compiled from the
// sources under /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/liblazypca_ref.so. Only tests/, __graft_entry__.smoke() and the
// CPU-baseline legs of bench.py load it, as the checker / the timed reference.
//
// Dense inputs arrive row-major (the layout the GPU path keeps in HBM) and are
// converted to the reference's canonical CSC (exact zeros dropped, as
// `sparsify` does, proj/core/src/matrix_io.cpp:296-311) before the reference
// entry point is called. Outputs come back in the reference's own layouts
// (column-major dense, fp64).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "lazypca/error.hpp"
#include "lazypca/jacobi.hpp"
#include "lazypca/kernels.hpp"
#include "lazypca/projection.hpp"
#include "lazypca/qr.hpp"
#include "lazypca/reducer.hpp"
#include "lazypca/threading.hpp"
#include "lazypca/tridiag_eigh.hpp"
#include "lazypca/truncated_svd.hpp"
#include "lazypca/matrix_io.hpp"
#include "lazypca/metrics.hpp"
#include "lazypca/spectral_norm.hpp"

using namespace lazypca;

namespace {

thread_local std::string g_err;
thread_local std::int64_t g_err_index = -1;

// Status codes shared with include/lazypca_b200.h so the tests can compare the
// two error surfaces one to one.
enum : int {
  kOk = 0,
  kDimension = 1,
  kInvalidArgument = 2,
  kRankDeficiency = 3,
  kConvergence = 4,
  kParse = 5,
  kOther = 9,
};

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    g_err.clear();
    g_err_index = -1;
    return kOk;
  } catch (const DimensionError& e) {
    g_err = e.what();
    return kDimension;
  } catch (const InvalidArgumentError& e) {
    g_err = e.what();
    return kInvalidArgument;
  } catch (const RankDeficiencyError& e) {
    g_err = e.what();
    g_err_index = e.index();
    return kRankDeficiency;
  } catch (const ConvergenceError& e) {
    g_err = e.what();
    return kConvergence;
  } catch (const ParseError& e) {
    g_err = e.what();
    g_err_index = e.line();
    return kParse;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kOther;
  }
}

template <typename T>
SparseMatrix csc_from_rowmajor(const T* x, index_t m, index_t n) {
  std::vector<index_t> ptr(static_cast<std::size_t>(n) + 1, 0);
  for (index_t j = 0; j < n; ++j) {
    index_t c = 0;
    for (index_t i = 0; i < m; ++i) c += x[i * n + j] != T(0);
    ptr[static_cast<std::size_t>(j) + 1] = ptr[static_cast<std::size_t>(j)] + c;
  }
  std::vector<index_t> idx(static_cast<std::size_t>(ptr.back()));
  std::vector<double> val(static_cast<std::size_t>(ptr.back()));
  for (index_t j = 0; j < n; ++j) {
    index_t p = ptr[static_cast<std::size_t>(j)];
    for (index_t i = 0; i < m; ++i) {
      const T v = x[i * n + j];
      if (v != T(0)) {
        idx[static_cast<std::size_t>(p)] = i;
        val[static_cast<std::size_t>(p)] = static_cast<double>(v);
        ++p;
      }
    }
  }
  return SparseMatrix::from_csc(m, n, std::move(ptr), std::move(idx), std::move(val));
}

SparseMatrix csc_any(const void* x, int dtype, index_t m, index_t n) {
  return dtype == 4 ? csc_from_rowmajor(static_cast<const float*>(x), m, n)
                    : csc_from_rowmajor(static_cast<const double*>(x), m, n);
}

DenseMatrix dense_from(const double* colmajor, index_t r, index_t c) {
  return DenseMatrix(r, c, std::vector<double>(colmajor, colmajor + r * c));
}

void copy_out(const DenseMatrix& a, double* out) {
  std::memcpy(out, a.data(), sizeof(double) * static_cast<std::size_t>(a.rows() * a.cols()));
}

ReducerConfig make_cfg(int method, std::int64_t k, std::int64_t l, std::uint64_t seed, int kind,
                       double density, std::int64_t block_rows) {
  ReducerConfig c;
  c.method = method == 0 ? ReducerMethod::rp : method == 1 ? ReducerMethod::spca
                                                           : ReducerMethod::lazy_spca;
  c.k = k;
  c.l = l;
  c.projection.kind = kind == 0 ? ProjectionKind::gaussian : ProjectionKind::very_sparse;
  c.projection.density = density;
  c.projection.seed = seed;
  c.block_rows = block_rows;
  c.streaming = block_rows > 0;
  return c;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
std::int64_t ref_last_error_index() { return g_err_index; }
void ref_set_thread_count(int n) { set_thread_count(n); }

// Omega as the reference generates it (proj/core/src/projection.cpp:71-126),
// returned dense column-major n x l (very sparse: the {-1,0,+1} pattern, unscaled).
int ref_regenerate(int kind, std::int64_t n, std::int64_t l, double density, std::uint64_t seed,
                   double* out, double* scale) {
  return guarded([&] {
    ProjectionSpec s{kind == 0 ? ProjectionKind::gaussian : ProjectionKind::very_sparse, n, l,
                     density, seed};
    const ProjectionMatrix p = regenerate(s);
    copy_out(p.is_dense() ? p.dense() : p.sparse().to_dense(), out);
    *scale = p.scale;
  });
}

int ref_density_for(int mode, std::int64_t k, double value, double* out) {
  return guarded([&] {
    DensityPolicy p = mode == 0 ? DensityPolicy::aggressive()
                      : mode == 1 ? DensityPolicy::conservative()
                                  : DensityPolicy::explicit_value(value);
    *out = density_for(p, k);
  });
}

// reduce() dispatcher (proj/core/src/reducer.cpp:337-346) on dense row-major X.
// v_out: n x k column-major; sigma_out: k values (left untouched for rp);
// timings: {sketch, qr, f_form, svd, total} seconds.
int ref_reduce(int method, const void* x, int dtype, std::int64_t m, std::int64_t n,
               std::int64_t k, std::int64_t l, std::uint64_t seed, int kind, double density,
               std::int64_t block_rows, double* v_out, double* sigma_out, double* scale_out,
               double* timings) {
  return guarded([&] {
    const SparseMatrix xs = csc_any(x, dtype, m, n);
    ReducerTimings t;
    const ReductionMap map = reduce(xs, make_cfg(method, k, l, seed, kind, density, block_rows), &t);
    copy_out(map.v, v_out);
    if (sigma_out)
      for (std::size_t i = 0; i < map.singular_values.size(); ++i) sigma_out[i] = map.singular_values[i];
    if (scale_out) *scale_out = map.scale;
    if (timings) {
      timings[0] = t.sketch;
      timings[1] = t.qr;
      timings[2] = t.f_form;
      timings[3] = t.svd;
      timings[4] = t.total;
    }
  });
}

// Fit + transform, timed the way bench.py's CPU leg reports it: the CSC
// conversion is outside the timed region, reduce() + apply_map() inside.
int ref_fit_transform(int method, const void* x, int dtype, std::int64_t m, std::int64_t n,
                      std::int64_t k, std::int64_t l, std::uint64_t seed, int kind,
                      double density, double* y_out, double* v_out, double* sigma_out,
                      double* seconds) {
  return guarded([&] {
    const SparseMatrix xs = csc_any(x, dtype, m, n);
    const auto t0 = std::chrono::steady_clock::now();
    const ReductionMap map = reduce(xs, make_cfg(method, k, l, seed, kind, density, 0));
    const DenseMatrix y = apply_map(map, xs);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (y_out) copy_out(y, y_out);
    if (v_out) copy_out(map.v, v_out);
    if (sigma_out)
      for (std::size_t i = 0; i < map.singular_values.size(); ++i) sigma_out[i] = map.singular_values[i];
  });
}

// ref_fit_transform on a caller's canonical CSC (col_ptr n+1, row_idx and
// values nnz; SparseMatrix::from_csc validates it), for sparse-X timing
// (tools/sparse_bench.py): reduce() + apply_map() timed, the copy into the
// reference's SparseMatrix outside.
int ref_fit_transform_csc(int method, std::int64_t m, std::int64_t n, const std::int64_t* col_ptr,
                          const std::int64_t* row_idx, const double* values, std::int64_t k, std::int64_t l,
                          std::uint64_t seed, int kind, double density, double* y_out, double* v_out,
                          double* sigma_out, double* seconds) {
  return guarded([&] {
    const std::int64_t nnz = col_ptr[n];
    const SparseMatrix xs = SparseMatrix::from_csc(m, n, std::vector<index_t>(col_ptr, col_ptr + n + 1),
                                                   std::vector<index_t>(row_idx, row_idx + nnz),
                                                   std::vector<double>(values, values + nnz));
    const auto t0 = std::chrono::steady_clock::now();
    const ReductionMap map = reduce(xs, make_cfg(method, k, l, seed, kind, density, 0));
    const DenseMatrix y = apply_map(map, xs);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (y_out) copy_out(y, y_out);
    if (v_out) copy_out(map.v, v_out);
    if (sigma_out)
      for (std::size_t i = 0; i < map.singular_values.size(); ++i) sigma_out[i] = map.singular_values[i];
  });
}

// Lazy SPCA with q power steps composed from the reference's own kernels
// (the reference has no power iterations; this is the builder's
// scheme of SURVEY 8(a) a16 restated on the reference's code):
//   U = build_sketch(X, Omega)                         (reducer.cpp:163-169)
//   q times: Z = gemm_t(U, X)^T, Q = householder_qr(Z).q, U = spmm(X, Q)
//   F = gemm_t(U, X); truncated_svd_via_gram(F, k)     (reducer.cpp:216-234)
//   Y = spmm(X, V)                                     (apply_map, reducer.cpp:348-353)
// Timed like ref_fit_transform (CSC conversion outside the timed region).
// For q = 0 the result equals reduce_lazy_spca + apply_map.
int ref_lazy_power_fit_transform(const void* x, int dtype, std::int64_t m, std::int64_t n, std::int64_t k,
                                 std::int64_t l, std::uint64_t seed, int kind, double density, int q,
                                 double* y_out, double* v_out, double* sigma_out, double* seconds) {
  return guarded([&] {
    const SparseMatrix xs = csc_any(x, dtype, m, n);
    const auto t0 = std::chrono::steady_clock::now();
    const ReducerConfig cfg = make_cfg(2, k, l, seed, kind, density, 0).resolved(n);
    const ProjectionMatrix omega = regenerate(cfg.projection);
    DenseMatrix u = build_sketch(xs, omega).u;
    for (int it = 0; it < q; ++it) {
      const DenseMatrix zt = gemm_t(u, xs);  // l x n
      DenseMatrix z(n, l);
      for (index_t j = 0; j < l; ++j)
        for (index_t i = 0; i < n; ++i) z(i, j) = zt(j, i);
      u = spmm(xs, householder_qr(z).q);
    }
    const TruncatedSVD svd = truncated_svd_via_gram(gemm_t(u, xs), k);
    const DenseMatrix y = spmm(xs, svd.v);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (y_out) copy_out(y, y_out);
    if (v_out) copy_out(svd.v, v_out);
    if (sigma_out)
      for (std::int64_t i = 0; i < k; ++i) sigma_out[i] = svd.singular_values[static_cast<std::size_t>(i)];
  });
}

// save_map_file / load_map_file (proj/core/src/reducer.cpp:355-412). method:
// 0 rp, 1 spca, 2 lazy_spca; sigma may be null (no singular values).
int ref_save_map_file(int method, std::int64_t k, std::int64_t l, std::int64_t n, std::uint64_t seed,
                      double density, double scale, const double* v, const double* sigma, const char* path) {
  return guarded([&] {
    ReductionMap map;
    map.method = method == 0 ? "rp" : method == 1 ? "spca" : "lazy_spca";
    map.k = k;
    map.l = l;
    map.n = n;
    map.seed = seed;
    map.density = density;
    map.scale = scale;
    map.v = dense_from(v, n, k);
    if (sigma) map.singular_values.assign(sigma, sigma + k);
    save_map_file(map, path);
  });
}

// Reads a map file; v_out (n*k) and sigma_out (k) may be null to query the shape.
int ref_load_map_file(const char* path, std::int64_t* k, std::int64_t* l, std::int64_t* n, std::uint64_t* seed,
                      double* density, double* scale, int* has_sigma, double* v_out, double* sigma_out) {
  return guarded([&] {
    const ReductionMap map = load_map_file(path);
    *k = map.k;
    *l = map.l;
    *n = map.n;
    *seed = map.seed;
    *density = map.density;
    *scale = map.scale;
    *has_sigma = map.singular_values.empty() ? 0 : 1;
    if (v_out) copy_out(map.v, v_out);
    if (sigma_out)
      for (std::size_t i = 0; i < map.singular_values.size(); ++i) sigma_out[i] = map.singular_values[i];
  });
}

// apply_map (proj/core/src/reducer.cpp:348-353): Y = X V, Y m x k column-major.
int ref_apply_map(const void* x, int dtype, std::int64_t m, std::int64_t n, const double* v,
                  std::int64_t k, double* y_out) {
  return guarded([&] {
    ReductionMap map;
    map.n = n;
    map.k = k;
    map.v = dense_from(v, n, k);
    copy_out(apply_map(map, csc_any(x, dtype, m, n)), y_out);
  });
}

// spmm(X, W) (proj/core/src/kernels.cpp:30-47): out m x w column-major.
int ref_spmm(const void* x, int dtype, std::int64_t m, std::int64_t n, const double* w,
             std::int64_t wc, double* out) {
  return guarded([&] { copy_out(spmm(csc_any(x, dtype, m, n), dense_from(w, n, wc)), out); });
}

// gemm_t(U, X) (proj/core/src/kernels.cpp:70-113): out l x n column-major.
int ref_gemm_t(const double* u, std::int64_t m, std::int64_t l, const void* x, int dtype,
               std::int64_t n, double* out) {
  return guarded([&] { copy_out(gemm_t(dense_from(u, m, l), csc_any(x, dtype, m, n)), out); });
}

// dense_aat (proj/core/src/kernels.cpp:148-172): out l x l column-major.
int ref_dense_aat(const double* f, std::int64_t l, std::int64_t n, double* out) {
  return guarded([&] { copy_out(dense_aat(dense_from(f, l, n)), out); });
}

// tridiag_eigh / jacobi_eigh: eigenvalues descending, eigenvectors column-major.
int ref_eigh(int which, const double* a, std::int64_t l, double* evals, double* evecs) {
  return guarded([&] {
    const DenseMatrix g = dense_from(a, l, l);
    const EigenDecomposition e = which == 0 ? tridiag_eigh(g) : jacobi_eigh(g);
    for (std::int64_t i = 0; i < l; ++i) evals[i] = e.eigenvalues[static_cast<std::size_t>(i)];
    copy_out(e.eigenvectors, evecs);
  });
}

// truncated_svd_via_gram (proj/core/src/truncated_svd.cpp:13-82).
int ref_truncated_svd(const double* f, std::int64_t l, std::int64_t n, std::int64_t k,
                      double* sigma, double* v_out, double* u_tilde_out) {
  return guarded([&] {
    const TruncatedSVD s = truncated_svd_via_gram(dense_from(f, l, n), k);
    for (std::int64_t i = 0; i < k; ++i) sigma[i] = s.singular_values[static_cast<std::size_t>(i)];
    copy_out(s.v, v_out);
    if (u_tilde_out) copy_out(s.u_tilde, u_tilde_out);
  });
}

// householder_qr (proj/core/src/qr.cpp:104-132): Q m x l, R l x l column-major.
int ref_householder_qr(const double* a, std::int64_t m, std::int64_t l, double* q, double* r) {
  return guarded([&] {
    const QRFactors f = householder_qr(dense_from(a, m, l));
    copy_out(f.q, q);
    copy_out(f.r, r);
  });
}

// chordal_distance (proj/core/src/metrics.cpp:123-136) on two n x k bases.
int ref_chordal(const double* v1, const double* v2, std::int64_t n, std::int64_t k, double* out) {
  return guarded([&] { *out = chordal_distance(dense_from(v1, n, k), dense_from(v2, n, k)); });
}

// reconstruction_error (proj/core/src/metrics.cpp:148-259) on dense row-major X
// and a column-major m x l sketch: out = {spectral, frobenius, sigma_{k+1}, bound},
// flags = {has sigma, has bound}.
int ref_reconstruction_error(int route, const void* x, int dtype, std::int64_t m, std::int64_t n,
                             const double* u, std::int64_t l, std::int64_t k, int with_bound,
                             std::int64_t densify_limit, double* out, int* flags) {
  return guarded([&] {
    const ReconstructionErrorReport r =
        reconstruction_error(csc_any(x, dtype, m, n), dense_from(u, m, l),
                             route == 0 ? ResidualRoute::qr : ResidualRoute::lazy, k, l, with_bound != 0,
                             densify_limit);
    out[0] = r.spectral_error;
    out[1] = r.frobenius_error;
    out[2] = r.sigma_k_plus_1.value_or(0.0);
    out[3] = r.bound.value_or(0.0);
    flags[0] = r.sigma_k_plus_1.has_value();
    flags[1] = r.bound.has_value();
  });
}

// row_space_reconstruction_error (metrics.cpp:261-308), V n x k column-major.
int ref_row_space_reconstruction_error(const void* x, int dtype, std::int64_t m, std::int64_t n, const double* v,
                                       std::int64_t k, double* out) {
  return guarded([&] {
    const ReconstructionErrorReport r = row_space_reconstruction_error(csc_any(x, dtype, m, n), dense_from(v, n, k));
    out[0] = r.spectral_error;
    out[1] = r.frobenius_error;
  });
}

// spectral_norm(SparseMatrix) (proj/core/src/spectral_norm.cpp:70-77).
int ref_spectral_norm(const void* x, int dtype, std::int64_t m, std::int64_t n, double* out) {
  return guarded([&] { *out = spectral_norm(csc_any(x, dtype, m, n)); });
}

// matrix_io (proj/core/src/matrix_io.cpp). Readers are two-call: sizes first
// (arrays null), then the arrays. Sparse: CSC; dense: column-major.
int ref_read_matrix_file(int kind, const char* path, std::int64_t* rows, std::int64_t* cols, std::int64_t* nnz,
                         std::int64_t* ptr, std::int64_t* idx, double* val) {
  return guarded([&] {
    if (kind == 0) {
      const SparseMatrix x = read_sparse_matrix_market_file(path);
      *rows = x.rows();
      *cols = x.cols();
      *nnz = x.nnz();
      if (ptr) std::copy(x.col_ptr().begin(), x.col_ptr().end(), ptr);
      if (idx) std::copy(x.row_idx().begin(), x.row_idx().end(), idx);
      if (val) std::copy(x.values().begin(), x.values().end(), val);
    } else {
      const DenseMatrix d = kind == 1 ? read_dense_matrix_market_file(path) : read_dense_csv_file(path);
      *rows = d.rows();
      *cols = d.cols();
      *nnz = -1;
      if (val) copy_out(d, val);
    }
  });
}

int ref_write_matrix_file(int kind, const char* path, std::int64_t rows, std::int64_t cols, const std::int64_t* ptr,
                          const std::int64_t* idx, const double* val) {
  return guarded([&] {
    if (kind == 0) {
      const std::int64_t nnz = ptr[cols];
      write_sparse_matrix_market_file(
          SparseMatrix::from_csc(rows, cols, std::vector<index_t>(ptr, ptr + cols + 1),
                                 std::vector<index_t>(idx, idx + nnz), std::vector<double>(val, val + nnz)),
          path);
    } else if (kind == 1) {
      write_dense_matrix_market_file(dense_from(val, rows, cols), path);
    } else {
      write_dense_csv_file(dense_from(val, rows, cols), path);
    }
  });
}

// Block b of a MatrixMarket / CSV row-block stream as CSC (two-call); *count =
// the number of blocks the stream produced in total.
int ref_stream_block(int kind, const char* path, std::int64_t block_rows, std::int64_t b, std::int64_t* count,
                     std::int64_t* rows, std::int64_t* cols, std::int64_t* nnz, std::int64_t* ptr, std::int64_t* idx,
                     double* val) {
  return guarded([&] {
    std::unique_ptr<RowBlockStream> s;
    if (kind == 0)
      s = std::make_unique<MatrixMarketRowBlockStream>(path, block_rows);
    else
      s = std::make_unique<CsvRowBlockStream>(path, block_rows);
    std::int64_t n = 0;
    while (auto blk = s->next()) {
      if (n == b) {
        const SparseMatrix& x = blk->block;
        *rows = x.rows();
        *cols = x.cols();
        *nnz = x.nnz();
        if (ptr) std::copy(x.col_ptr().begin(), x.col_ptr().end(), ptr);
        if (idx) std::copy(x.row_idx().begin(), x.row_idx().end(), idx);
        if (val) std::copy(x.values().begin(), x.values().end(), val);
      }
      ++n;
    }
    *count = n;
  });
}

}  // extern "C"
