// Header-only C++ shim: the reference `lazypca` API (namespace lazypca,
// proj/core/include/lazypca/*.hpp) rebuilt over the lazypca_b200 C ABI, so a
// caller of the reference recompiles against this header and links
// liblazypca_b200.so instead of lazypca::core. Value types keep the reference's
// layouts (column-major fp64 DenseMatrix, canonical CSC SparseMatrix) and the
// C status codes are rethrown as the reference's exception classes
// (proj/core/include/lazypca/error.hpp:10-58).
#pragma once

#include <cmath>
#include <cstdint>
#include <exception>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "lazypca_b200.h"

namespace lazypca {

using index_t = std::int64_t;

// ---- errors (error.hpp) ---------------------------------------------------------
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class DimensionError : public Error {
 public:
  explicit DimensionError(const std::string& w) : Error(w) {}
};
class InvalidArgumentError : public Error {
 public:
  explicit InvalidArgumentError(const std::string& w) : Error(w) {}
};
class RankDeficiencyError : public Error {
 public:
  RankDeficiencyError(const std::string& w, std::int64_t index = -1) : Error(w), index_(index) {}
  std::int64_t index() const { return index_; }

 private:
  std::int64_t index_;
};
class ConvergenceError : public Error {
 public:
  ConvergenceError(const std::string& w, double gap = 0.0) : Error(w), gap_(gap) {}
  double last_gap() const { return gap_; }

 private:
  double gap_;
};
class ParseError : public Error {
 public:
  ParseError(const std::string& w, std::int64_t line = 0) : Error(w), line_(line) {}
  std::int64_t line() const { return line_; }

 private:
  std::int64_t line_;
};
// Device / collective failures have no reference analogue; they derive from Error.
class DeviceError : public Error {
 public:
  explicit DeviceError(const std::string& w) : Error(w) {}
};

namespace detail {
inline void check(lpca_status s) {
  if (s == LPCA_OK) return;
  const std::string msg = lpca_last_error();
  switch (s) {
    case LPCA_ERR_DIMENSION: throw DimensionError(msg);
    case LPCA_ERR_INVALID_ARGUMENT: throw InvalidArgumentError(msg);
    case LPCA_ERR_RANK_DEFICIENCY: throw RankDeficiencyError(msg, lpca_last_error_index());
    case LPCA_ERR_CONVERGENCE: throw ConvergenceError(msg, lpca_last_error_gap());
    case LPCA_ERR_PARSE: throw ParseError(msg, lpca_last_error_index());
    default: throw DeviceError(msg);
  }
}
// One context per process-thread on device 0 unless the caller installs one.
inline lpca_ctx*& current_ctx() {
  static thread_local lpca_ctx* ctx = nullptr;
  return ctx;
}
inline lpca_ctx* ctx() {
  lpca_ctx*& c = current_ctx();
  if (!c) check(lpca_ctx_create(0, &c));
  return c;
}
}  // namespace detail

// Installs a caller-owned context (e.g. one rank of a row-sharded NCCL group).
inline void use_context(lpca_ctx* c) { detail::current_ctx() = c; }

// threading.hpp:15-17 — accepted for compatibility; the GPU path has no host pool.
inline void set_thread_count(int) {}
inline int thread_count() { return 0; }

// ---- value types (dense_matrix.hpp, sparse_matrix.hpp) ------------------------------
class DenseMatrix {
 public:
  DenseMatrix() : rows_(0), cols_(0) {}
  DenseMatrix(index_t r, index_t c) : rows_(r), cols_(c), data_(static_cast<std::size_t>(r * c), 0.0) {}
  DenseMatrix(index_t r, index_t c, std::vector<double> cm) : rows_(r), cols_(c), data_(std::move(cm)) {}
  static DenseMatrix identity(index_t n) {
    DenseMatrix m(n, n);
    for (index_t i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
  index_t rows() const { return rows_; }
  index_t cols() const { return cols_; }
  bool empty() const { return rows_ == 0 || cols_ == 0; }
  double& operator()(index_t i, index_t j) { return data_[static_cast<std::size_t>(j * rows_ + i)]; }
  double operator()(index_t i, index_t j) const { return data_[static_cast<std::size_t>(j * rows_ + i)]; }
  double* col(index_t j) { return data_.data() + j * rows_; }
  const double* col(index_t j) const { return data_.data() + j * rows_; }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }

 private:
  index_t rows_, cols_;
  std::vector<double> data_;
};

class SparseMatrix {
 public:
  SparseMatrix() : rows_(0), cols_(0), col_ptr_{0} {}
  static SparseMatrix from_csc(index_t rows, index_t cols, std::vector<index_t> col_ptr,
                               std::vector<index_t> row_idx, std::vector<double> values) {
    SparseMatrix s;
    s.rows_ = rows;
    s.cols_ = cols;
    s.col_ptr_ = std::move(col_ptr);
    s.row_idx_ = std::move(row_idx);
    s.values_ = std::move(values);
    return s;  // canonical-form validation happens in the library on use
  }
  index_t rows() const { return rows_; }
  index_t cols() const { return cols_; }
  index_t nnz() const { return static_cast<index_t>(values_.size()); }
  const std::vector<index_t>& col_ptr() const { return col_ptr_; }
  const std::vector<index_t>& row_idx() const { return row_idx_; }
  const std::vector<double>& values() const { return values_; }
  lpca_matrix_view view() const {
    lpca_matrix_view v{};
    v.dtype = LPCA_F64;
    v.layout = LPCA_CSC;
    v.location = LPCA_HOST;
    v.rows = rows_;
    v.cols = cols_;
    v.data = values_.data();
    v.col_ptr = col_ptr_.data();
    v.row_idx = row_idx_.data();
    v.nnz = nnz();
    return v;
  }

 private:
  index_t rows_, cols_;
  std::vector<index_t> col_ptr_, row_idx_;
  std::vector<double> values_;
};

// ---- configuration (projection.hpp, reducer.hpp) -------------------------------------
enum class ProjectionKind { gaussian = LPCA_GAUSSIAN, very_sparse = LPCA_VERY_SPARSE };
enum class ReducerMethod { rp = LPCA_RP, spca = LPCA_SPCA, lazy_spca = LPCA_LAZY_SPCA };

inline std::string to_string(ReducerMethod m) {
  return m == ReducerMethod::rp ? "rp" : m == ReducerMethod::spca ? "spca" : "lazy_spca";
}
inline ReducerMethod reducer_method_from_string(const std::string& t) {
  if (t == "rp") return ReducerMethod::rp;
  if (t == "spca") return ReducerMethod::spca;
  if (t == "lazy_spca") return ReducerMethod::lazy_spca;
  throw InvalidArgumentError("unknown method '" + t + "' (expected rp, spca, or lazy_spca)");
}

struct DensityPolicy {
  enum class Mode { aggressive, conservative, explicit_value };
  Mode mode = Mode::conservative;
  double value = 0.0;
  static DensityPolicy aggressive() { return {Mode::aggressive, 0.0}; }
  static DensityPolicy conservative() { return {Mode::conservative, 0.0}; }
  static DensityPolicy explicit_value(double v) { return {Mode::explicit_value, v}; }
};

inline double density_for(const DensityPolicy& p, index_t k) {
  double out = 0.0;
  detail::check(lpca_density_for(static_cast<int32_t>(p.mode), k, p.value, &out));
  return out;
}

struct ProjectionSpec {
  ProjectionKind kind = ProjectionKind::gaussian;
  index_t n = 0;
  index_t l = 0;
  double density = 1.0;
  std::uint64_t seed = 0;
};

struct ReducerConfig {
  ReducerMethod method = ReducerMethod::spca;
  index_t k = 0;
  index_t l = 0;
  ProjectionSpec projection;
  index_t block_rows = 0;
  bool streaming = false;
  bool deterministic = true;
  int power_iters = 0;  // extension (not in the reference)

  lpca_config c_config() const {
    lpca_config c{};
    c.method = static_cast<int32_t>(method);
    c.projection_kind = static_cast<int32_t>(projection.kind);
    c.k = k;
    c.l = l;
    c.proj_n = projection.n;
    c.proj_l = projection.l;
    c.density = projection.density;
    c.seed = projection.seed;
    c.block_rows = block_rows;
    c.streaming = streaming;
    c.deterministic = deterministic;
    c.power_iters = power_iters;
    return c;
  }
  ReducerConfig resolved(index_t data_cols) const {
    const lpca_config in = c_config();
    lpca_config out{};
    detail::check(lpca_config_resolve(&in, data_cols, &out));
    ReducerConfig r = *this;
    r.l = out.l;
    r.projection.n = out.proj_n;
    r.projection.l = out.proj_l;
    r.streaming = out.streaming != 0;
    return r;
  }
};

struct ReducerTimings {
  double sketch = 0.0, qr = 0.0, f_form = 0.0, svd = 0.0, total = 0.0;
};

struct ReductionMap {
  std::string method;
  index_t k = 0, l = 0, n = 0;
  std::uint64_t seed = 0;
  double density = 1.0;
  double scale = 1.0;
  DenseMatrix v;
  std::vector<double> singular_values;
};

namespace detail {
inline ReductionMap to_host(lpca_map* m) {
  std::unique_ptr<lpca_map, lpca_status (*)(lpca_map*)> guard(m, lpca_map_destroy);
  lpca_map_info info{};
  check(lpca_map_info_get(m, &info));
  ReductionMap out;
  out.method = to_string(static_cast<ReducerMethod>(info.method));
  out.k = info.k;
  out.l = info.l;
  out.n = info.n;
  out.seed = info.seed;
  out.density = info.density;
  out.scale = info.scale;
  out.v = DenseMatrix(info.n, info.k);
  if (info.n * info.k > 0) check(lpca_map_copy_v(m, out.v.data(), LPCA_HOST));
  if (info.has_singular_values) {
    out.singular_values.resize(static_cast<std::size_t>(info.k));
    check(lpca_map_copy_sigma(m, out.singular_values.data()));
  }
  return out;
}
inline ReductionMap fit(const SparseMatrix& x, ReducerConfig cfg, ReducerMethod m, ReducerTimings* t) {
  cfg.method = m;
  const lpca_config c = cfg.c_config();
  const lpca_matrix_view v = x.view();
  lpca_map* out = nullptr;
  lpca_timings tm{};
  check(lpca_fit(ctx(), &c, &v, &out, &tm));
  if (t) {
    t->sketch += tm.sketch + tm.power;
    t->qr += tm.qr;
    t->f_form += tm.f_form;
    t->svd += tm.svd;
    t->total += tm.total + tm.h2d;
  }
  return to_host(out);
}
}  // namespace detail

// reducer.hpp:69-92
inline ReductionMap reduce_rp(const SparseMatrix& x, const ReducerConfig& c, ReducerTimings* t = nullptr) {
  return detail::fit(x, c, ReducerMethod::rp, t);
}
inline ReductionMap reduce_spca(const SparseMatrix& x, const ReducerConfig& c, ReducerTimings* t = nullptr) {
  return detail::fit(x, c, ReducerMethod::spca, t);
}
inline ReductionMap reduce_lazy_spca(const SparseMatrix& x, const ReducerConfig& c,
                                     ReducerTimings* t = nullptr) {
  return detail::fit(x, c, ReducerMethod::lazy_spca, t);
}
inline ReductionMap reduce(const SparseMatrix& x, const ReducerConfig& c, ReducerTimings* t = nullptr) {
  return detail::fit(x, c, c.method, t);
}

// ---- map files (reducer.hpp:96-99): the reference's byte format -------------------
inline void save_map_file(const ReductionMap& map, const std::string& path) {
  lpca_map_info info{};
  info.method = static_cast<int32_t>(reducer_method_from_string(map.method));
  info.k = map.k;
  info.l = map.l;
  info.n = map.n;
  info.seed = map.seed;
  info.density = map.density;
  info.scale = map.scale;
  info.has_singular_values = map.singular_values.empty() ? 0 : 1;
  detail::check(lpca_map_file_write(path.c_str(), &info, map.v.data(),
                                    map.singular_values.empty() ? nullptr : map.singular_values.data()));
}
inline ReductionMap load_map_file(const std::string& path) {
  lpca_map_info info{};
  detail::check(lpca_map_file_read(path.c_str(), &info, nullptr, 0, nullptr));
  ReductionMap out;
  out.method = to_string(static_cast<ReducerMethod>(info.method));
  out.k = info.k;
  out.l = info.l;
  out.n = info.n;
  out.seed = info.seed;
  out.density = info.density;
  out.scale = info.scale;
  out.v = DenseMatrix(info.n, info.k);
  if (info.has_singular_values) out.singular_values.resize(static_cast<std::size_t>(info.k));
  detail::check(lpca_map_file_read(path.c_str(), &info, out.v.data(), info.n * info.k,
                                   info.has_singular_values ? out.singular_values.data() : nullptr));
  return out;
}

// ---- streaming (sparse_matrix.hpp:53-79, reducer.hpp:82-85) -----------------------
struct RowBlock {
  index_t slice_index = 0;
  SparseMatrix block;
};
class RowBlockStream {
 public:
  virtual ~RowBlockStream() = default;
  virtual std::optional<RowBlock> next() = 0;
};
// Lazy row partition of an in-memory matrix (sparse_matrix.cpp:125-139).
class SliceRowBlockStream final : public RowBlockStream {
 public:
  SliceRowBlockStream(const SparseMatrix& x, index_t block_rows) : x_(&x), block_rows_(block_rows) {
    if (block_rows < 1) throw InvalidArgumentError("block_rows must be at least 1");
    slice_count_ = (x.rows() + block_rows - 1) / block_rows;
  }
  std::optional<RowBlock> next() override {
    if (next_slice_ >= slice_count_) return std::nullopt;
    const index_t lo = next_slice_ * block_rows_;
    const index_t hi = lo + block_rows_ < x_->rows() ? lo + block_rows_ : x_->rows();
    std::vector<index_t> cp{0}, ri;
    std::vector<double> va;
    for (index_t j = 0; j < x_->cols(); ++j) {  // rows are sorted within each column
      for (index_t p = x_->col_ptr()[j]; p < x_->col_ptr()[j + 1]; ++p) {
        const index_t r = x_->row_idx()[p];
        if (r >= lo && r < hi) {
          ri.push_back(r - lo);
          va.push_back(x_->values()[p]);
        }
      }
      cp.push_back(static_cast<index_t>(ri.size()));
    }
    RowBlock out{next_slice_, SparseMatrix::from_csc(hi - lo, x_->cols(), std::move(cp), std::move(ri), std::move(va))};
    ++next_slice_;
    return out;
  }

 private:
  const SparseMatrix* x_;
  index_t block_rows_, slice_count_ = 0, next_slice_ = 0;
};

// ---- matrix files (matrix_io.hpp), read and written by the library ----------------
namespace detail {
inline lpca_matrix_file* open_file(lpca_status (*reader)(const char*, lpca_matrix_file**), const std::string& p) {
  lpca_matrix_file* f = nullptr;
  check(reader(p.c_str(), &f));
  return f;
}
}  // namespace detail
inline SparseMatrix read_sparse_matrix_market_file(const std::string& path) {
  std::unique_ptr<lpca_matrix_file, void (*)(lpca_matrix_file*)> f(
      detail::open_file(lpca_read_sparse_matrix_market, path), lpca_matrix_file_free);
  int64_t r = 0, c = 0, z = 0;
  detail::check(lpca_matrix_file_info(f.get(), &r, &c, &z));
  std::vector<index_t> cp(static_cast<std::size_t>(c) + 1), ri(static_cast<std::size_t>(z));
  std::vector<double> va(static_cast<std::size_t>(z));
  detail::check(lpca_matrix_file_copy(f.get(), cp.data(), ri.data(), va.data()));
  return SparseMatrix::from_csc(r, c, std::move(cp), std::move(ri), std::move(va));
}
namespace detail {
inline DenseMatrix read_dense(lpca_status (*reader)(const char*, lpca_matrix_file**), const std::string& path) {
  std::unique_ptr<lpca_matrix_file, void (*)(lpca_matrix_file*)> f(open_file(reader, path), lpca_matrix_file_free);
  int64_t r = 0, c = 0, z = 0;
  check(lpca_matrix_file_info(f.get(), &r, &c, &z));
  DenseMatrix out(r, c);
  check(lpca_matrix_file_copy(f.get(), nullptr, nullptr, out.data()));
  return out;
}
}  // namespace detail
inline DenseMatrix read_dense_matrix_market_file(const std::string& path) {
  return detail::read_dense(lpca_read_dense_matrix_market, path);
}
inline DenseMatrix read_dense_csv_file(const std::string& path) { return detail::read_dense(lpca_read_dense_csv, path); }
inline void write_sparse_matrix_market_file(const SparseMatrix& x, const std::string& path) {
  detail::check(lpca_write_sparse_matrix_market(path.c_str(), x.rows(), x.cols(), x.col_ptr().data(),
                                                x.row_idx().data(), x.values().data()));
}
inline void write_dense_matrix_market_file(const DenseMatrix& x, const std::string& path) {
  detail::check(lpca_write_dense_matrix_market(path.c_str(), x.rows(), x.cols(), x.data()));
}
inline void write_dense_csv_file(const DenseMatrix& x, const std::string& path) {
  detail::check(lpca_write_dense_csv(path.c_str(), x.rows(), x.cols(), x.data()));
}

// Row blocks straight from a file (matrix_io.hpp:41-80). The streaming reducers
// drive these natively; next() also works (a copy of the block as CSC).
class FileRowBlockStream : public RowBlockStream {
 public:
  ~FileRowBlockStream() override { lpca_file_stream_close(s_); }
  FileRowBlockStream(const FileRowBlockStream&) = delete;
  FileRowBlockStream& operator=(const FileRowBlockStream&) = delete;
  lpca_file_stream* handle() const { return s_; }
  std::optional<RowBlock> next() override {
    lpca_matrix_view v{};
    int64_t slice = 0;
    const int32_t r = lpca_file_stream_next(s_, &v, &slice);
    if (r < 0) detail::check(static_cast<lpca_status>(-r));
    if (r == 0) return std::nullopt;
    std::vector<index_t> cp, ri;
    std::vector<double> va;
    if (v.layout == LPCA_CSC) {
      cp.assign(v.col_ptr, v.col_ptr + v.cols + 1);
      ri.assign(v.row_idx, v.row_idx + v.nnz);
      const double* d = static_cast<const double*>(v.data);
      va.assign(d, d + v.nnz);
    } else {  // dense row-major block (CSV): the reference's sparsified form
      const double* d = static_cast<const double*>(v.data);
      cp.assign(static_cast<std::size_t>(v.cols) + 1, 0);
      for (index_t j = 0; j < v.cols; ++j) {
        for (index_t i = 0; i < v.rows; ++i)
          if (d[i * v.ld + j] != 0.0) {
            ri.push_back(i);
            va.push_back(d[i * v.ld + j]);
          }
        cp[static_cast<std::size_t>(j) + 1] = static_cast<index_t>(ri.size());
      }
    }
    return RowBlock{slice, SparseMatrix::from_csc(v.rows, v.cols, std::move(cp), std::move(ri), std::move(va))};
  }

 protected:
  explicit FileRowBlockStream(lpca_file_stream* s) : s_(s) {}

 private:
  lpca_file_stream* s_;
};
class MatrixMarketRowBlockStream final : public FileRowBlockStream {
 public:
  MatrixMarketRowBlockStream(const std::string& path, index_t block_rows)
      : FileRowBlockStream(open(path, block_rows)) {}

 private:
  static lpca_file_stream* open(const std::string& path, index_t block_rows) {
    lpca_file_stream* s = nullptr;
    detail::check(lpca_open_matrix_market_stream(path.c_str(), block_rows, &s));
    return s;
  }
};
class CsvRowBlockStream final : public FileRowBlockStream {
 public:
  CsvRowBlockStream(const std::string& path, index_t block_rows) : FileRowBlockStream(open(path, block_rows)) {}

 private:
  static lpca_file_stream* open(const std::string& path, index_t block_rows) {
    lpca_file_stream* s = nullptr;
    detail::check(lpca_open_csv_stream(path.c_str(), block_rows, &s));
    return s;
  }
};

namespace detail {
struct StreamPump {  // lpca_next_block_fn over a RowBlockStream; keeps the current block alive
  RowBlockStream* s;
  std::optional<RowBlock> cur;
  std::exception_ptr err;
  static int32_t next(void* self, lpca_matrix_view* v, int64_t* slice) {
    auto* p = static_cast<StreamPump*>(self);
    try {
      p->cur = p->s->next();
      if (!p->cur) return 0;
      *v = p->cur->block.view();
      *slice = p->cur->slice_index;
      return 1;
    } catch (...) {
      p->err = std::current_exception();
      return -1;
    }
  }
};
inline ReductionMap fit_stream(RowBlockStream& blocks, ReducerConfig cfg, ReducerMethod m, ReducerTimings* t) {
  cfg.method = m;
  const lpca_config c = cfg.c_config();
  StreamPump pump{&blocks, std::nullopt, nullptr};
  lpca_map* out = nullptr;
  lpca_timings tm{};
  auto* file = dynamic_cast<FileRowBlockStream*>(&blocks);  // file streams run natively
  const lpca_status st = file ? lpca_fit_stream(ctx(), &c, &lpca_file_stream_next, file->handle(), &out, &tm)
                              : lpca_fit_stream(ctx(), &c, &StreamPump::next, &pump, &out, &tm);
  if (pump.err) std::rethrow_exception(pump.err);
  check(st);
  if (t) {
    t->sketch += tm.sketch;
    t->qr += tm.qr;
    t->f_form += tm.f_form;
    t->svd += tm.svd;
    t->total += tm.total;
  }
  return to_host(out);
}
}  // namespace detail

// reduce_{spca,lazy_spca}_streaming (reducer.hpp:82-85, reducer.cpp:236-335)
inline ReductionMap reduce_spca_streaming(RowBlockStream& blocks, const ReducerConfig& c,
                                          ReducerTimings* t = nullptr) {
  return detail::fit_stream(blocks, c, ReducerMethod::spca, t);
}
inline ReductionMap reduce_lazy_spca_streaming(RowBlockStream& blocks, const ReducerConfig& c,
                                               ReducerTimings* t = nullptr) {
  return detail::fit_stream(blocks, c, ReducerMethod::lazy_spca, t);
}

inline DenseMatrix apply_map(const ReductionMap& map, const SparseMatrix& x) {
  lpca_map_info info{};
  info.method = static_cast<int32_t>(reducer_method_from_string(map.method));
  info.k = map.k;
  info.l = map.l;
  info.n = map.n;
  info.seed = map.seed;
  info.density = map.density;
  info.scale = map.scale;
  lpca_map* m = nullptr;
  detail::check(lpca_map_create(detail::ctx(), &info, map.v.data(), nullptr, &m));
  std::unique_ptr<lpca_map, lpca_status (*)(lpca_map*)> guard(m, lpca_map_destroy);
  DenseMatrix y(x.rows(), map.k);
  const lpca_matrix_view v = x.view();
  detail::check(lpca_transform(detail::ctx(), m, &v, y.data(), LPCA_F64, LPCA_COL_MAJOR, LPCA_HOST, 0, nullptr));
  return y;
}

// projection.hpp:48-72 (dense representation of either family)
struct ProjectionMatrix {
  ProjectionSpec spec;
  double scale = 1.0;
  DenseMatrix omega;
};
inline ProjectionMatrix regenerate(const ProjectionSpec& s) {
  ProjectionMatrix p;
  p.spec = s;
  p.omega = DenseMatrix(s.n, s.l);
  detail::check(lpca_regenerate(detail::ctx(), static_cast<int32_t>(s.kind), s.n, s.l, s.density, s.seed,
                                p.omega.data(), LPCA_HOST, &p.scale));
  return p;
}

// kernels.hpp:17-36 (fp64, reference summation order)
inline DenseMatrix spmm(const SparseMatrix& a, const DenseMatrix& b) {
  DenseMatrix out(a.rows(), b.cols());
  const lpca_matrix_view v = a.view();
  detail::check(lpca_spmm(detail::ctx(), &v, b.data(), b.cols(), LPCA_HOST, out.data(), LPCA_HOST));
  return out;
}
inline DenseMatrix gemm_t(const DenseMatrix& u, const SparseMatrix& x) {
  DenseMatrix out(u.cols(), x.cols());
  const lpca_matrix_view v = x.view();
  detail::check(lpca_gemm_t(detail::ctx(), u.data(), u.rows(), u.cols(), LPCA_HOST, &v, out.data(), LPCA_HOST));
  return out;
}
inline DenseMatrix dense_aat(const DenseMatrix& f) {
  DenseMatrix out(f.rows(), f.rows());
  detail::check(lpca_dense_aat(detail::ctx(), f.data(), f.rows(), f.cols(), LPCA_HOST, out.data()));
  return out;
}

struct TruncatedSVD {
  DenseMatrix u_tilde;
  std::vector<double> singular_values;
  DenseMatrix v;
};
inline TruncatedSVD truncated_svd_via_gram(const DenseMatrix& f, index_t k) {
  TruncatedSVD s;
  s.singular_values.resize(static_cast<std::size_t>(k > 0 ? k : 0));
  s.v = DenseMatrix(f.cols(), k);
  s.u_tilde = DenseMatrix(f.rows(), k);
  detail::check(lpca_truncated_svd_via_gram(detail::ctx(), f.data(), f.rows(), f.cols(), k, LPCA_HOST,
                                            s.singular_values.data(), s.v.data(), s.u_tilde.data()));
  return s;
}

}  // namespace lazypca
