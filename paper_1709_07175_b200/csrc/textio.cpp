// Text formats around the reducer: MatrixMarket
// coordinate / array files, CSV, row-block streams over them for
// lpca_fit_stream, and map files. Host-only translation unit (g++).
//
// The formats' rules, as the reference applies them (proj/core/src/matrix_io.cpp,
// reducer.cpp:355-412), restated here:
//  * MatrixMarket: a banner `%%MatrixMarket matrix <coordinate|array>
//    <real|integer|double> general` (words compared case-insensitively), then
//    '%' comment lines and blank lines, then the size line (rows cols [nnz]:
//    exactly that many integers), then the payload. Coordinate entries are
//    `row col value`, 1-based, range-checked against the size line; every line
//    is parsed (comments and blank lines skipped) and the entry count must equal
//    nnz. Array payloads are whitespace-separated values, column-major, exactly
//    rows x cols of them.
//  * Values are strtod numbers and must be finite.
//  * Coordinate data becomes canonical CSC: entries ordered by (column, row),
//    duplicates summed, zero sums dropped (SparseMatrix::from_triplets).
//  * CSV: one row per non-blank line, ',' between values, all rows as long as
//    the first.
//  * Writers print each value in the shortest "%.<p>g" form that reads back to
//    the same double.
//  * Map files: one JSON line {method, k, l, seed, density, c, n[,
//    singular_values]} (nlohmann/json's ordered serialiser, the reference's own),
//    then V as a dense MatrixMarket array whose line numbers restart at 1.
// Errors are ParseErrors carrying the line number, with the reference's
// messages, which callers match on.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "../../include/lazypca_b200.h"
#include "common.cuh"

using lpca::Error;
using lpca::index_t;

struct lpca_matrix_file {
  bool sparse = false;
  index_t rows = 0, cols = 0;
  std::vector<std::int64_t> col_ptr, row_idx;  // CSC (sparse)
  std::vector<double> values;                  // CSC values, or dense column-major
};

namespace {

[[noreturn]] void fail(const std::string& what, std::int64_t line) { throw Error(lpca::kParse, what, line); }

// ---- input: a file read line by line, with a resettable line counter ---------
class TextFile {
 public:
  explicit TextFile(const std::string& path) : path_(path), fp_(std::fopen(path.c_str(), "r")) {
    if (!fp_) fail("cannot open '" + path + "' for reading", 0);
  }
  ~TextFile() {
    std::free(buf_);
    if (fp_) std::fclose(fp_);
  }
  TextFile(const TextFile&) = delete;
  TextFile& operator=(const TextFile&) = delete;

  // The next line without its '\n'; false at end of file.
  bool next(std::string& line) {
    const ssize_t got = ::getline(&buf_, &cap_, fp_);
    if (got < 0) return false;
    std::size_t len = static_cast<std::size_t>(got);
    if (len > 0 && buf_[len - 1] == '\n') --len;
    line.assign(buf_, len);
    ++line_no_;
    return true;
  }
  std::int64_t line_no() const { return line_no_; }
  void restart_count() { line_no_ = 0; }
  const std::string& path() const { return path_; }

 private:
  std::string path_;
  std::FILE* fp_ = nullptr;
  char* buf_ = nullptr;
  std::size_t cap_ = 0;
  std::int64_t line_no_ = 0;
};

bool is_space(char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; }

bool all_space(const std::string& s) {
  return std::all_of(s.begin(), s.end(), [](char c) { return is_space(c); });
}

bool is_comment(const std::string& s) { return !s.empty() && s[0] == '%'; }

// ---- a cursor over one line --------------------------------------------------
class Cursor {
 public:
  Cursor(const std::string& s, std::int64_t line) : p_(s.c_str()), line_(line) {}
  void skip_space() {
    while (is_space(*p_)) ++p_;
  }
  bool at_end() {
    skip_space();
    return *p_ == '\0';
  }
  char peek() const { return *p_; }
  void advance() { ++p_; }
  // A whitespace-delimited word ("" at the end of the line).
  std::string word() {
    skip_space();
    const char* b = p_;
    while (*p_ && !is_space(*p_)) ++p_;
    return std::string(b, p_);
  }
  // strtoll; false (cursor unmoved) when no digits follow.
  bool integer(long long* out) {
    char* e = nullptr;
    errno = 0;
    const long long v = std::strtoll(p_, &e, 10);
    if (e == p_) return false;
    p_ = e;
    *out = v;
    return true;
  }
  // A finite strtod value.
  double real() {
    char* e = nullptr;
    errno = 0;
    const double v = std::strtod(p_, &e);
    if (e == p_) fail("expected a numeric value", line_);
    if (!std::isfinite(v)) fail("non-finite value", line_);
    p_ = e;
    return v;
  }

 private:
  const char* p_;
  std::int64_t line_;
};

std::string to_lower(std::string s) {
  std::transform(s.begin(), s.end(), s.begin(), [](char c) { return static_cast<char>(std::tolower(static_cast<unsigned char>(c))); });
  return s;
}

// ---- MatrixMarket -------------------------------------------------------------
struct MmHead {
  bool coordinate = false;
  std::int64_t size[3] = {0, 0, 0};
};

// Banner, comments and blank lines, then the size line's `count` integers.
// `want_coordinate`: -1 either, 0 array, 1 coordinate (checked after the size
// line is found, before it is parsed).
MmHead read_mm_head(TextFile& f, int count, int want_coordinate) {
  std::string line;
  if (!f.next(line)) fail("empty MatrixMarket file", 1);
  Cursor c(line, f.line_no());
  const std::string tag = c.word(), object = c.word(), format = c.word(), field = c.word(), sym = c.word();
  if (to_lower(tag) != "%%matrixmarket") fail("missing %%MatrixMarket banner", f.line_no());
  if (to_lower(object) != "matrix") fail("unsupported MatrixMarket object '" + object + "'", f.line_no());
  MmHead h;
  const std::string fmt = to_lower(format);
  if (fmt != "coordinate" && fmt != "array") fail("unsupported MatrixMarket format '" + format + "'", f.line_no());
  h.coordinate = fmt == "coordinate";
  const std::string fld = to_lower(field);
  if (fld != "real" && fld != "integer" && fld != "double")
    fail("unsupported MatrixMarket field '" + field + "'", f.line_no());
  if (to_lower(sym) != "general") fail("unsupported MatrixMarket symmetry '" + sym + "'", f.line_no());
  bool found = false;
  while (f.next(line)) {
    if (is_comment(line) || all_space(line)) continue;
    found = true;
    break;
  }
  if (!found) fail("MatrixMarket file ends before the size line", f.line_no());
  if (want_coordinate == 1 && !h.coordinate) fail("expected a coordinate (sparse) MatrixMarket file", f.line_no());
  if (want_coordinate == 0 && h.coordinate) fail("expected an array (dense) MatrixMarket file", f.line_no());
  Cursor s(line, f.line_no());
  for (int i = 0; i < count; ++i) {
    long long v = 0;
    s.skip_space();
    if (!s.integer(&v) || errno == ERANGE) fail("expected " + std::to_string(count) + " integers", f.line_no());
    h.size[i] = v;
  }
  if (!s.at_end()) fail("trailing tokens after size line", f.line_no());
  for (int i = 0; i < count; ++i)
    if (h.size[i] < 0) fail("negative size entry", f.line_no());
  return h;
}

struct Triple {
  index_t row, col;
  double value;
};

// One coordinate entry; false for a blank line.
bool coordinate_entry(const std::string& line, std::int64_t line_no, index_t rows, index_t cols, Triple& t) {
  if (all_space(line)) return false;
  Cursor c(line, line_no);
  long long i = 0, j = 0;
  if (!c.integer(&i)) fail("expected row index", line_no);
  if (!c.integer(&j)) fail("expected column index", line_no);
  t.value = c.real();
  if (!c.at_end()) fail("trailing tokens after entry", line_no);
  if (i < 1 || i > rows) fail("row index " + std::to_string(i) + " outside 1.." + std::to_string(rows), line_no);
  if (j < 1 || j > cols) fail("column index " + std::to_string(j) + " outside 1.." + std::to_string(cols), line_no);
  t.row = static_cast<index_t>(i - 1);
  t.col = static_cast<index_t>(j - 1);
  return true;
}

// Walks every coordinate entry after the head (comment and blank lines skipped).
template <typename Visit>
std::int64_t for_each_entry(TextFile& f, index_t rows, index_t cols, Visit&& visit) {
  std::string line;
  std::int64_t count = 0;
  while (f.next(line)) {
    if (is_comment(line)) continue;
    Triple t;
    if (!coordinate_entry(line, f.line_no(), rows, cols, t)) continue;
    visit(t);
    ++count;
  }
  return count;
}

void check_entry_count(std::int64_t seen, std::int64_t nnz, std::int64_t line_no) {
  if (seen != nnz)
    fail("entry count " + std::to_string(seen) + " does not match header nnz " + std::to_string(nnz), line_no);
}

// Canonical CSC of a triple list (the same std::sort order on the same input as
// from_triplets, so duplicates are summed in the same order and round alike).
void build_csc(index_t rows, index_t cols, std::vector<Triple>& ts, lpca_matrix_file& out) {
  std::sort(ts.begin(), ts.end(), [](const Triple& a, const Triple& b) { return a.col != b.col ? a.col < b.col : a.row < b.row; });
  out.sparse = true;
  out.rows = rows;
  out.cols = cols;
  out.col_ptr.assign(static_cast<std::size_t>(cols) + 1, 0);
  out.row_idx.clear();
  out.values.clear();
  std::size_t p = 0;
  for (index_t j = 0; j < cols; ++j) {
    while (p < ts.size() && ts[p].col == j) {
      const index_t r = ts[p].row;
      double sum = 0.0;
      bool firstv = true;
      for (; p < ts.size() && ts[p].col == j && ts[p].row == r; ++p) {
        sum = firstv ? ts[p].value : sum + ts[p].value;
        firstv = false;
      }
      if (sum != 0.0) {
        out.row_idx.push_back(r);
        out.values.push_back(sum);
      }
    }
    out.col_ptr[static_cast<std::size_t>(j) + 1] = static_cast<std::int64_t>(out.row_idx.size());
  }
}

std::unique_ptr<lpca_matrix_file> read_coordinate(const std::string& path) {
  TextFile f(path);
  const MmHead h = read_mm_head(f, 3, 1);
  std::vector<Triple> ts;
  ts.reserve(static_cast<std::size_t>(h.size[2]));
  const std::int64_t seen = for_each_entry(f, h.size[0], h.size[1], [&](const Triple& t) { ts.push_back(t); });
  check_entry_count(seen, h.size[2], f.line_no());
  auto out = std::make_unique<lpca_matrix_file>();
  build_csc(h.size[0], h.size[1], ts, *out);
  return out;
}

// An array payload (column-major values) after the head.
std::vector<double> read_array_payload(TextFile& f, std::int64_t rows, std::int64_t cols) {
  std::vector<double> data;
  data.reserve(static_cast<std::size_t>(rows * cols));
  std::string line;
  while (f.next(line)) {
    if (is_comment(line) || all_space(line)) continue;
    Cursor c(line, f.line_no());
    while (!c.at_end()) data.push_back(c.real());
  }
  if (static_cast<std::int64_t>(data.size()) != rows * cols)
    fail("array payload has " + std::to_string(data.size()) + " values, expected " + std::to_string(rows * cols),
         f.line_no());
  return data;
}

std::unique_ptr<lpca_matrix_file> read_array(const std::string& path) {
  TextFile f(path);
  const MmHead h = read_mm_head(f, 2, 0);
  auto out = std::make_unique<lpca_matrix_file>();
  out->rows = h.size[0];
  out->cols = h.size[1];
  out->values = read_array_payload(f, h.size[0], h.size[1]);
  return out;
}

// ---- CSV ------------------------------------------------------------------------
void csv_row(const std::string& line, std::int64_t line_no, std::vector<double>& row) {
  row.clear();
  Cursor c(line, line_no);
  for (;;) {
    row.push_back(c.real());
    if (c.at_end()) return;
    if (c.peek() != ',') fail("expected ',' between values", line_no);
    c.advance();
  }
}

void check_width(std::size_t got, std::size_t want, std::int64_t line_no) {
  if (got != want) fail("row has " + std::to_string(got) + " values, expected " + std::to_string(want), line_no);
}

std::unique_ptr<lpca_matrix_file> read_csv(const std::string& path) {
  TextFile f(path);
  std::vector<double> rowmajor, row;
  std::size_t width = 0;
  index_t rows = 0;
  std::string line;
  while (f.next(line)) {
    if (all_space(line)) continue;
    csv_row(line, f.line_no(), row);
    if (rows == 0) width = row.size();
    check_width(row.size(), width, f.line_no());
    rowmajor.insert(rowmajor.end(), row.begin(), row.end());
    ++rows;
  }
  auto out = std::make_unique<lpca_matrix_file>();
  out->rows = rows;
  out->cols = static_cast<index_t>(width);
  out->values.resize(rowmajor.size());
  for (index_t i = 0; i < rows; ++i)
    for (index_t j = 0; j < out->cols; ++j)
      out->values[static_cast<std::size_t>(j * rows + i)] = rowmajor[static_cast<std::size_t>(i * out->cols + j)];
  return out;
}

// ---- output -----------------------------------------------------------------------
// Shortest "%.<p>g" spelling that strtod reads back as the same double.
class Shortest {
 public:
  const char* operator()(double v) {
    for (int p = 1; p <= 17; ++p) {
      std::snprintf(buf_, sizeof buf_, "%.*g", p, v);
      if (std::strtod(buf_, nullptr) == v) break;
    }
    return buf_;
  }

 private:
  char buf_[40];
};

class TextOut {
 public:
  explicit TextOut(const std::string& path) : fp_(std::fopen(path.c_str(), "w")) {
    if (!fp_) fail("cannot open '" + path + "' for writing", 0);
  }
  ~TextOut() {
    if (fp_) std::fclose(fp_);
  }
  TextOut(const TextOut&) = delete;
  TextOut& operator=(const TextOut&) = delete;
  TextOut& str(const char* s) {
    std::fputs(s, fp_);
    return *this;
  }
  TextOut& str(const std::string& s) { return str(s.c_str()); }
  TextOut& num(long long v) {
    std::fprintf(fp_, "%lld", v);
    return *this;
  }
  TextOut& real(double v) { return str(fmt_(v)); }
  TextOut& ch(char c) {
    std::fputc(c, fp_);
    return *this;
  }
  bool ok() const { return fp_ && !std::ferror(fp_); }

 private:
  std::FILE* fp_;
  Shortest fmt_;
};

void write_array(TextOut& o, std::int64_t rows, std::int64_t cols, const double* colmajor) {
  o.str("%%MatrixMarket matrix array real general\n").num(rows).ch(' ').num(cols).ch('\n');
  for (std::int64_t e = 0; e < rows * cols; ++e) o.real(colmajor[e]).ch('\n');
}

// ---- row-block streams ---------------------------------------------------------
}  // namespace

struct lpca_file_stream {
  virtual ~lpca_file_stream() = default;
  virtual bool next(lpca_matrix_view* v, int64_t* slice) = 0;
};

namespace {

// MatrixMarketRowBlockStream: validated and counted once at open; each block is
// one more scan of the file keeping the rows of its slice.
class CoordinateBlocks final : public lpca_file_stream {
 public:
  CoordinateBlocks(const std::string& path, index_t block_rows) : path_(path), block_rows_(block_rows) {
    TextFile f(path);
    const MmHead h = read_mm_head(f, 3, 1);
    rows_ = h.size[0];
    cols_ = h.size[1];
    blocks_ = rows_ == 0 ? 0 : (rows_ + block_rows - 1) / block_rows;
    per_block_.assign(static_cast<std::size_t>(std::max<index_t>(blocks_, 1)), 0);
    const std::int64_t seen =
        for_each_entry(f, rows_, cols_, [&](const Triple& t) { ++per_block_[static_cast<std::size_t>(t.row / block_rows_)]; });
    check_entry_count(seen, h.size[2], f.line_no());
  }
  bool next(lpca_matrix_view* v, int64_t* slice) override {
    if (done_ >= blocks_) return false;
    const index_t s = done_++;
    const index_t lo = s * block_rows_, hi = std::min(rows_, lo + block_rows_);
    TextFile f(path_);
    read_mm_head(f, 3, 1);
    std::vector<Triple> ts;
    ts.reserve(static_cast<std::size_t>(per_block_[static_cast<std::size_t>(s)]));
    for_each_entry(f, rows_, cols_, [&](const Triple& t) {
      if (t.row >= lo && t.row < hi) ts.push_back(Triple{t.row - lo, t.col, t.value});
    });
    build_csc(hi - lo, cols_, ts, block_);
    *v = lpca_matrix_view{LPCA_F64, LPCA_CSC, LPCA_HOST, 0, hi - lo, cols_, 0, block_.values.data(),
                          block_.col_ptr.data(), block_.row_idx.data(), static_cast<int64_t>(block_.values.size())};
    *slice = s;
    return true;
  }

 private:
  std::string path_;
  index_t block_rows_, rows_ = 0, cols_ = 0, blocks_ = 0, done_ = 0;
  std::vector<std::int64_t> per_block_;
  lpca_matrix_file block_;
};

// CsvRowBlockStream: reads on through the file; the first row is parsed at open
// (it fixes the width). Blocks go out dense row-major fp64.
class CsvBlocks final : public lpca_file_stream {
 public:
  CsvBlocks(const std::string& path, index_t block_rows) : file_(path), block_rows_(block_rows) {
    std::string line;
    while (file_.next(line)) {
      if (all_space(line)) continue;
      csv_row(line, file_.line_no(), first_);
      width_ = first_.size();
      have_first_ = true;
      return;
    }
    ended_ = true;
  }
  bool next(lpca_matrix_view* v, int64_t* slice) override {
    if (ended_) return false;
    block_.clear();
    index_t filled = 0;
    if (have_first_) {
      block_ = first_;
      have_first_ = false;
      filled = 1;
    }
    std::string line;
    while (filled < block_rows_ && file_.next(line)) {
      if (all_space(line)) continue;
      csv_row(line, file_.line_no(), row_);
      check_width(row_.size(), width_, file_.line_no());
      block_.insert(block_.end(), row_.begin(), row_.end());
      ++filled;
    }
    if (filled < block_rows_) ended_ = true;
    if (filled == 0) return false;
    const index_t w = static_cast<index_t>(width_);
    *v = lpca_matrix_view{LPCA_F64, LPCA_ROW_MAJOR, LPCA_HOST, 0, filled, w, w, block_.data(), nullptr, nullptr, 0};
    *slice = next_slice_++;
    return true;
  }

 private:
  TextFile file_;
  index_t block_rows_, next_slice_ = 0;
  std::size_t width_ = 0;
  std::vector<double> first_, row_, block_;
  bool have_first_ = false, ended_ = false;
};

// ---- map files -------------------------------------------------------------------
const char* method_name(int32_t m) {
  if (m == LPCA_RP) return "rp";
  if (m == LPCA_SPCA) return "spca";
  if (m == LPCA_LAZY_SPCA) return "lazy_spca";
  throw Error(lpca::kInvalidArgument, "unknown reducer method " + std::to_string(m));
}

int32_t method_of(const std::string& s) {
  for (int32_t m : {LPCA_RP, LPCA_SPCA, LPCA_LAZY_SPCA})
    if (s == method_name(m)) return m;
  throw Error(lpca::kInvalidArgument, "unknown reducer method '" + s + "'");
}

struct MapFile {
  lpca_map_info info{};
  std::vector<double> v, sigma;
};

MapFile parse_map(const std::string& path) {
  TextFile f(path);
  std::string line;
  if (!f.next(line)) fail("map file is empty", 1);
  MapFile m;
  try {
    const nlohmann::json h = nlohmann::json::parse(line);
    m.info.method = method_of(h.at("method").get<std::string>());
    m.info.k = h.at("k").get<index_t>();
    m.info.l = h.at("l").get<index_t>();
    m.info.seed = h.at("seed").get<std::uint64_t>();
    m.info.density = h.at("density").get<double>();
    m.info.scale = h.at("c").get<double>();
    m.info.n = h.at("n").get<index_t>();
    if (h.contains("singular_values")) {
      m.sigma = h.at("singular_values").get<std::vector<double>>();
      m.info.has_singular_values = 1;
    }
  } catch (const nlohmann::json::exception& e) {
    fail(std::string("map header: ") + e.what(), 1);
  }
  f.restart_count();  // the payload is read as a file of its own
  const MmHead a = read_mm_head(f, 2, 0);
  m.v = read_array_payload(f, a.size[0], a.size[1]);
  if (a.size[0] != m.info.n || a.size[1] != m.info.k)
    throw Error(lpca::kDimension, "map payload is " + std::to_string(a.size[0]) + "x" + std::to_string(a.size[1]) +
                                      " but the header says " + std::to_string(m.info.n) + "x" +
                                      std::to_string(m.info.k));
  if (m.info.has_singular_values && static_cast<index_t>(m.sigma.size()) != m.info.k)
    throw Error(lpca::kDimension, "map header: singular_values length does not match k");
  return m;
}

void emit_map(const std::string& path, const lpca_map_info& info, const double* v, const double* sigma) {
  nlohmann::ordered_json h;
  h["method"] = method_name(info.method);
  h["k"] = info.k;
  h["l"] = info.l;
  h["seed"] = info.seed;
  h["density"] = info.density;
  h["c"] = info.scale;
  h["n"] = info.n;
  if (info.has_singular_values && sigma) h["singular_values"] = std::vector<double>(sigma, sigma + info.k);
  TextOut o(path);
  o.str(h.dump()).ch('\n');
  write_array(o, info.n, info.k, v);
  if (!o.ok()) fail("write to '" + path + "' failed", 0);
}

template <typename F>
lpca_status guarded(F&& fn) {
  try {
    fn();
    return LPCA_OK;
  } catch (const Error& e) {
    lpca::set_last_error(e.what(), e.index, e.gap);
    return static_cast<lpca_status>(e.code);
  } catch (const std::exception& e) {
    lpca::set_last_error(e.what(), -1, 0.0);
    return LPCA_ERR_INTERNAL;
  }
}

void need(bool ok) {
  if (!ok) throw Error(lpca::kInvalidArgument, "null argument");
}

void need_block_rows(int64_t block_rows) {
  if (block_rows < 1) throw Error(lpca::kInvalidArgument, "block_rows must be at least 1");
}

}  // namespace

// ================================ C ABI ============================================
extern "C" {

lpca_status lpca_read_sparse_matrix_market(const char* path, lpca_matrix_file** out) {
  return guarded([&] {
    need(path && out);
    *out = read_coordinate(path).release();
  });
}

lpca_status lpca_read_dense_matrix_market(const char* path, lpca_matrix_file** out) {
  return guarded([&] {
    need(path && out);
    *out = read_array(path).release();
  });
}

lpca_status lpca_read_dense_csv(const char* path, lpca_matrix_file** out) {
  return guarded([&] {
    need(path && out);
    *out = read_csv(path).release();
  });
}

lpca_status lpca_matrix_file_info(const lpca_matrix_file* f, int64_t* rows, int64_t* cols, int64_t* nnz) {
  return guarded([&] {
    if (!f) throw Error(lpca::kInvalidArgument, "null matrix file");
    if (rows) *rows = f->rows;
    if (cols) *cols = f->cols;
    if (nnz) *nnz = f->sparse ? static_cast<int64_t>(f->values.size()) : -1;
  });
}

lpca_status lpca_matrix_file_copy(const lpca_matrix_file* f, int64_t* col_ptr, int64_t* row_idx, double* values) {
  return guarded([&] {
    if (!f) throw Error(lpca::kInvalidArgument, "null matrix file");
    if (f->sparse && col_ptr) std::copy(f->col_ptr.begin(), f->col_ptr.end(), col_ptr);
    if (f->sparse && row_idx) std::copy(f->row_idx.begin(), f->row_idx.end(), row_idx);
    if (values) std::copy(f->values.begin(), f->values.end(), values);
  });
}

lpca_status lpca_matrix_file_view(const lpca_matrix_file* f, lpca_matrix_view* out) {
  return guarded([&] {
    need(f && out);
    *out = f->sparse ? lpca_matrix_view{LPCA_F64, LPCA_CSC, LPCA_HOST, 0, f->rows, f->cols, 0, f->values.data(),
                                        f->col_ptr.data(), f->row_idx.data(), static_cast<int64_t>(f->values.size())}
                     : lpca_matrix_view{LPCA_F64, LPCA_COL_MAJOR, LPCA_HOST, 0, f->rows, f->cols, f->rows,
                                        f->values.data(), nullptr, nullptr, 0};
  });
}

void lpca_matrix_file_free(lpca_matrix_file* f) { delete f; }

lpca_status lpca_write_sparse_matrix_market(const char* path, int64_t rows, int64_t cols, const int64_t* col_ptr,
                                            const int64_t* row_idx, const double* values) {
  return guarded([&] {
    need(path && (cols == 0 || col_ptr));
    TextOut o(path);
    o.str("%%MatrixMarket matrix coordinate real general\n").num(rows).ch(' ').num(cols).ch(' ');
    o.num(cols > 0 ? col_ptr[cols] : 0).ch('\n');
    for (int64_t j = 0; j < cols; ++j)
      for (int64_t p = col_ptr[j]; p < col_ptr[j + 1]; ++p) o.num(row_idx[p] + 1).ch(' ').num(j + 1).ch(' ').real(values[p]).ch('\n');
  });
}

lpca_status lpca_write_dense_matrix_market(const char* path, int64_t rows, int64_t cols, const double* colmajor) {
  return guarded([&] {
    need(path && (rows * cols == 0 || colmajor));
    TextOut o(path);
    write_array(o, rows, cols, colmajor);
  });
}

lpca_status lpca_write_dense_csv(const char* path, int64_t rows, int64_t cols, const double* colmajor) {
  return guarded([&] {
    need(path && (rows * cols == 0 || colmajor));
    TextOut o(path);
    for (int64_t i = 0; i < rows; ++i) {
      for (int64_t j = 0; j < cols; ++j) {
        if (j > 0) o.ch(',');
        o.real(colmajor[j * rows + i]);
      }
      o.ch('\n');
    }
  });
}

lpca_status lpca_open_matrix_market_stream(const char* path, int64_t block_rows, lpca_file_stream** out) {
  return guarded([&] {
    need(path && out);
    need_block_rows(block_rows);
    *out = new CoordinateBlocks(path, block_rows);
  });
}

lpca_status lpca_open_csv_stream(const char* path, int64_t block_rows, lpca_file_stream** out) {
  return guarded([&] {
    need(path && out);
    need_block_rows(block_rows);
    *out = new CsvBlocks(path, block_rows);
  });
}

int32_t lpca_file_stream_next(void* user, lpca_matrix_view* block, int64_t* slice) {
  try {
    auto* s = static_cast<lpca_file_stream*>(user);
    need(s && block && slice);
    return s->next(block, slice) ? 1 : 0;
  } catch (const Error& e) {  // for a direct caller, and for the reducer, which rethrows it
    lpca::set_last_error(e.what(), e.index, e.gap);
    lpca::set_callback_error(e);
    return -static_cast<int32_t>(e.code);
  } catch (const std::exception& e) {
    lpca::set_last_error(e.what(), -1, 0.0);
    lpca::set_callback_error(Error(lpca::kInternal, e.what()));
    return -static_cast<int32_t>(lpca::kInternal);
  }
}

void lpca_file_stream_close(lpca_file_stream* s) { delete s; }

lpca_status lpca_map_file_write(const char* path, const lpca_map_info* info, const double* v_host,
                                const double* sigma_host) {
  return guarded([&] {
    need(path && info && (v_host || info->n * info->k == 0));
    emit_map(path, *info, v_host, sigma_host);
  });
}

lpca_status lpca_map_file_read(const char* path, lpca_map_info* info, double* v_host, int64_t v_capacity,
                               double* sigma_host) {
  return guarded([&] {
    need(path && info);
    const MapFile m = parse_map(path);
    *info = m.info;
    if (!v_host) return;
    if (v_capacity < static_cast<int64_t>(m.v.size()))
      throw Error(lpca::kInvalidArgument, "map file: V needs " + std::to_string(m.v.size()) + " doubles");
    std::copy(m.v.begin(), m.v.end(), v_host);
    if (sigma_host && m.info.has_singular_values) std::copy(m.sigma.begin(), m.sigma.end(), sigma_host);
  });
}

lpca_status lpca_map_save(const lpca_map* map, const char* path) {
  lpca_map_info info{};
  lpca_status st = lpca_map_info_get(map, &info);
  if (st != LPCA_OK) return st;
  std::vector<double> v(static_cast<std::size_t>(info.n * info.k)), sigma(static_cast<std::size_t>(info.k));
  if (!v.empty() && (st = lpca_map_copy_v(map, v.data(), LPCA_HOST)) != LPCA_OK) return st;
  if (info.has_singular_values && (st = lpca_map_copy_sigma(map, sigma.data())) != LPCA_OK) return st;
  return lpca_map_file_write(path, &info, v.data(), info.has_singular_values ? sigma.data() : nullptr);
}

lpca_status lpca_map_load(lpca_ctx* ctx, const char* path, lpca_map** out) {
  lpca_map_info info{};
  std::vector<double> v, sigma;
  const lpca_status st = guarded([&] {
    need(path != nullptr);
    MapFile m = parse_map(path);
    info = m.info;
    v = std::move(m.v);
    sigma = std::move(m.sigma);
  });
  if (st != LPCA_OK) return st;
  return lpca_map_create(ctx, &info, v.data(), info.has_singular_values ? sigma.data() : nullptr, out);
}

}  // extern "C"
