// Matrix files, the reference's formats and rules (proj/core/src/matrix_io.cpp,
// matrix_io.hpp:1-80): MatrixMarket coordinate (sparse) and array (dense)
// files, CSV, byte-identical writers (shortest round-trip values), readers
// with the reference's ParseError messages and line numbers, and row-block
// streams that feed lpca_fit_stream straight from a file.
//
// Host-only translation unit (g++). Restated from the reference's behaviour:
//  * banner `%%MatrixMarket matrix {coordinate|array} {real|integer|double} general`
//    (case-insensitive), `%` comment lines and blank lines skipped before the size
//    line; entries parsed with strtod (the same accepted spellings), non-finite
//    values rejected;
//  * coordinate entries 1-based, checked against the size line, duplicates summed
//    and explicit zeros dropped into the canonical CSC (SparseMatrix::from_triplets);
//  * CSV: one row per non-blank line, ',' between values, equal row lengths.
// The stream design is the reference's (one block resident; MatrixMarket blocks
// rescan the file, CSV blocks read on), but a CSV block is handed over dense
// row-major fp64 instead of being sparsified: the device path takes it as is.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/lazypca_b200.h"
#include "common.cuh"

using lpca::Error;
using lpca::index_t;

struct lpca_matrix_file {
  bool sparse = false;
  index_t rows = 0, cols = 0;
  std::vector<std::int64_t> col_ptr, row_idx;  // sparse (CSC)
  std::vector<double> values;                  // sparse values, or dense column-major
};

namespace {

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

Error parse_error(const std::string& what, std::int64_t line = -1) { return Error(lpca::kParse, what, line); }

std::string lower(std::string s) {
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

bool blank(const std::string& s) {
  for (unsigned char c : s)
    if (!std::isspace(c)) return false;
  return true;
}

std::string shortest(double v) {
  char buf[32];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) return buf;
  }
  return buf;
}

std::ifstream open_in(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw parse_error("cannot open '" + path + "' for reading");
  return in;
}

std::ofstream open_out(const std::string& path) {
  std::ofstream out(path);
  if (!out) throw parse_error("cannot open '" + path + "' for writing");
  return out;
}

// Banner, comments, blank lines; returns whether the file is coordinate and the
// size line, with line_no at the size line.
bool mm_preamble(std::istream& in, std::int64_t& line_no, std::string& size_line) {
  std::string line;
  if (!std::getline(in, line)) throw parse_error("empty MatrixMarket file", 1);
  ++line_no;
  std::istringstream ls(line);
  std::string banner, object, format, field, symmetry;
  ls >> banner >> object >> format >> field >> symmetry;
  if (lower(banner) != "%%matrixmarket") throw parse_error("missing %%MatrixMarket banner", line_no);
  if (lower(object) != "matrix") throw parse_error("unsupported MatrixMarket object '" + object + "'", line_no);
  const std::string fmt = lower(format);
  const bool coordinate = fmt == "coordinate";
  if (!coordinate && fmt != "array") throw parse_error("unsupported MatrixMarket format '" + format + "'", line_no);
  const std::string fld = lower(field);
  if (fld != "real" && fld != "integer" && fld != "double")
    throw parse_error("unsupported MatrixMarket field '" + field + "'", line_no);
  if (lower(symmetry) != "general") throw parse_error("unsupported MatrixMarket symmetry '" + symmetry + "'", line_no);
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line[0] == '%') continue;
    if (blank(line)) continue;
    size_line = line;
    return coordinate;
  }
  throw parse_error("MatrixMarket file ends before the size line", line_no);
}

void size_ints(const std::string& line, std::int64_t line_no, std::int64_t* out, int count) {
  std::istringstream ls(line);
  for (int i = 0; i < count; ++i)
    if (!(ls >> out[i])) throw parse_error("expected " + std::to_string(count) + " integers", line_no);
  std::string rest;
  if (ls >> rest) throw parse_error("trailing tokens after size line", line_no);
}

double number(const char* s, char** end, std::int64_t line_no) {
  errno = 0;
  const double v = std::strtod(s, end);
  if (*end == s) throw parse_error("expected a numeric value", line_no);
  if (!std::isfinite(v)) throw parse_error("non-finite value", line_no);
  return v;
}

struct Entry {
  index_t row, col;
  double value;
};

// One coordinate line (false: blank). Same checks and messages as the reference.
bool coord_line(const std::string& line, std::int64_t line_no, index_t rows, index_t cols, Entry& e) {
  if (line.empty() || blank(line)) return false;
  char* pos = nullptr;
  errno = 0;
  const long long i = std::strtoll(line.c_str(), &pos, 10);
  if (pos == line.c_str()) throw parse_error("expected row index", line_no);
  const char* after = pos;
  const long long j = std::strtoll(after, &pos, 10);
  if (pos == after) throw parse_error("expected column index", line_no);
  e.value = number(pos, &pos, line_no);
  for (; *pos != '\0'; ++pos)
    if (!std::isspace(static_cast<unsigned char>(*pos))) throw parse_error("trailing tokens after entry", line_no);
  if (i < 1 || i > rows)
    throw parse_error("row index " + std::to_string(i) + " outside 1.." + std::to_string(rows), line_no);
  if (j < 1 || j > cols)
    throw parse_error("column index " + std::to_string(j) + " outside 1.." + std::to_string(cols), line_no);
  e.row = static_cast<index_t>(i - 1);
  e.col = static_cast<index_t>(j - 1);
  return true;
}

// Canonical CSC from triplets: column-major order, rows ascending, duplicates
// summed, zero sums dropped (SparseMatrix::from_triplets, sparse_matrix.cpp:11-48;
// the same std::sort on the same sequence, so duplicates sum in the same order).
void to_csc(index_t rows, index_t cols, std::vector<Entry>& es, lpca_matrix_file& f) {
  std::sort(es.begin(), es.end(),
                   [](const Entry& a, const Entry& b) { return a.col != b.col ? a.col < b.col : a.row < b.row; });
  f.sparse = true;
  f.rows = rows;
  f.cols = cols;
  f.col_ptr.assign(static_cast<std::size_t>(cols) + 1, 0);
  f.row_idx.clear();
  f.values.clear();
  for (std::size_t p = 0; p < es.size();) {
    std::size_t q = p + 1;
    double v = es[p].value;
    for (; q < es.size() && es[q].row == es[p].row && es[q].col == es[p].col; ++q) v += es[q].value;
    if (v != 0.0) {
      f.row_idx.push_back(es[p].row);
      f.values.push_back(v);
      ++f.col_ptr[static_cast<std::size_t>(es[p].col) + 1];
    }
    p = q;
  }
  for (index_t j = 0; j < cols; ++j) f.col_ptr[static_cast<std::size_t>(j) + 1] += f.col_ptr[static_cast<std::size_t>(j)];
}

// Values of one CSV line into row.
void csv_line(const std::string& line, std::int64_t line_no, std::vector<double>& row) {
  const char* s = line.c_str();
  char* end = nullptr;
  while (true) {
    row.push_back(number(s, &end, line_no));
    s = end;
    while (std::isspace(static_cast<unsigned char>(*s))) ++s;
    if (*s == '\0') break;
    if (*s != ',') throw parse_error("expected ',' between values", line_no);
    ++s;
  }
}

std::unique_ptr<lpca_matrix_file> read_sparse_mm(const std::string& path) {
  auto in = open_in(path);
  std::int64_t line_no = 0;
  std::string size_line;
  if (!mm_preamble(in, line_no, size_line))
    throw parse_error("expected a coordinate (sparse) MatrixMarket file", line_no);
  std::int64_t d[3];
  size_ints(size_line, line_no, d, 3);
  if (d[0] < 0 || d[1] < 0 || d[2] < 0) throw parse_error("negative size entry", line_no);
  std::vector<Entry> es;
  es.reserve(static_cast<std::size_t>(d[2]));
  std::string line;
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line[0] == '%') continue;
    Entry e;
    if (coord_line(line, line_no, d[0], d[1], e)) es.push_back(e);
  }
  if (static_cast<std::int64_t>(es.size()) != d[2])
    throw parse_error("entry count " + std::to_string(es.size()) + " does not match header nnz " + std::to_string(d[2]),
                      line_no);
  auto f = std::make_unique<lpca_matrix_file>();
  to_csc(d[0], d[1], es, *f);
  return f;
}

std::unique_ptr<lpca_matrix_file> read_dense_mm(const std::string& path) {
  auto in = open_in(path);
  std::int64_t line_no = 0;
  std::string size_line;
  if (mm_preamble(in, line_no, size_line)) throw parse_error("expected an array (dense) MatrixMarket file", line_no);
  std::int64_t d[2];
  size_ints(size_line, line_no, d, 2);
  if (d[0] < 0 || d[1] < 0) throw parse_error("negative size entry", line_no);
  auto f = std::make_unique<lpca_matrix_file>();
  f->rows = d[0];
  f->cols = d[1];
  f->values.reserve(static_cast<std::size_t>(d[0] * d[1]));
  std::string line;
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line[0] == '%') continue;
    if (blank(line)) continue;
    const char* s = line.c_str();
    char* end = nullptr;
    while (*s != '\0') {
      while (std::isspace(static_cast<unsigned char>(*s))) ++s;
      if (*s == '\0') break;
      f->values.push_back(number(s, &end, line_no));
      s = end;
    }
  }
  if (f->values.size() != static_cast<std::size_t>(d[0] * d[1]))
    throw parse_error("array payload has " + std::to_string(f->values.size()) + " values, expected " +
                          std::to_string(d[0] * d[1]),
                      line_no);
  return f;
}

std::unique_ptr<lpca_matrix_file> read_csv(const std::string& path) {
  auto in = open_in(path);
  std::vector<std::vector<double>> rows;
  std::string line;
  std::int64_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (blank(line)) continue;
    std::vector<double> row;
    csv_line(line, line_no, row);
    if (!rows.empty() && row.size() != rows.front().size())
      throw parse_error("row has " + std::to_string(row.size()) + " values, expected " +
                            std::to_string(rows.front().size()),
                        line_no);
    rows.push_back(std::move(row));
  }
  auto f = std::make_unique<lpca_matrix_file>();
  f->rows = static_cast<index_t>(rows.size());
  f->cols = rows.empty() ? 0 : static_cast<index_t>(rows.front().size());
  f->values.resize(static_cast<std::size_t>(f->rows * f->cols));
  for (index_t i = 0; i < f->rows; ++i)
    for (index_t j = 0; j < f->cols; ++j)
      f->values[static_cast<std::size_t>(j * f->rows + i)] = rows[static_cast<std::size_t>(i)][static_cast<std::size_t>(j)];
  return f;
}

}  // namespace

// ---- row-block streams (MatrixMarketRowBlockStream / CsvRowBlockStream) -------
struct lpca_file_stream {
  bool csv = false;
  std::string path;
  index_t block_rows = 0, rows = 0, cols = 0, slices = 0, next_slice = 0;
  std::vector<std::int64_t> block_nnz;  // MatrixMarket: entries per block (counting pass)
  // CSV
  std::ifstream in;
  std::int64_t line_no = 0;
  std::vector<double> pending;
  bool pending_valid = false, done = false;
  // the current block (valid until the next call)
  lpca_matrix_file block;
  std::vector<double> dense;  // CSV block, row-major
};

namespace {

void open_mm_stream(lpca_file_stream& s) {
  auto in = open_in(s.path);
  std::int64_t line_no = 0;
  std::string size_line;
  if (!mm_preamble(in, line_no, size_line))
    throw parse_error("expected a coordinate (sparse) MatrixMarket file", line_no);
  std::int64_t d[3];
  size_ints(size_line, line_no, d, 3);
  s.rows = d[0];
  s.cols = d[1];
  s.slices = s.rows == 0 ? 0 : (s.rows + s.block_rows - 1) / s.block_rows;
  s.block_nnz.assign(static_cast<std::size_t>(s.slices == 0 ? 1 : s.slices), 0);
  std::string line;
  std::int64_t seen = 0;
  while (std::getline(in, line)) {  // counting pass: validates every entry once
    ++line_no;
    if (!line.empty() && line[0] == '%') continue;
    Entry e;
    if (!coord_line(line, line_no, s.rows, s.cols, e)) continue;
    ++s.block_nnz[static_cast<std::size_t>(e.row / s.block_rows)];
    ++seen;
  }
  if (seen != d[2])
    throw parse_error("entry count " + std::to_string(seen) + " does not match header nnz " + std::to_string(d[2]),
                      line_no);
}

bool next_mm_block(lpca_file_stream& s, lpca_matrix_view* v, int64_t* slice) {
  if (s.next_slice >= s.slices) return false;
  const index_t sl = s.next_slice++;
  const index_t lo = sl * s.block_rows, hi = std::min(lo + s.block_rows, s.rows);
  auto in = open_in(s.path);
  std::int64_t line_no = 0;
  std::string size_line;
  mm_preamble(in, line_no, size_line);
  std::vector<Entry> es;
  es.reserve(static_cast<std::size_t>(s.block_nnz[static_cast<std::size_t>(sl)]));
  std::string line;
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line[0] == '%') continue;
    Entry e;
    if (!coord_line(line, line_no, s.rows, s.cols, e)) continue;
    if (e.row >= lo && e.row < hi) es.push_back({e.row - lo, e.col, e.value});
  }
  to_csc(hi - lo, s.cols, es, s.block);
  *v = lpca_matrix_view{LPCA_F64, LPCA_CSC, LPCA_HOST, 0, hi - lo, s.cols, 0, s.block.values.data(),
                        s.block.col_ptr.data(), s.block.row_idx.data(), static_cast<int64_t>(s.block.values.size())};
  *slice = sl;
  return true;
}

void open_csv_stream(lpca_file_stream& s) {
  s.in.open(s.path);
  if (!s.in) throw parse_error("cannot open '" + s.path + "' for reading");
  std::string line;
  while (std::getline(s.in, line)) {
    ++s.line_no;
    if (blank(line)) continue;
    csv_line(line, s.line_no, s.pending);
    s.pending_valid = true;
    s.cols = static_cast<index_t>(s.pending.size());
    return;
  }
  s.done = true;  // empty file: no blocks
}

bool next_csv_block(lpca_file_stream& s, lpca_matrix_view* v, int64_t* slice) {
  if (s.done) return false;
  s.dense.clear();
  index_t filled = 0;
  if (s.pending_valid) {
    s.dense.insert(s.dense.end(), s.pending.begin(), s.pending.end());
    s.pending_valid = false;
    ++filled;
  }
  std::string line;
  std::vector<double> row;
  while (filled < s.block_rows && std::getline(s.in, line)) {
    ++s.line_no;
    if (blank(line)) continue;
    row.clear();
    csv_line(line, s.line_no, row);
    if (static_cast<index_t>(row.size()) != s.cols)
      throw parse_error("row has " + std::to_string(row.size()) + " values, expected " + std::to_string(s.cols),
                        s.line_no);
    s.dense.insert(s.dense.end(), row.begin(), row.end());
    ++filled;
  }
  if (filled < s.block_rows) s.done = true;
  if (filled == 0) return false;
  *v = lpca_matrix_view{LPCA_F64, LPCA_ROW_MAJOR, LPCA_HOST, 0, filled, s.cols, s.cols, s.dense.data(),
                        nullptr, nullptr, 0};
  *slice = s.next_slice++;
  return true;
}

}  // namespace

extern "C" {

lpca_status lpca_read_sparse_matrix_market(const char* path, lpca_matrix_file** out) {
  return guarded([&] {
    if (!path || !out) throw Error(lpca::kInvalidArgument, "null argument");
    *out = read_sparse_mm(path).release();
  });
}

lpca_status lpca_read_dense_matrix_market(const char* path, lpca_matrix_file** out) {
  return guarded([&] {
    if (!path || !out) throw Error(lpca::kInvalidArgument, "null argument");
    *out = read_dense_mm(path).release();
  });
}

lpca_status lpca_read_dense_csv(const char* path, lpca_matrix_file** out) {
  return guarded([&] {
    if (!path || !out) throw Error(lpca::kInvalidArgument, "null argument");
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
    if (f->sparse) {
      if (col_ptr) std::copy(f->col_ptr.begin(), f->col_ptr.end(), col_ptr);
      if (row_idx) std::copy(f->row_idx.begin(), f->row_idx.end(), row_idx);
    }
    if (values) std::copy(f->values.begin(), f->values.end(), values);
  });
}

lpca_status lpca_matrix_file_view(const lpca_matrix_file* f, lpca_matrix_view* out) {
  return guarded([&] {
    if (!f || !out) throw Error(lpca::kInvalidArgument, "null argument");
    if (f->sparse)
      *out = lpca_matrix_view{LPCA_F64, LPCA_CSC, LPCA_HOST, 0, f->rows, f->cols, 0, f->values.data(),
                              f->col_ptr.data(), f->row_idx.data(), static_cast<int64_t>(f->values.size())};
    else
      *out = lpca_matrix_view{LPCA_F64, LPCA_COL_MAJOR, LPCA_HOST, 0, f->rows, f->cols, f->rows, f->values.data(),
                              nullptr, nullptr, 0};
  });
}

void lpca_matrix_file_free(lpca_matrix_file* f) { delete f; }

lpca_status lpca_write_sparse_matrix_market(const char* path, int64_t rows, int64_t cols, const int64_t* col_ptr,
                                            const int64_t* row_idx, const double* values) {
  return guarded([&] {
    if (!path || (cols > 0 && !col_ptr)) throw Error(lpca::kInvalidArgument, "null argument");
    auto out = open_out(path);
    const int64_t nnz = cols > 0 ? col_ptr[cols] : 0;
    out << "%%MatrixMarket matrix coordinate real general\n" << rows << ' ' << cols << ' ' << nnz << '\n';
    for (int64_t j = 0; j < cols; ++j)
      for (int64_t p = col_ptr[j]; p < col_ptr[j + 1]; ++p)
        out << row_idx[p] + 1 << ' ' << j + 1 << ' ' << shortest(values[p]) << '\n';
  });
}

lpca_status lpca_write_dense_matrix_market(const char* path, int64_t rows, int64_t cols, const double* colmajor) {
  return guarded([&] {
    if (!path || (rows * cols > 0 && !colmajor)) throw Error(lpca::kInvalidArgument, "null argument");
    auto out = open_out(path);
    out << "%%MatrixMarket matrix array real general\n" << rows << ' ' << cols << '\n';
    for (int64_t j = 0; j < cols; ++j)
      for (int64_t i = 0; i < rows; ++i) out << shortest(colmajor[j * rows + i]) << '\n';
  });
}

lpca_status lpca_write_dense_csv(const char* path, int64_t rows, int64_t cols, const double* colmajor) {
  return guarded([&] {
    if (!path || (rows * cols > 0 && !colmajor)) throw Error(lpca::kInvalidArgument, "null argument");
    auto out = open_out(path);
    for (int64_t i = 0; i < rows; ++i) {
      for (int64_t j = 0; j < cols; ++j) {
        if (j) out << ',';
        out << shortest(colmajor[j * rows + i]);
      }
      out << '\n';
    }
  });
}

lpca_status lpca_open_matrix_market_stream(const char* path, int64_t block_rows, lpca_file_stream** out) {
  return guarded([&] {
    if (!path || !out) throw Error(lpca::kInvalidArgument, "null argument");
    if (block_rows < 1) throw Error(lpca::kInvalidArgument, "block_rows must be at least 1");
    auto s = std::make_unique<lpca_file_stream>();
    s->path = path;
    s->block_rows = block_rows;
    open_mm_stream(*s);
    *out = s.release();
  });
}

lpca_status lpca_open_csv_stream(const char* path, int64_t block_rows, lpca_file_stream** out) {
  return guarded([&] {
    if (!path || !out) throw Error(lpca::kInvalidArgument, "null argument");
    if (block_rows < 1) throw Error(lpca::kInvalidArgument, "block_rows must be at least 1");
    auto s = std::make_unique<lpca_file_stream>();
    s->csv = true;
    s->path = path;
    s->block_rows = block_rows;
    open_csv_stream(*s);
    *out = s.release();
  });
}

int32_t lpca_file_stream_next(void* user, lpca_matrix_view* block, int64_t* slice) {
  auto* s = static_cast<lpca_file_stream*>(user);
  try {
    if (!s || !block || !slice) throw Error(lpca::kInvalidArgument, "null argument");
    return (s->csv ? next_csv_block(*s, block, slice) : next_mm_block(*s, block, slice)) ? 1 : 0;
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

}  // extern "C"
