// Map files, byte-compatible with the reference: save_map / load_map
// (proj/core/src/reducer.cpp:355-412) write a one-line JSON header (ordered
// keys method, k, l, seed, density, c, n[, singular_values]) and then V as a
// dense MatrixMarket array, column-major, one shortest-round-trip value per line
// (write_dense_matrix_market / format_double, matrix_io.cpp:132-141, 232-237);
// reading follows read_dense_matrix_market (matrix_io.cpp:40-81, 194-225) with
// the same ParseError line numbers and DimensionError checks.
//
// Host-only translation unit (g++). The JSON header goes through nlohmann/json,
// the reference's own serialiser, so numbers print identically.
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

#include <nlohmann/json.hpp>

#include "../../include/lazypca_b200.h"
#include "common.cuh"

using lpca::Error;
using lpca::index_t;

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

const char* method_name(int32_t m) {
  switch (m) {
    case LPCA_RP: return "rp";
    case LPCA_SPCA: return "spca";
    case LPCA_LAZY_SPCA: return "lazy_spca";
  }
  throw Error(lpca::kInvalidArgument, "unknown reducer method " + std::to_string(m));
}

int32_t method_code(const std::string& s) {
  if (s == "rp") return LPCA_RP;
  if (s == "spca") return LPCA_SPCA;
  if (s == "lazy_spca") return LPCA_LAZY_SPCA;
  throw Error(lpca::kInvalidArgument, "unknown reducer method '" + s + "'");
}

// Shortest %.*g form that round-trips (format_double's rule).
std::string shortest(double v) {
  char buf[32];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) return buf;
  }
  return buf;
}

std::string lower(std::string s) {
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

bool blank(const std::string& s) {
  for (unsigned char c : s)
    if (!std::isspace(c)) return false;
  return true;
}

Error parse_error(const std::string& what, std::int64_t line) { return Error(lpca::kParse, what, line); }

void write_map(std::ostream& out, const lpca_map_info& info, const double* v, const double* sigma) {
  nlohmann::ordered_json header;
  header["method"] = method_name(info.method);
  header["k"] = info.k;
  header["l"] = info.l;
  header["seed"] = info.seed;
  header["density"] = info.density;
  header["c"] = info.scale;
  header["n"] = info.n;
  if (info.has_singular_values && sigma) header["singular_values"] = std::vector<double>(sigma, sigma + info.k);
  out << header.dump() << '\n';
  out << "%%MatrixMarket matrix array real general\n";
  out << info.n << ' ' << info.k << '\n';
  for (index_t j = 0; j < info.k; ++j)
    for (index_t i = 0; i < info.n; ++i) out << shortest(v[j * info.n + i]) << '\n';
}

struct Loaded {
  lpca_map_info info{};
  std::vector<double> v, sigma;
};

Loaded read_map(std::istream& in) {
  Loaded m;
  std::string line;
  if (!std::getline(in, line)) throw parse_error("map file is empty", 1);
  nlohmann::json header;
  try {
    header = nlohmann::json::parse(line);
  } catch (const nlohmann::json::exception& e) {
    throw parse_error(std::string("map header: ") + e.what(), 1);
  }
  try {
    m.info.method = method_code(header.at("method").get<std::string>());
    m.info.k = header.at("k").get<index_t>();
    m.info.l = header.at("l").get<index_t>();
    m.info.seed = header.at("seed").get<std::uint64_t>();
    m.info.density = header.at("density").get<double>();
    m.info.scale = header.at("c").get<double>();
    m.info.n = header.at("n").get<index_t>();
    if (header.contains("singular_values")) {
      m.sigma = header.at("singular_values").get<std::vector<double>>();
      m.info.has_singular_values = 1;
    }
  } catch (const nlohmann::json::exception& e) {
    throw parse_error(std::string("map header: ") + e.what(), 1);
  }
  // dense MatrixMarket array (line numbers count from the file start, as the
  // reference's reader does: it restarts at 0 after the header line)
  std::int64_t line_no = 0;
  if (!std::getline(in, line)) throw parse_error("empty MatrixMarket file", 1);
  ++line_no;
  bool coordinate = false;
  {
    std::istringstream ls(line);
    std::string banner, object, format, field, symmetry;
    ls >> banner >> object >> format >> field >> symmetry;
    if (lower(banner) != "%%matrixmarket") throw parse_error("missing %%MatrixMarket banner", line_no);
    if (lower(object) != "matrix") throw parse_error("unsupported MatrixMarket object '" + object + "'", line_no);
    const std::string fmt = lower(format);
    coordinate = fmt == "coordinate";
    if (!coordinate && fmt != "array") throw parse_error("unsupported MatrixMarket format '" + format + "'", line_no);
    const std::string fld = lower(field);
    if (fld != "real" && fld != "integer" && fld != "double")
      throw parse_error("unsupported MatrixMarket field '" + field + "'", line_no);
    if (lower(symmetry) != "general") throw parse_error("unsupported MatrixMarket symmetry '" + symmetry + "'", line_no);
  }
  std::string size_line;
  bool have_size = false;
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line[0] == '%') continue;
    if (blank(line)) continue;
    size_line = line;
    have_size = true;
    break;
  }
  if (!have_size) throw parse_error("MatrixMarket file ends before the size line", line_no);
  if (coordinate) throw parse_error("expected an array (dense) MatrixMarket file", line_no);
  std::int64_t dims[2];
  {
    std::istringstream ls(size_line);
    for (auto& d : dims)
      if (!(ls >> d)) throw parse_error("expected 2 integers", line_no);
    std::string rest;
    if (ls >> rest) throw parse_error("trailing tokens after size line", line_no);
  }
  if (dims[0] < 0 || dims[1] < 0) throw parse_error("negative size entry", line_no);
  std::vector<double> data;
  data.reserve(static_cast<std::size_t>(dims[0] * dims[1]));
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line[0] == '%') continue;
    if (blank(line)) continue;
    const char* s = line.c_str();
    char* end = nullptr;
    while (*s != '\0') {
      while (std::isspace(static_cast<unsigned char>(*s))) ++s;
      if (*s == '\0') break;
      errno = 0;
      const double v = std::strtod(s, &end);
      if (end == s) throw parse_error("expected a numeric value", line_no);
      if (!std::isfinite(v)) throw parse_error("non-finite value", line_no);
      data.push_back(v);
      s = end;
    }
  }
  if (data.size() != static_cast<std::size_t>(dims[0] * dims[1]))
    throw parse_error("array payload has " + std::to_string(data.size()) + " values, expected " +
                          std::to_string(dims[0] * dims[1]),
                      line_no);
  if (dims[0] != m.info.n || dims[1] != m.info.k)
    throw Error(lpca::kDimension, "map payload is " + std::to_string(dims[0]) + "x" + std::to_string(dims[1]) +
                                      " but the header says " + std::to_string(m.info.n) + "x" +
                                      std::to_string(m.info.k));
  if (m.info.has_singular_values && static_cast<index_t>(m.sigma.size()) != m.info.k)
    throw Error(lpca::kDimension, "map header: singular_values length does not match k");
  m.v = std::move(data);
  return m;
}

}  // namespace

extern "C" {

lpca_status lpca_map_file_write(const char* path, const lpca_map_info* info, const double* v_host,
                                const double* sigma_host) {
  return guarded([&] {
    if (!path || !info || (!v_host && info->n * info->k > 0)) throw Error(lpca::kInvalidArgument, "null argument");
    std::ofstream out(path);
    if (!out) throw parse_error(std::string("cannot open '") + path + "' for writing", 0);
    write_map(out, *info, v_host, sigma_host);
    if (!out) throw parse_error(std::string("write to '") + path + "' failed", 0);
  });
}

lpca_status lpca_map_file_read(const char* path, lpca_map_info* info, double* v_host, int64_t v_capacity,
                               double* sigma_host) {
  return guarded([&] {
    if (!path || !info) throw Error(lpca::kInvalidArgument, "null argument");
    std::ifstream in(path);
    if (!in) throw parse_error(std::string("cannot open '") + path + "' for reading", 0);
    const Loaded m = read_map(in);
    *info = m.info;
    if (v_host) {
      if (v_capacity < static_cast<int64_t>(m.v.size()))
        throw Error(lpca::kInvalidArgument, "map file: V needs " + std::to_string(m.v.size()) + " doubles");
      std::copy(m.v.begin(), m.v.end(), v_host);
      if (sigma_host && m.info.has_singular_values) std::copy(m.sigma.begin(), m.sigma.end(), sigma_host);
    }
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
  lpca_status st = lpca_map_file_read(path, &info, nullptr, 0, nullptr);
  if (st != LPCA_OK) return st;
  std::vector<double> v(static_cast<std::size_t>(info.n * info.k)), sigma(static_cast<std::size_t>(info.k));
  st = lpca_map_file_read(path, &info, v.data(), static_cast<int64_t>(v.size()), sigma.data());
  if (st != LPCA_OK) return st;
  return lpca_map_create(ctx, &info, v.data(), info.has_singular_values ? sigma.data() : nullptr, out);
}

}  // extern "C"
