// The reference-shaped C++ shim end to end: a reference caller's code (dense
// CSC X, reduce_lazy_spca / reduce_spca_streaming over SliceRowBlockStream,
// apply_map, matrix files and a file row-block stream) relinked against
// liblazypca_b200. Exit 0 = streaming agrees with in-core to 1e-10, the file
// stream with the in-memory slices bitwise, and the transform has the right shape.
#include <cmath>
#include <cstdio>
#include <random>

#include "lazypca_b200.hpp"

int main() {
  const lazypca::index_t m = 1500, n = 80;
  std::mt19937_64 g(3);
  std::normal_distribution<double> nd;
  std::vector<lazypca::index_t> cp{0}, ri;
  std::vector<double> va;
  std::vector<double> a(m * 8), b(8 * n);
  for (auto& v : a) v = nd(g);
  for (auto& v : b) v = nd(g);
  for (lazypca::index_t j = 0; j < n; ++j) {
    for (lazypca::index_t i = 0; i < m; ++i) {
      double s = 0.01 * nd(g);
      for (int t = 0; t < 8; ++t) s += a[i * 8 + t] * std::pow(0.8, t) * b[t * n + j];
      ri.push_back(i);
      va.push_back(s);
    }
    cp.push_back(static_cast<lazypca::index_t>(ri.size()));
  }
  const auto x = lazypca::SparseMatrix::from_csc(m, n, cp, ri, va);
  lazypca::ReducerConfig c;
  c.k = 4;
  c.l = 8;
  c.projection.seed = 5;
  int bad = 0;
  for (auto method : {lazypca::ReducerMethod::lazy_spca, lazypca::ReducerMethod::spca}) {
    c.method = method;
    const auto in_core = lazypca::reduce(x, c);
    lazypca::SliceRowBlockStream blocks(x, 400);
    const auto st = method == lazypca::ReducerMethod::spca ? lazypca::reduce_spca_streaming(blocks, c)
                                                           : lazypca::reduce_lazy_spca_streaming(blocks, c);
    for (int r = 0; r < 4; ++r) {
      const double e = std::abs(st.singular_values[r] - in_core.singular_values[r]) / in_core.singular_values[r];
      if (!(e < 1e-10)) {
        std::printf("method %d sigma %d rel err %g\n", static_cast<int>(method), r, e);
        bad = 1;
      }
    }
    const auto y = lazypca::apply_map(st, x);
    if (y.rows() != m || y.cols() != 4) bad = 1;
    lazypca::save_map_file(st, "/tmp/lpca_shim_test.map");  // map file round trip
    const auto back = lazypca::load_map_file("/tmp/lpca_shim_test.map");
    if (back.v.data()[5] != st.v.data()[5] || back.singular_values != st.singular_values || back.method != st.method)
      bad = 1;
  }
  // matrix_io: the same X through a MatrixMarket file and the file stream
  lazypca::write_sparse_matrix_market_file(x, "/tmp/lpca_shim_test.mtx");
  const auto xr = lazypca::read_sparse_matrix_market_file("/tmp/lpca_shim_test.mtx");
  if (xr.values() != x.values() || xr.row_idx() != x.row_idx()) bad = 1;
  {
    c.method = lazypca::ReducerMethod::lazy_spca;
    lazypca::SliceRowBlockStream slices(x, 400);
    lazypca::MatrixMarketRowBlockStream file("/tmp/lpca_shim_test.mtx", 400);
    const auto a = lazypca::reduce_lazy_spca_streaming(slices, c);
    const auto b = lazypca::reduce_lazy_spca_streaming(file, c);
    if (a.singular_values != b.singular_values || a.v.data()[7] != b.v.data()[7]) {
      std::printf("file stream differs from slices\n");
      bad = 1;
    }
  }
  try {
    lazypca::SliceRowBlockStream empty(lazypca::SparseMatrix::from_csc(0, n, std::vector<lazypca::index_t>(n + 1, 0), {}, {}), 10);
    lazypca::reduce_lazy_spca_streaming(empty, c);
    bad = 1;
  } catch (const lazypca::InvalidArgumentError&) {
  }
  return bad;
}
