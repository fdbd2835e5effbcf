"""GPU: streaming fits fed straight from files (lpca_file_stream_next driven
by lpca_fit_stream, no Python in the block loop) equal the same fits over
in-memory row slices; a parse error mid-stream aborts the fit with the
reference's ParseError and line."""
import numpy as np
import pytest

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

pytestmark = pytest.mark.gpu


def _cfg(k=6, l=12):
    return lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=k, l=l, projection=lp.ProjectionSpec(seed=5))


def test_matrix_market_stream_equals_slices(ctx, tmp_path):
    x = O.synth_lowrank(0, 2000, 150, 15, 0.9, 0.05, 3)
    x = x * (np.abs(x) > 0.8)
    s = lp.SparseMatrix.from_dense(x)
    p = tmp_path / "x.mtx"
    lp.write_sparse_matrix_market(s, str(p))
    for br in (300, 2000):
        a = lp.reduce_lazy_spca_streaming(lp.MatrixMarketRowBlockStream(str(p), br), _cfg(), ctx=ctx)
        b = lp.reduce_lazy_spca_streaming(lp.SliceRowBlockStream(s, br), _cfg(), ctx=ctx)
        assert np.array_equal(a.v, b.v) and np.array_equal(a.singular_values, b.singular_values)


def test_csv_stream_equals_dense_slices(ctx, tmp_path):
    x = O.synth_lowrank(0, 1500, 120, 12, 0.9, 0.05, 4)
    p = tmp_path / "x.csv"
    lp.write_dense_csv(x, str(p))
    a = lp.reduce_spca_streaming(lp.CsvRowBlockStream(str(p), 400), _cfg(), ctx=ctx)
    b = lp.reduce_spca_streaming(lp.SliceRowBlockStream(x, 400), _cfg(), ctx=ctx)
    assert np.max(np.abs(a.singular_values - b.singular_values) / b.singular_values) < 1e-12
    assert np.max(O.principal_angles(a.v, b.v)) < 1e-9


def test_parse_error_mid_stream_aborts_the_fit(ctx, tmp_path):
    x = O.synth_lowrank(0, 300, 40, 5, 0.9, 0.05, 5)
    p = tmp_path / "bad.csv"
    lp.write_dense_csv(x, str(p))
    lines = p.read_text().splitlines()
    lines[250] = lines[250] + ",1"  # a long row in the third block
    p.write_text("\n".join(lines) + "\n")
    with pytest.raises(lp.ParseError) as e:
        lp.reduce_lazy_spca_streaming(lp.CsvRowBlockStream(str(p), 100), _cfg(), ctx=ctx)
    assert e.value.line() == 251
    assert "row has 41 values, expected 40" in str(e.value)
