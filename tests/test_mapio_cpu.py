"""CPU: map files (save_map / load_map, proj/core/src/reducer.cpp:355-412) are
byte-identical to the compiled reference's and cross-readable both ways; the
reader's error classes and line numbers follow read_dense_matrix_market
(proj/core/src/matrix_io.cpp:40-81, 194-225)."""
import numpy as np
import pytest

import paper_1709_07175_b200 as lp
from oracle import refbind


@pytest.fixture(scope="module")
def ref():
    if not refbind.available():
        pytest.skip("compiled reference unavailable")
    return refbind


def _values(n, k, seed):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((n, k)) * 10.0 ** rng.integers(-8, 8, (n, k))
    v.flat[:6] = [0.1, 1.0, -2.5, 1e-300, 123456789012345678.0, 0.0]
    return v


@pytest.mark.parametrize("with_sigma", [True, False])
def test_map_file_bytes_match_reference(tmp_path, ref, with_sigma):
    n, k, l = 37, 5, 9
    v = _values(n, k, 1)
    sig = np.array([3.25, 1.0000000000000002, 0.1, 7e-5, 1e-17]) if with_sigma else None
    ours, theirs = tmp_path / "ours.map", tmp_path / "ref.map"
    lp.write_map_file(str(ours), lp.ReducerMethod.lazy_spca, v, sig, l=l, seed=2 ** 63 + 5, density=0.046051701859880914,
                      scale=np.sqrt(9.0))
    ref.save_map_file(str(theirs), 2, k, l, n, 2 ** 63 + 5, 0.046051701859880914, np.sqrt(9.0), v, sig)
    assert ours.read_bytes() == theirs.read_bytes()
    # cross-reading both ways
    back = lp.read_map_file(str(theirs))
    assert np.array_equal(back["v"], v) and back["seed"] == 2 ** 63 + 5 and back["l"] == l
    assert (back["singular_values"] is None) == (sig is None)
    r = ref.load_map_file(str(ours))
    assert np.array_equal(r["v"], v) and r["k"] == k and r["scale"] == np.sqrt(9.0)


@pytest.mark.parametrize("method,code", [(lp.ReducerMethod.rp, 0), (lp.ReducerMethod.spca, 1)])
def test_method_names_round_trip(tmp_path, ref, method, code):
    v = _values(4, 2, 3)
    p, q = tmp_path / "a.map", tmp_path / "b.map"
    lp.write_map_file(str(p), method, v)
    ref.save_map_file(str(q), code, 2, 2, 4, 0, 1.0, 1.0, v, None)
    assert p.read_bytes() == q.read_bytes()
    assert lp.read_map_file(str(p))["method"] == method


def test_map_file_errors(tmp_path):
    bad = tmp_path / "bad.map"
    bad.write_text("")
    with pytest.raises(lp.ParseError, match="empty") as e:
        lp.read_map_file(str(bad))
    assert e.value.line() == 1
    bad.write_text("{not json\n")
    with pytest.raises(lp.ParseError, match="map header") as e:
        lp.read_map_file(str(bad))
    assert e.value.line() == 1
    hdr = '{"method":"lazy_spca","k":2,"l":3,"seed":1,"density":1.0,"c":1.0,"n":2}\n'
    bad.write_text(hdr + "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n")
    with pytest.raises(lp.ParseError, match="array") as e:
        lp.read_map_file(str(bad))
    assert e.value.line() == 2
    bad.write_text(hdr + "%%MatrixMarket matrix array real general\n% c\n2 2\n1\n2\nx\n")
    with pytest.raises(lp.ParseError, match="numeric") as e:
        lp.read_map_file(str(bad))
    assert e.value.line() == 6
    bad.write_text(hdr + "%%MatrixMarket matrix array real general\n3 2\n" + "1\n" * 6)
    with pytest.raises(lp.DimensionError, match="header says 2x2"):
        lp.read_map_file(str(bad))
    bad.write_text('{"method":"lazy_spca","k":2,"l":3,"seed":1,"density":1.0,"c":1.0,"n":2,'
                   '"singular_values":[1.0]}\n%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n')
    with pytest.raises(lp.DimensionError, match="singular_values"):
        lp.read_map_file(str(bad))
    with pytest.raises(lp.ParseError, match="cannot open"):
        lp.read_map_file(str(tmp_path / "missing.map"))


@pytest.mark.parametrize("body,exc", [
    ("", lp.ParseError),
    ("{not json\n", lp.ParseError),
    ('{"method":"lazy_spca","k":2,"l":3,"seed":1,"density":1.0,"c":1.0,"n":2}\n'
     "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n", lp.ParseError),
    ('{"method":"lazy_spca","k":2,"l":3,"seed":1,"density":1.0,"c":1.0,"n":2}\n'
     "%%MatrixMarket matrix array real general\n% c\n2 2\n1\n2\nx\n", lp.ParseError),
    ('{"method":"lazy_spca","k":2,"l":3,"seed":1,"density":1.0,"c":1.0,"n":2}\n'
     "%%MatrixMarket matrix array real general\n3 2\n" + "1\n" * 6, lp.DimensionError),
    ('{"method":"lazy_spca","k":2,"seed":1,"density":1.0,"c":1.0,"n":2}\n'
     "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", lp.ParseError),
])
def test_map_file_errors_match_reference(tmp_path, ref, body, exc):
    """Same error class and line number as the reference's load_map_file."""
    p = tmp_path / "x.map"
    p.write_text(body)
    with pytest.raises(exc) as ours:
        lp.read_map_file(str(p))
    with pytest.raises(ref.RefError) as theirs:
        ref.load_map_file(str(p))
    codes = {lp.ParseError: 5, lp.DimensionError: 1}
    assert theirs.value.code == codes[exc]
    if exc is lp.ParseError:
        assert ours.value.line() == theirs.value.index
