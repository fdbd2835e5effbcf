"""CPU: matrix files (csrc/matrixio.cpp) against the compiled reference's
matrix_io (proj/core/src/matrix_io.cpp): byte-identical writers, equal readers
(CSC canonicalisation with summed duplicates and dropped zeros), the same
ParseError messages and line numbers on malformed files, and the same row
blocks from the MatrixMarket / CSV streams. No GPU: host code only."""
import numpy as np
import pytest

import paper_1709_07175_b200 as lp


def _sparse(seed, m=40, n=25, density=0.2):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n)) * (rng.uniform(0, 1, (m, n)) < density)
    a[rng.uniform(0, 1, a.shape) < 0.05] *= 1e-300  # tiny values round-trip too
    return a


def test_writers_are_byte_identical(tmp_path, ref):
    a = _sparse(1)
    s = lp.SparseMatrix.from_dense(a)
    for kind, ours, name in ((0, lambda p: lp.write_sparse_matrix_market(s, p), "s.mtx"),
                             (1, lambda p: lp.write_dense_matrix_market(a, p), "d.mtx"),
                             (2, lambda p: lp.write_dense_csv(a, p), "d.csv")):
        p1, p2 = tmp_path / ("ours_" + name), tmp_path / ("ref_" + name)
        ours(str(p1))
        if kind == 0:
            ref.write_matrix_file(0, str(p2), s.rows(), s.cols(), s.col_ptr, s.row_idx, s.values)
        else:
            ref.write_matrix_file(kind, str(p2), a.shape[0], a.shape[1], val=a)
        assert p1.read_bytes() == p2.read_bytes()


def test_readers_match_reference_including_duplicates(tmp_path, ref):
    p = tmp_path / "dup.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n% comment\n\n4 3 7\n"
                 "1 1 1.5\n3 2 -2\n1 1 0.25\n2 3 1e-3\n4 1 5\n3 2 2\n2 2 0\n")
    x = lp.read_sparse_matrix_market(str(p))
    r = ref.read_matrix_file(0, str(p))
    assert (x.rows(), x.cols()) == r[:2]
    assert np.array_equal(x.col_ptr, r[2]) and np.array_equal(x.row_idx, r[3]) and np.array_equal(x.values, r[4])
    a = _sparse(2)
    d, c = tmp_path / "a.mtx", tmp_path / "a.csv"
    lp.write_dense_matrix_market(a, str(d))
    lp.write_dense_csv(a, str(c))
    assert np.array_equal(lp.read_dense_matrix_market(str(d)), ref.read_matrix_file(1, str(d)))
    assert np.array_equal(lp.read_dense_csv(str(c)), ref.read_matrix_file(2, str(c)))
    assert np.array_equal(lp.read_dense_csv(str(c)), a)


BAD = [
    ("s", "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 1\n"),
    ("s", "%%MatrixMarket tensor coordinate real general\n2 2 1\n1 1 1\n"),
    ("s", "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1\n"),
    ("s", "not a banner\n2 2 1\n"),
    ("s", "%%MatrixMarket matrix coordinate real general\n% only comments\n"),
    ("s", "%%MatrixMarket matrix coordinate real general\n2 2\n"),
    ("s", "%%MatrixMarket matrix coordinate real general\n2 2 1 9\n1 1 1\n"),
    ("s", "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n3 1 1\n"),
    ("s", "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 0 1\n"),
    ("s", "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 nan\n"),
    ("s", "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1 extra\n"),
    ("s", "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n"),
    ("s", "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n"),
    ("d", "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n"),
    ("d", "%%MatrixMarket matrix array real general\n2 2\n1\n2\nx\n4\n"),
    ("d", "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n"),
    ("c", "1,2,3\n4,5\n"),
    ("c", "1,2\n3;4\n"),
    ("c", "1,inf\n"),
    ("c", "1,,2\n"),
]


@pytest.mark.parametrize("case", range(len(BAD)))
def test_parse_errors_match_reference(tmp_path, ref, case):
    kind, text = BAD[case]
    p = tmp_path / ("bad.csv" if kind == "c" else "bad.mtx")
    p.write_text(text)
    reader = {"s": lp.read_sparse_matrix_market, "d": lp.read_dense_matrix_market, "c": lp.read_dense_csv}[kind]
    with pytest.raises(lp.ParseError) as ours:
        reader(str(p))
    with pytest.raises(ref.RefError) as theirs:
        ref.read_matrix_file({"s": 0, "d": 1, "c": 2}[kind], str(p))
    assert str(ours.value) == str(theirs.value)
    assert ours.value.line() == theirs.value.index


@pytest.mark.parametrize("block_rows", [1, 7, 40, 100])
def test_streams_match_reference_blocks(tmp_path, ref, block_rows):
    a = _sparse(3)
    s = lp.SparseMatrix.from_dense(a)
    mm, csv = tmp_path / "x.mtx", tmp_path / "x.csv"
    lp.write_sparse_matrix_market(s, str(mm))
    lp.write_dense_csv(a, str(csv))
    want = ref.stream_blocks(0, str(mm), block_rows)
    got = []
    st = lp.MatrixMarketRowBlockStream(str(mm), block_rows)
    while (b := st.next()) is not None:
        got.append(b)
    assert len(got) == len(want)
    for i, (b, w) in enumerate(zip(got, want)):
        assert b.slice_index == i
        assert (b.block.rows(), b.block.cols()) == w[:2]
        assert np.array_equal(b.block.col_ptr, w[2]) and np.array_equal(b.block.values, w[4])
    # CSV blocks: dense here, the reference's sparsified CSC of the same rows
    want = ref.stream_blocks(1, str(csv), block_rows)
    st = lp.CsvRowBlockStream(str(csv), block_rows)
    got = []
    while (b := st.next()) is not None:
        got.append(b)
    assert len(got) == len(want)
    for b, w in zip(got, want):
        assert np.array_equal(lp.SparseMatrix.from_dense(b.block).values, w[4])


def test_stream_parse_error_surfaces(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("1,2\n3,4\n5\n")
    st = lp.CsvRowBlockStream(str(p), 1)
    st.next()
    st.next()
    with pytest.raises(lp.ParseError) as e:
        st.next()
    assert e.value.line() == 3
