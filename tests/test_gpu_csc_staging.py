"""GPU: a host CSC view is checked and turned into the device CSR/CSC copies by
kernels (csrc/sparse.cu, stage_csc_device in csrc/lpca.cu). The errors must be
the reference's SparseMatrix::from_csc errors (sparse_matrix.cpp:50-80) — same
class, same message, same column — including which one wins when a view has
several: the first entry in column-major order, for that entry the first check
(range, strictly increasing, explicit zero, non-finite), and a decreasing
col_ptr only after every entry of the columns before it. The reference raises
them through oracle/ref_capi.cpp's ref_fit_transform_csc."""
import numpy as np
import pytest

import paper_1709_07175_b200 as lp

pytestmark = pytest.mark.gpu

M, N = 40, 30


def _valid():
    rng = np.random.default_rng(8)
    d = rng.uniform(0.5, 1.5, (M, N)) * (rng.random((M, N)) < 0.1)
    d[0, :] = 1.0  # every column non-empty
    s = lp.SparseMatrix.from_dense(d)
    return s.col_ptr.copy(), s.row_idx.copy(), s.values.copy()


def _entry(cp, j, t=1):
    """index of the t-th entry of column j"""
    assert cp[j + 1] - cp[j] > t
    return cp[j] + t


def _cases():
    out = {}
    cp, ri, va = _valid()
    r = ri.copy(); r[_entry(cp, 3)] = M + 2
    out["row out of range"] = (cp, r, va)
    r = ri.copy(); p = _entry(cp, 2); r[p] = r[p - 1]
    out["rows not increasing"] = (cp, r, va)
    v = va.copy(); v[_entry(cp, 4)] = 0.0
    out["explicit zero"] = (cp, ri, v)
    v = va.copy(); v[_entry(cp, 1)] = np.nan
    out["non-finite"] = (cp, ri, v)
    c = cp.copy(); c[5] = c[4] - 1  # column 4's range runs backwards
    out["col_ptr decreasing"] = (c, ri, va)
    c = cp.copy(); c[4] = c[5] + 1  # column 3's range runs into column 4's rows first
    out["col_ptr overlapping the next column"] = (c, ri, va)
    c = cp.copy(); c[4] = c[5] + 1
    v = va.copy(); v[_entry(cp, 1)] = 0.0  # an entry error in an earlier column wins
    out["entry error before a bad col_ptr"] = (c, ri, v)
    r = ri.copy(); r[_entry(cp, 1)] = -1
    v = va.copy(); v[_entry(cp, 2)] = 0.0
    out["first of two entry errors"] = (cp, r, v)
    r = ri.copy(); p = _entry(cp, 5); r[p] = r[p - 1]
    v = va.copy(); v[p] = 0.0  # one entry failing two checks: the increasing check first
    out["one entry, two checks"] = (cp, r, v)
    return out


CASES = _cases()


@pytest.mark.parametrize("host", ["0", "1"])  # device staging / the host fallback (too little memory)
@pytest.mark.parametrize("sparse", ["1", "0"])  # kept sparse (CSR built) / densified
@pytest.mark.parametrize("name", sorted(CASES))
def test_csc_errors_match_the_reference(ctx, ref, name, sparse, host, monkeypatch):
    monkeypatch.setenv("LPCA_SPARSE", sparse)
    monkeypatch.setenv("LPCA_CSC_HOST", host)
    cp, ri, va = CASES[name]
    with pytest.raises(Exception) as want:
        ref.fit_transform_csc(2, M, N, cp, ri, va, 4, 6, 3)
    x = lp.SparseMatrix(M, N, cp, ri, va)
    cfg = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=4, l=6, projection=lp.ProjectionSpec(seed=3))
    with pytest.raises(lp.Error) as got:
        lp.reduce(x, cfg, ctx=ctx)
    assert str(got.value) == str(want.value)
    assert type(got.value) is {1: lp.DimensionError, 2: lp.InvalidArgumentError}[want.value.code]


@pytest.mark.parametrize("host", ["0", "1"])
def test_valid_csc_fit_equals_the_reference(ctx, ref, host, monkeypatch):
    monkeypatch.setenv("LPCA_CSC_HOST", host)
    cp, ri, va = _valid()
    _, v_ref, s_ref, _ = ref.fit_transform_csc(2, M, N, cp, ri, va, 4, 6, 3, want_y=False)
    x = lp.SparseMatrix(M, N, cp, ri, va)
    cfg = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=4, l=6, projection=lp.ProjectionSpec(seed=3))
    got = lp.reduce(x, cfg, ctx=ctx)
    assert np.max(np.abs(got.singular_values - s_ref) / s_ref) < 1e-12


@pytest.mark.parametrize("host", ["0", "1"])
def test_col_ptr_past_nnz_is_refused_without_reading_past_the_arrays(ctx, host, monkeypatch):
    """A col_ptr entry beyond nnz (the last one still equal to nnz) makes a
    later column decrease; the entries are never read past the arrays (the
    reference reads out of bounds here, so only the library's behaviour is
    checked): the decreasing col_ptr is reported."""
    monkeypatch.setenv("LPCA_CSC_HOST", host)
    cp, ri, va = _valid()
    c = cp.copy()
    c[3] = cp[-1] + 10 ** 12
    x = lp.SparseMatrix(M, N, c, ri, va)
    cfg = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=4, l=6, projection=lp.ProjectionSpec(seed=3))
    with pytest.raises(lp.InvalidArgumentError, match="col_ptr must be non-decreasing"):
        lp.reduce(x, cfg, ctx=ctx)


@pytest.mark.parametrize("l", [20, 100, 150])
def test_very_sparse_omega_on_sparse_x_matches_the_reference(ctx, ref, l):
    """The sign-mask sketch (spmm_csr_pm1) sums each U[i][c] over the row's
    nonzeros in ascending j like the reference's spmm(CSC, CSC)
    (kernels.cpp:49-68): with the exact-order passes the map equals the
    reference's to eigensolver roundoff and Y bitwise."""
    rng = np.random.default_rng(31)
    m, n, k = 3000, 2000, l // 2
    d = rng.uniform(0.5, 1.5, (m, n)) * (rng.random((m, n)) < 0.0244)
    xs = lp.SparseMatrix.from_dense(d)
    dens = lp.density_for(lp.DensityPolicy.aggressive(), l)
    y_ref, v_ref, s_ref, _ = ref.fit_transform_csc(2, m, n, xs.col_ptr, xs.row_idx, xs.values, k, l, 5, kind=1,
                                                   density=dens)
    cfg = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=k, l=l,
                           projection=lp.ProjectionSpec(kind=lp.ProjectionKind.very_sparse, density=dens, seed=5))
    ctx.set_exact_order(True)
    try:
        mp = lp.reduce(xs, cfg, ctx=ctx)
        y = lp.apply_map(mp, xs, ctx=ctx)
    finally:
        ctx.set_exact_order(False)
    assert np.max(np.abs(mp.singular_values - s_ref) / s_ref) < 1e-13
    kk = k // 2
    from oracle import lazypca_oracle as O
    assert np.max(O.principal_angles(mp.v[:, :kk], v_ref[:, :kk])) < 1e-10
    assert np.array_equal(y, ref.apply_map(d, mp.v))
