"""GPU: the sparse-X path (CSR/CSC gathers, csrc/sparse.cu) against the compiled
reference on the same CSC inputs — the kernels (spmm, gemm_t,
proj/core/src/kernels.cpp:30-113) bitwise, the reducers and the transform in
exact-order mode to eigensolver roundoff (F and Y bitwise), streaming Lazy
SPCA over sparse blocks likewise."""
import numpy as np
import pytest

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

pytestmark = pytest.mark.gpu


def _sparse(m, n, density, seed, lowrank=True):
    rng = np.random.default_rng(seed)
    mask = rng.uniform(0, 1, (m, n)) < density
    base = O.synth_lowrank(0, m, n, 15, 0.9, 0.05, seed) if lowrank else rng.standard_normal((m, n))
    return base * mask


def _cfg(method, k, l, seed=13, block_rows=0):
    return lp.ReducerConfig(method=method, k=k, l=l, projection=lp.ProjectionSpec(seed=seed), block_rows=block_rows)


@pytest.mark.parametrize("w", [7, 37, 150, 600])
def test_sparse_kernels_bitwise(ctx, ref, w):
    d = _sparse(3000, 1200, 0.03, 1, lowrank=False)
    xs = lp.SparseMatrix.from_dense(d)
    rng = np.random.default_rng(2)
    wm = rng.uniform(-1, 1, (1200, w))
    wm[rng.uniform(0, 1, wm.shape) < 0.05] = 0.0  # exact zeros are skipped like the reference
    assert np.array_equal(lp.spmm(xs, wm, ctx), ref.spmm(d, wm))
    if w <= 512:
        u = rng.uniform(-1, 1, (3000, w))
        assert np.array_equal(lp.gemm_t(u, xs, ctx), ref.gemm_t(u, d))


@pytest.mark.parametrize("method,code", [(lp.ReducerMethod.lazy_spca, 2), (lp.ReducerMethod.spca, 1)])
def test_sparse_fit_and_transform_vs_reference(ctx, ref, method, code):
    d = _sparse(4000, 900, 0.0244, 3)  # the paper's density
    xs = lp.SparseMatrix.from_dense(d)
    k, l = 8, 20
    v_ref, s_ref, _, _ = ref.reduce(code, d, k, l, 13)
    ctx.set_exact_order(True)
    try:
        m = lp.reduce(xs, _cfg(method, k, l), ctx=ctx)
        y = lp.apply_map(m, xs, ctx=ctx)
    finally:
        ctx.set_exact_order(False)
    if method == lp.ReducerMethod.lazy_spca:  # F bitwise; the eigensolver differs only by roundoff
        assert np.max(np.abs(m.singular_values - s_ref) / s_ref) < 1e-13
        assert np.max(O.principal_angles(m.v, v_ref)) < 1e-10
    else:  # CholeskyQR2 vs Householder QR: equal up to roundoff
        assert np.max(np.abs(m.singular_values - s_ref) / s_ref) < 1e-10
        assert np.max(O.principal_angles(m.v, v_ref)) < 1e-8
    assert np.array_equal(y, ref.apply_map(d, m.v))


def test_sparse_streaming_lazy_is_bitwise_reference(ctx, ref):
    d = _sparse(3000, 700, 0.05, 4)
    k, l, br = 6, 14, 800
    v_ref, s_ref, _, _ = ref.reduce(2, d, k, l, 13, block_rows=br)
    ctx.set_exact_order(True)
    try:
        m = lp.reduce_lazy_spca_streaming(lp.SliceRowBlockStream(lp.SparseMatrix.from_dense(d), br),
                                          _cfg(lp.ReducerMethod.lazy_spca, k, l), ctx=ctx)
    finally:
        ctx.set_exact_order(False)
    assert np.max(np.abs(m.singular_values - s_ref) / s_ref) < 1e-13
    assert np.max(O.principal_angles(m.v, v_ref)) < 1e-10


def test_sparse_and_densified_paths_agree(ctx, monkeypatch):
    d = _sparse(5000, 800, 0.02, 5)
    xs = lp.SparseMatrix.from_dense(d)
    cfg = _cfg(lp.ReducerMethod.lazy_spca, 10, 16)
    a = lp.reduce(xs, cfg, ctx=ctx)
    monkeypatch.setenv("LPCA_SPARSE", "0")
    b = lp.reduce(xs, cfg, ctx=ctx)
    assert np.max(np.abs(a.singular_values - b.singular_values) / b.singular_values) < 1e-12
    assert np.max(O.principal_angles(a.v, b.v)) < 1e-9
