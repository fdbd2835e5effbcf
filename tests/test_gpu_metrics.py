"""GPU: verification metrics at scale (proj/core/src/metrics.cpp) — chordal
distance against the compiled reference, distance_preservation against the
restated pair draw (metrics.cpp:320-335) and host distances, dense and sparse X."""
import numpy as np
import pytest

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

pytestmark = pytest.mark.gpu


def _orth(n, k, seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, k)))
    return q


def test_chordal_distance_matches_reference(ctx, ref):
    a = _orth(3000, 40, 1)
    b = _orth(3000, 40, 2)
    near = np.linalg.qr(a + 1e-9 * np.random.default_rng(3).standard_normal(a.shape))[0]
    for x, y in ((a, b), (a, near), (a, a)):
        ours, theirs = lp.chordal_distance(x, y, ctx=ctx), ref.chordal(x, y)
        assert abs(ours - theirs) <= 1e-12 * max(1.0, theirs) + 1e-15
    assert lp.chordal_distance(a, a, ctx=ctx) < 1e-13
    # different k, and the error classes
    assert lp.chordal_distance(a, b[:, :10], ctx=ctx) > 0
    with pytest.raises(lp.DimensionError):
        lp.chordal_distance(a, b[:100], ctx=ctx)
    with pytest.raises(lp.InvalidArgumentError, match="orthonormal"):
        lp.chordal_distance(a * 2.0, b, ctx=ctx)


@pytest.mark.parametrize("sparse", [False, True])
def test_distance_preservation(ctx, sparse):
    x = O.synth_lowrank(0, 2500, 300, 20, 0.9, 0.01, 4)
    if sparse:
        x = x * (np.random.default_rng(5).uniform(0, 1, x.shape) < 0.05)
    xin = lp.SparseMatrix.from_dense(x) if sparse else x
    cfg = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=8, l=16, projection=lp.ProjectionSpec(seed=7))
    ma = lp.reduce_lazy_spca(xin, cfg, ctx=ctx)
    mb = lp.reduce_spca(xin, cfg, ctx=ctx)
    rep = lp.distance_preservation(xin, ma, mb, max_pairs=1000, seed=9, ctx=ctx)
    pairs = np.array(O.pair_sample(x.shape[0], 1000, 9))
    assert np.array_equal(rep.pair_i, pairs[:, 0]) and np.array_equal(rep.pair_j, pairs[:, 1])
    orig = np.linalg.norm(x[pairs[:, 0]] - x[pairs[:, 1]], axis=1)
    ya, yb = x @ ma.v, x @ mb.v
    ra = np.linalg.norm(ya[pairs[:, 0]] - ya[pairs[:, 1]], axis=1)
    rb = np.linalg.norm(yb[pairs[:, 0]] - yb[pairs[:, 1]], axis=1)
    assert np.allclose(rep.original, orig, rtol=1e-12)
    assert np.allclose(rep.reduced_a, ra, rtol=1e-10)
    assert np.allclose(rep.reduced_b, rb, rtol=1e-10)
    assert rep.max_contraction_violation == pytest.approx(max((ra - orig).max(), (rb - orig).max()), abs=1e-9)
    assert rep.max_contraction_violation <= 1e-9  # orthonormal maps contract
    assert rep.max_map_discrepancy == pytest.approx(np.abs(ra - rb).max(), abs=1e-9)
    # few rows: every pair, in order
    small = lp.distance_preservation(x[:20], ma, max_pairs=1000, ctx=ctx)
    assert len(small.pair_i) == 190 and small.pair_i[0] == 0 and small.pair_j[0] == 1
    assert small.max_map_discrepancy == 0.0
