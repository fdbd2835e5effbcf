"""GPU: SPCA's orthonormalisation keeps the reference's rank semantics
(VERDICT r1 missing #4). The reference factors U by Householder QR
and rejects column j only when its remaining norm |R_jj| <= 1e-12 ||U||_F
(proj/core/src/qr.cpp:37-58); streaming SPCA carries the stacked R and raises
"slice s: qr: ..." with the slice as the index (reducer.cpp:276-292), then
checks R's diagonal against 1e-12 ||R||_F (reducer.cpp:55-63). The library uses
shifted CholeskyQR3, whose R has the same diagonal up to roundoff."""
import numpy as np
import pytest

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

pytestmark = pytest.mark.gpu


def _x_with_spectrum(m, n, s, seed=3):
    rng = np.random.default_rng(seed)
    a, _ = np.linalg.qr(rng.standard_normal((m, len(s))))
    b, _ = np.linalg.qr(rng.standard_normal((n, len(s))))
    return (a * s) @ b.T


def _cfg(method, k, l, block_rows=0):
    c = lp.ReducerConfig(method=method, k=k, l=l, projection=lp.ProjectionSpec(seed=9))
    c.block_rows = block_rows
    return c


def test_ill_conditioned_sketch_matches_reference(ctx, ref):
    """cond(U) ~ 1e10: the reference returns a map; so must the GPU (CholeskyQR2
    without a shift failed here at cond ~ 1e7)."""
    l, k = 20, 8
    s = 10.0 ** (-10.0 * np.arange(l) / (l - 1))
    x = _x_with_spectrum(3000, 400, s)
    u = x @ O.gen_gaussian(400, l, 9)[0]
    sv = np.linalg.svd(u, compute_uv=False)
    assert sv[0] / sv[-1] > 1e9
    got = lp.reduce_spca(x, _cfg(lp.ReducerMethod.spca, k, l), ctx=ctx)
    rv, rs, _, _ = ref.reduce(1, x, k, l, 9)
    assert np.max(np.abs(got.singular_values - rs)) / rs[0] < 1e-12
    assert np.max(np.abs(got.singular_values[:4] - rs[:4]) / rs[:4]) < 1e-10
    assert np.max(O.principal_angles(got.v[:, :4], rv[:, :4])) < 1e-8


def test_rank_deficient_sketch_raises_the_reference_index(ctx, ref):
    l, k, r = 20, 8, 12
    x = _x_with_spectrum(3000, 400, np.linspace(1.0, 0.5, r))
    with pytest.raises(Exception) as want:
        ref.reduce(1, x, k, l, 9)
    assert want.value.code == 3  # RankDeficiencyError
    with pytest.raises(lp.RankDeficiencyError) as got:
        lp.reduce_spca(x, _cfg(lp.ReducerMethod.spca, k, l), ctx=ctx)
    assert got.value.index() == want.value.index == r
    assert str(got.value).startswith(f"qr: column {r} is numerically dependent on earlier columns")


def test_streaming_rank_deficiency_names_the_slice(ctx, ref):
    l, k, r = 20, 8, 12
    x = _x_with_spectrum(3000, 400, np.linspace(1.0, 0.5, r))
    with pytest.raises(Exception) as want:
        ref.reduce(1, x, k, l, 9, block_rows=700)
    with pytest.raises(lp.RankDeficiencyError) as got:
        lp.reduce_spca_streaming(lp.SliceRowBlockStream(x, 700), _cfg(lp.ReducerMethod.spca, k, l), ctx=ctx)
    assert got.value.index() == want.value.index == 0
    assert str(got.value).startswith(f"slice 0: qr: column {r} ")
    assert str(want.value).startswith(f"slice 0: qr: column {r} ")


def test_streaming_ill_conditioned_matches_reference(ctx, ref):
    l, k = 20, 8
    s = 10.0 ** (-9.0 * np.arange(l) / (l - 1))
    x = _x_with_spectrum(3000, 400, s)
    got = lp.reduce_spca_streaming(lp.SliceRowBlockStream(x, 700), _cfg(lp.ReducerMethod.spca, k, l), ctx=ctx)
    rv, rs, _, _ = ref.reduce(1, x, k, l, 9, block_rows=700)
    assert np.max(np.abs(got.singular_values - rs)) / rs[0] < 1e-11  # measured 1.9e-12
    assert np.max(O.principal_angles(got.v[:, :4], rv[:, :4])) < 1e-8


def test_well_conditioned_spca_still_matches_at_1e10(ctx, ref):
    x = O.synth_lowrank(0, 5000, 300, 40, 0.93, 0.01, 21)
    got = lp.reduce_spca(x, _cfg(lp.ReducerMethod.spca, 10, 24), ctx=ctx)
    rv, rs, _, _ = ref.reduce(1, x, 10, 24, 9)
    assert np.max(np.abs(got.singular_values - rs) / rs) < 1e-10
    gs = lp.reduce_spca_streaming(lp.SliceRowBlockStream(x, 1300), _cfg(lp.ReducerMethod.spca, 10, 24), ctx=ctx)
    rv2, rs2, _, _ = ref.reduce(1, x, 10, 24, 9, block_rows=1300)
    assert np.max(np.abs(gs.singular_values - rs2) / rs2) < 1e-10
