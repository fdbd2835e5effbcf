"""GPU: the one-CTA Cholesky (blocked by 8-column panels) and the shared-memory
L^-1 behind SPCA's shifted CholeskyQR3 and the power step, at sketch widths that
exercise their edges: l = 2 (the reference's minimum), l below one panel, l one past a panel, ragged last panels,
the largest l the one-CTA path takes (236: the packed triangle fills shared
memory) and the first l past it (240: the multi-launch panel path). fp64 data,
against the compiled reference's SPCA (reducer.cpp:192-214; qr.cpp:37-132) at
the north-star fp64 bar (sigma 1e-10 per value), and the Lazy power fit against
the reference kernels composed (oracle/ref_capi.cpp ref_lazy_power_fit_transform).
A rank-deficient sketch whose dependent column falls inside a later panel
raises the reference's index."""
import numpy as np
import pytest

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

pytestmark = pytest.mark.gpu

M, N = 3000, 400


def _x():
    return O.synth_lowrank(0, M, N, 300, 0.985, 0.01, 21)


def _cfg(method, k, l, q=0):
    return lp.ReducerConfig(method=method, k=k, l=l, projection=lp.ProjectionSpec(seed=9), power_iters=q)


@pytest.mark.parametrize("l", [2, 5, 8, 9, 17, 63, 236, 240])
def test_spca_matches_reference_across_panel_shapes(ctx, ref, l):
    x = _x()
    k = max(1, l // 2)
    got = lp.reduce_spca(x, _cfg(lp.ReducerMethod.spca, k, l), ctx=ctx)
    rv, rs, _, _ = ref.reduce(1, x, k, l, 9)
    err = np.max(np.abs(got.singular_values - rs) / rs)
    print(f"spca l={l}: sigma {err:.1e}")
    assert err < 1e-10, (l, err)
    kk = max(1, k // 2)
    assert np.max(O.principal_angles(got.v[:, :kk], rv[:, :kk])) < 1e-8, l


@pytest.mark.parametrize("l", [9, 63, 236, 240])
def test_power_step_orthonormalisation_matches_composed_reference(ctx, ref, l):
    x = _x()
    k = l // 2
    got = lp.reduce_lazy_spca(x, _cfg(lp.ReducerMethod.lazy_spca, k, l, q=1), ctx=ctx)
    _, rv, rs, _ = ref.lazy_power_fit_transform(x, k, l, 9, 1, want_y=False)
    err = np.max(np.abs(got.singular_values - rs) / rs)
    print(f"lazy q=1 l={l}: sigma {err:.1e}")
    assert err < 1e-10, (l, err)
    kk = k // 2
    assert np.max(O.principal_angles(got.v[:, :kk], rv[:, :kk])) < 1e-8, l


def test_rank_deficiency_inside_a_later_panel(ctx, ref):
    l, k, r = 30, 8, 19  # column 19: the fourth of the third 8-column panel
    rng = np.random.default_rng(3)
    a, _ = np.linalg.qr(rng.standard_normal((M, r)))
    b, _ = np.linalg.qr(rng.standard_normal((N, r)))
    x = (a * np.linspace(1.0, 0.5, r)) @ b.T
    with pytest.raises(Exception) as want:
        ref.reduce(1, x, k, l, 9)
    assert want.value.code == 3  # RankDeficiencyError
    with pytest.raises(lp.RankDeficiencyError) as got:
        lp.reduce_spca(x, _cfg(lp.ReducerMethod.spca, k, l), ctx=ctx)
    assert got.value.index() == want.value.index == r
