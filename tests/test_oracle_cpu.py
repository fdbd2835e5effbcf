"""CPU: the oracle restatement pinned against the reference's golden vectors.

tests/golden/*.npz were produced by the compiled reference (make_golden.py);
here the numpy restatement (oracle/lazypca_oracle.py) must reproduce them —
bit for bit for Omega (integer RNG + IEEE arithmetic), to ~1e-12 for the
floating-point reducers — before it is trusted as the GPU checker.
"""
import math

import numpy as np
import pytest

from oracle import lazypca_oracle as O


def _omega_cases(golden):
    keys = [k for k in golden.omega.files if not k.endswith(("_scale", "_density"))]
    for key in keys:
        kind, n, l, s = key.split("_")
        yield key, int(kind[1:]), int(n[1:]), int(l[1:]), int(s[1:]), float(golden.omega[key + "_density"])


def test_omega_bit_exact_against_reference_golden(golden):
    for key, kind, n, l, seed, d in _omega_cases(golden):
        if kind == 0:
            om, sc = O.gen_gaussian(n, l, seed)
        else:
            om, sc = O.gen_very_sparse(n, l, d, seed)
        ref = golden.omega[key]
        assert np.array_equal(om.view(np.uint64), np.asfortranarray(ref).view(np.uint64)), key
        assert sc == float(golden.omega[key + "_scale"])


def test_omega_moments_like_reference_suite():
    # test_projection.cpp "gaussian entries pass CLT-scale moment checks"
    om, sc = O.gen_gaussian(10000, 50, 42)
    assert sc == pytest.approx(math.sqrt(50.0), rel=1e-14)
    assert abs(om.mean()) <= 0.01
    assert 0.98 <= om.var() <= 1.02


def test_density_policy_known_answers(golden):
    # test_projection.cpp:103-121
    assert O.density_for("aggressive", 100) == pytest.approx(0.046051701859880914, rel=1e-15)
    assert O.density_for("conservative", 100) == pytest.approx(0.1, rel=1e-15)
    assert O.density_for("aggressive", 100) == float(golden.kat["density_aggr_100"])
    with pytest.raises(ValueError):
        O.density_for("aggressive", 1)


def test_reducers_match_reference_golden(golden):
    r = golden.reducers
    x = r["x"]
    v, sig, sc = O.reduce_lazy_spca(x, 6, 10, 7)
    assert np.max(np.abs(sig - r["lazy_spca_sigma"]) / r["lazy_spca_sigma"]) < 1e-12
    assert np.max(np.abs(v - r["lazy_spca_v"])) < 1e-10
    v, sig, sc = O.reduce_spca(x, 6, 10, 7)
    assert np.max(np.abs(sig - r["spca_sigma"]) / r["spca_sigma"]) < 1e-12
    assert np.max(np.abs(v - r["spca_v"])) < 1e-10
    v, sc = O.reduce_rp(x.shape[1], 8, 7)
    assert np.array_equal(v, r["rp_v"]) and sc == float(r["rp_scale"])
    assert np.max(np.abs(O.apply_map(x, r["lazy_spca_v"]) - r["lazy_spca_y"])) < 1e-11


def test_truncated_svd_matches_reference_golden(golden):
    r = golden.reducers
    sig, v, ut = O.truncated_svd_via_gram(r["f"], 6)
    assert np.max(np.abs(sig - r["tsvd_sigma"]) / r["tsvd_sigma"][0]) < 1e-12
    assert np.max(np.abs(v - r["tsvd_v"])) < 1e-9


def test_diagonal_known_answer(golden):
    # test_reducer.cpp:118-135
    x = np.diag([5.0, 4.0, 3.0, 2.0, 1.0])
    om = np.zeros((5, 2))
    om[0, 0] = om[1, 1] = 1.0
    q = O.orth(x @ om)
    sig, v, _ = O.truncated_svd_via_gram(q.T @ x, 2)
    assert np.allclose(sig, golden.kat["diag_sigma"], rtol=1e-12)
    assert np.allclose(np.abs(v), np.abs(golden.kat["diag_v"]), atol=1e-12)


def test_rank_deficiency_guard():
    # test_reducer.cpp "rank-deficient data trips the lazy route's spectrum guard"
    rng = np.random.default_rng(62)
    x = np.outer(rng.uniform(-1, 1, 20), rng.uniform(-1, 1, 10))
    with pytest.raises(O.RankDeficiency):
        O.reduce_lazy_spca(x, 3, 3, 37)


def test_spca_lazy_share_subspace_at_k_equals_l(golden):
    # Proposition 2 (test_reducer.cpp:137-162): chordal <= 1e-8 at k = l
    x = golden.reducers["x"]
    vs, _, _ = O.reduce_spca(x, 8, 8, 11)
    vl, _, _ = O.reduce_lazy_spca(x, 8, 8, 11)
    assert O.chordal_distance(vs, vl) <= 1e-8


def test_power_scheme_keeps_subspace_and_improves_capture():
    # Builder extension (not in the reference): q=1 captures the top subspace better.
    x = O.synth_lowrank(0, 800, 200, 40, 0.95, 0.01, 3)
    _, s_true, vt = np.linalg.svd(x, full_matrices=False)
    top = vt[:8].T
    v0, _, _ = O.reduce_lazy_spca(x, 8, 12, 5, power_iters=0)
    v1, _, _ = O.reduce_lazy_spca(x, 8, 12, 5, power_iters=1)
    assert O.chordal_distance(v1, top) < O.chordal_distance(v0, top)


def test_pair_sampler_is_deterministic():
    a = O.pair_sample(1000, 50, 9)
    b = O.pair_sample(1000, 50, 9)
    assert a == b and all(i < j for i, j in a)


def test_oracle_matches_live_reference(ref):
    """Where the compiled reference is available, pin the oracle on fresh cases too."""
    x = O.synth_lowrank(0, 900, 150, 20, 0.9, 0.01, 77)
    for method, fn in [(2, O.reduce_lazy_spca), (1, O.reduce_spca)]:
        v, sig, _ = fn(x, 7, 12, 3)
        rv, rs, _, _ = ref.reduce(method, x, 7, 12, 3)
        assert np.max(np.abs(sig - rs) / rs) < 1e-11
        assert np.max(np.abs(v - rv)) < 1e-9
    om, _ = O.gen_gaussian(3000, 3, 2**63 + 5)
    rom, _ = ref.regenerate(0, 3000, 3, 1.0, 2**63 + 5)
    assert np.array_equal(om, rom)
