"""CPU: the residual-norm metrics' host pieces and the oracle that pins them.

* bound_value (proj/core/src/metrics.cpp:136-146) against the reference's own
  known answers (proj/tests/test_metrics.cpp:84-92) — host arithmetic, no GPU.
* The compiled reference's reconstruction_error / row_space_reconstruction_error /
  spectral_norm against independent numpy (SVD) values, so the GPU parity tests
  compare against a checked oracle."""
import numpy as np
import pytest

import paper_1709_07175_b200 as lp


def test_bound_value_known_answers():
    assert lp.bound_value(100, 100, 8, 10, 1.0) == pytest.approx(127.49110640673518, rel=1e-15)
    assert lp.bound_value(100, 100, 8, 10, 0.5) == pytest.approx(127.49110640673518 * 0.5, rel=1e-15)
    assert lp.bound_value(100, 25, 8, 10, 1.0) == pytest.approx(1.0 + 4.0 * np.sqrt(10.0) * 5.0, rel=1e-15)
    for l in (9, 8):
        with pytest.raises(lp.InvalidArgumentError, match="l >= k \\+ 2"):
            lp.bound_value(100, 100, 8, l, 1.0)


def _problem(seed, m=60, n=40, l=8, density=0.5):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (m, n)) * (rng.uniform(0, 1, (m, n)) < density)
    u = rng.uniform(-1, 1, (m, l))
    return x, u


@pytest.mark.parametrize("route", [0, 1])
def test_oracle_reconstruction_error_vs_numpy(ref, route):
    x, u = _problem(1)
    q, _ = np.linalg.qr(u)
    r = x - q @ (q.T @ x)
    spec, frob, s, b = ref.reconstruction_error(route, x, u, 5, 8, with_bound=True)
    assert frob == pytest.approx(np.linalg.norm(r), rel=1e-10)
    assert spec == pytest.approx(np.linalg.norm(r, 2), rel=1e-6)
    sv = np.linalg.svd(x, compute_uv=False)
    assert s == pytest.approx(sv[5], rel=1e-10)
    assert b == pytest.approx(lp.bound_value(60, 40, 5, 8, sv[5]), rel=1e-10)


def test_oracle_row_space_and_spectral_norm_vs_numpy(ref):
    x, _ = _problem(2)
    v, _ = np.linalg.qr(np.random.default_rng(3).standard_normal((40, 6)))
    spec, frob = ref.row_space_reconstruction_error(x, v)
    r = x - (x @ v) @ v.T
    assert frob == pytest.approx(np.linalg.norm(r), rel=1e-10)
    assert spec == pytest.approx(np.linalg.norm(r, 2), rel=1e-6)
    assert ref.spectral_norm(x) == pytest.approx(np.linalg.norm(x, 2), rel=1e-6)
