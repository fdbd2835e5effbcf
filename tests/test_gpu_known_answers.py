"""GPU: the literal known-answer and property checks of the reference's unit
tests, run through this library's device kernels.

* diag(5,4,3,2,1) with the exact sketch Omega = [e1 e2]: spmm, Q, gemm_t and the
  Gram-route SVD give sigma = (5, 4) and V = (e1, e2) (test_reducer.cpp:118-135);
* chordal-distance endpoints: 0 for a subspace with itself, 2 for orthogonal
  complements at k = 2 (test_metrics.cpp:32-41);
* Omega on the device: the very sparse projection at density 1 is a sign matrix
  with scale sqrt(l); at density 0.1 it hits its density and sign balance with
  scale sqrt(l * 0.1) (test_projection.cpp:78-101); invalid specs are refused
  (test_projection.cpp:64-76);
* the variance-preserving scale: 100 random unit vectors in R^1000 keep their
  mean squared norm within 5% after the scaled projection, both families
  (test_projection.cpp:126-150)."""
import numpy as np
import pytest

import paper_1709_07175_b200 as lp

pytestmark = pytest.mark.gpu


def test_exact_sketch_recovers_a_diagonal_spectrum(ctx):
    x = lp.SparseMatrix.from_triplets(5, 5, [(i, i, 5.0 - i) for i in range(5)])
    omega = np.zeros((5, 2))
    omega[0, 0] = omega[1, 1] = 1.0
    u = lp.spmm(x, omega, ctx=ctx)
    q = np.linalg.qr(u)[0]
    f = lp.gemm_t(q, x, ctx=ctx)
    svd = lp.truncated_svd_via_gram(f, 2, ctx=ctx)
    assert svd.singular_values == pytest.approx([5.0, 4.0], rel=1e-12)
    assert abs(svd.v[0, 0]) == pytest.approx(1.0, rel=1e-12)
    assert abs(svd.v[1, 1]) == pytest.approx(1.0, rel=1e-12)


def test_chordal_distance_endpoints(ctx):
    v = np.linalg.qr(np.random.default_rng(71).standard_normal((12, 4)))[0]
    assert lp.chordal_distance(v, v, ctx=ctx) <= 1e-12
    v1, v2 = np.zeros((4, 2)), np.zeros((4, 2))
    v1[0, 0] = v1[1, 1] = 1.0
    v2[2, 0] = v2[3, 1] = 1.0
    assert lp.chordal_distance(v1, v2, ctx=ctx) == pytest.approx(2.0, rel=1e-14)


def _spec(kind, n, l, density, seed):
    s = lp.ProjectionSpec(kind=kind, density=density, seed=seed)
    s.n, s.l = n, l
    return s


def test_very_sparse_projection_at_density_one_is_a_sign_matrix(ctx):
    p = lp.regenerate(_spec(lp.ProjectionKind.very_sparse, 40, 6, 1.0, 5), ctx=ctx)
    assert np.count_nonzero(p.omega) == 240
    assert np.all(np.abs(p.omega) == 1.0)
    assert p.scale == pytest.approx(np.sqrt(6.0), rel=1e-14)


def test_very_sparse_projection_hits_its_density_and_sign_balance(ctx):
    p = lp.regenerate(_spec(lp.ProjectionKind.very_sparse, 20000, 50, 0.1, 31), ctx=ctx)
    nnz = np.count_nonzero(p.omega)
    assert 0.099 <= nnz / 1e6 <= 0.101
    plus = np.count_nonzero(p.omega > 0)
    assert abs(plus - nnz / 2) <= 4.0 * np.sqrt(nnz * 0.25)
    assert p.scale == pytest.approx(np.sqrt(50 * 0.1), rel=1e-14)


@pytest.mark.parametrize("kind,n,l,density", [
    (lp.ProjectionKind.gaussian, 10, 0, 1.0), (lp.ProjectionKind.gaussian, 10, 1, 1.0),
    (lp.ProjectionKind.gaussian, 10, 11, 1.0), (lp.ProjectionKind.very_sparse, 10, 4, 0.0),
    (lp.ProjectionKind.very_sparse, 10, 4, 1.5)])
def test_invalid_projection_specs_are_refused(ctx, kind, n, l, density):
    with pytest.raises(lp.InvalidArgumentError):
        lp.regenerate(_spec(kind, n, l, density, 0), ctx=ctx)


@pytest.mark.parametrize("kind,density", [(lp.ProjectionKind.gaussian, 1.0),
                                          (lp.ProjectionKind.very_sparse, 0.1)])
def test_variance_preserving_scale(ctx, kind, density):
    rng = np.random.default_rng(44)
    x = rng.uniform(-1.0, 1.0, (100, 1000))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    p = lp.regenerate(_spec(kind, 1000, 200, density, 7), ctx=ctx)
    y = lp.spmm(x, p.scaled_dense(), ctx=ctx)
    mean = float(np.mean(np.sum(y * y, axis=1)))
    assert 0.95 <= mean <= 1.05, mean
