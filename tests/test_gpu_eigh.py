"""GPU: the device symmetric eigensolvers (tridiagonal route and Jacobi) against
the reference's tridiag_eigh / jacobi_eigh and LAPACK, on the spectra the fit
produces (G = F F^T with sigma^4 decay) and on the reference's edge cases."""
import numpy as np
import pytest

import paper_1709_07175_b200 as lp

pytestmark = pytest.mark.gpu

METHODS = ["tridiag", "jacobi"]


def _gram_like(l, n, rho, seed):
    rng = np.random.default_rng(seed)
    s = (rho ** np.arange(l)) ** 2 * 1e6 + 1e-3
    a, _ = np.linalg.qr(rng.standard_normal((l, l)))
    b, _ = np.linalg.qr(rng.standard_normal((n, l)))
    f = (a * s) @ b.T
    g = f @ f.T
    return (g + g.T) / 2


def _check(a, e, tol_res=1e-12, tol_orth=1e-12):
    lsz = a.shape[0]
    w = np.linalg.eigvalsh(a)[::-1]
    scale = max(np.abs(w).max(), 1e-300)
    assert np.all(np.diff(e.eigenvalues) <= 0), "eigenvalues not descending"
    assert np.max(np.abs(e.eigenvalues - w)) <= 1e-13 * scale * max(1, lsz / 10)
    v = e.eigenvectors
    assert np.linalg.norm(v.T @ v - np.eye(lsz)) <= tol_orth * lsz
    assert np.linalg.norm(a @ v - v * e.eigenvalues) <= tol_res * np.linalg.norm(a) * lsz


@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("l,n,rho", [(20, 1000, 0.9), (110, 4096, 0.97), (220, 4096, 0.98)])
def test_gram_spectra(ctx, method, l, n, rho):
    a = _gram_like(l, n, rho, l)
    _check(a, lp.eigh(a, ctx, method))


@pytest.mark.parametrize("l", [31, 32, 33, 64, 65, 127, 128, 129, 160, 300, 512])
def test_tridiag_size_classes(ctx, l):
    """Every kernel variant boundary: register tridiagonalisation (l <= 32, 64,
    128), shared/global above it; register back-transformation up to 512."""
    a = _gram_like(l, 4 * l, 0.97, l)
    _check(a, lp.eigh(a, ctx, "tridiag"))
    rng = np.random.default_rng(l)
    b = rng.standard_normal((l, l))
    b = (b + b.T) / 2  # indefinite, unstructured
    _check(b, lp.eigh(b, ctx, "tridiag"))


@pytest.mark.parametrize("l", [300, 512])
def test_gram_spectra_large_tridiag(ctx, l):
    a = _gram_like(l, 4 * l, 0.99, l)
    _check(a, lp.eigh(a, ctx, "tridiag"))


@pytest.mark.parametrize("method", METHODS)
def test_known_answers(ctx, golden, method):
    k = golden.kat
    e = lp.eigh(k["eig3_a"], ctx, method)
    assert np.allclose(e.eigenvalues, [4.0, 2.0, -1.0], atol=1e-12)
    e4 = lp.eigh(k["eig4_a"], ctx, method)
    assert np.allclose(e4.eigenvalues, [3.0, 3.0, 1.0, -2.0], atol=1e-12)
    _check(k["eig4_a"], e4)


@pytest.mark.parametrize("method", METHODS)
def test_tiny_and_degenerate(ctx, method):
    _check(np.array([[2.5]]), lp.eigh(np.array([[2.5]]), ctx, method))
    a2 = np.array([[2.0, 1.0], [1.0, 2.0]])
    _check(a2, lp.eigh(a2, ctx, method))
    _check(np.zeros((5, 5)), lp.eigh(np.zeros((5, 5)), ctx, method))
    _check(np.eye(7) * 3.0, lp.eigh(np.eye(7) * 3.0, ctx, method))
    rng = np.random.default_rng(3)
    u = rng.standard_normal((40, 3))
    low = u @ u.T  # rank 3, 37 zero eigenvalues
    _check(low, lp.eigh(low, ctx, method), tol_res=1e-12, tol_orth=1e-11)
    q, _ = np.linalg.qr(rng.standard_normal((30, 30)))
    rep = q @ np.diag(np.repeat([5.0, 2.0, -1.0], 10)) @ q.T
    rep = (rep + rep.T) / 2
    _check(rep, lp.eigh(rep, ctx, method))


def test_tridiag_matches_reference_tridiag_eigh(ctx, ref):
    a = _gram_like(64, 512, 0.95, 9)
    want, _ = ref.eigh(a, "tridiag")
    got = lp.eigh(a, ctx, "tridiag")
    assert np.max(np.abs(got.eigenvalues - want)) <= 1e-13 * want[0]


def test_asymmetric_input_rejected(ctx):
    for method in METHODS:
        with pytest.raises(lp.InvalidArgumentError):
            lp.eigh(np.array([[1.0, 2.0], [0.0, 1.0]]), ctx, method)
