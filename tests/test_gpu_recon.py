"""GPU: residual-norm metrics on the device (proj/core/src/metrics.cpp:148-308,
spectral_norm.cpp:23-77) against the compiled reference on the same inputs:
dense fp64 / fp32 and sparse X, both residual routes, the attached bound, the
row-space variant, spectral_norm, and the reference's own property tests
(proj/tests/test_metrics.cpp:94-150): route agreement, exact cover, monotone
in the sketch width."""
import numpy as np
import pytest

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

pytestmark = pytest.mark.gpu

QR, LAZY = lp.ResidualRoute.qr, lp.ResidualRoute.lazy


def _problem(seed, m=300, n=120, l=10, density=0.3):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (m, n)) * (rng.uniform(0, 1, (m, n)) < density)
    u = rng.uniform(-1, 1, (m, l))
    return x, u


@pytest.mark.parametrize("kind", ["f64", "f32", "sparse"])
@pytest.mark.parametrize("route", [QR, LAZY])
def test_reconstruction_error_vs_reference(ctx, ref, kind, route):
    x, u = _problem(1)
    if kind == "f32":
        x = x.astype(np.float32)
    xin = lp.SparseMatrix.from_dense(x) if kind == "sparse" else x
    rep = lp.reconstruction_error(xin, u, route, 6, 10, with_bound=True, ctx=ctx)
    spec, frob, s, b = ref.reconstruction_error(int(route), x, u, 6, 10, with_bound=True)
    assert rep.frobenius_error == pytest.approx(frob, rel=1e-11)
    assert rep.spectral_error == pytest.approx(spec, rel=1e-7)  # both stop at a 1e-8 relative gap
    assert rep.sigma_k_plus_1 == pytest.approx(s, rel=1e-10)
    assert rep.bound == pytest.approx(b, rel=1e-10)


def test_routes_agree_and_norm_ordering(ctx):
    for trial in range(4):
        x, u = _problem(10 + trial, m=80, n=50, l=6, density=0.4)
        q = lp.reconstruction_error(x, u, QR, 4, 6, ctx=ctx)
        z = lp.reconstruction_error(x, u, LAZY, 4, 6, ctx=ctx)
        assert 0.0 <= q.spectral_error <= q.frobenius_error + 1e-12
        assert abs(q.spectral_error - z.spectral_error) <= 1e-9 * (1 + q.spectral_error)
        assert abs(q.frobenius_error - z.frobenius_error) <= 1e-9 * (1 + q.frobenius_error)
        assert q.bound is None and q.sigma_k_plus_1 is None


def test_exact_cover_reconstructs_to_zero(ctx):
    x = O.synth_lowrank(0, 240, 160, 4, 0.9, 0.0, 3)  # rank 4
    omega = np.random.default_rng(5).standard_normal((160, 4))
    u = x @ omega
    scale = lp.spectral_norm(x, ctx=ctx)
    for route in (QR, LAZY):
        assert lp.reconstruction_error(x, u, route, 4, 4, ctx=ctx).spectral_error <= 1e-9 * scale


def test_wider_sketch_never_hurts(ctx):
    x, u8 = _problem(20, m=150, n=90, l=8)
    narrow = lp.reconstruction_error(x, u8[:, :6], QR, 4, 6, ctx=ctx).spectral_error
    wide = lp.reconstruction_error(x, u8, QR, 4, 8, ctx=ctx).spectral_error
    assert wide <= narrow + 1e-10


def test_bound_omitted_when_l_is_k_plus_1_and_above_the_densify_limit(ctx):
    x, u = _problem(30, m=60, n=40, l=8)
    assert lp.reconstruction_error(x, u, QR, 7, 8, with_bound=True, ctx=ctx).bound is None
    assert lp.reconstruction_error(x, u, QR, 5, 8, with_bound=True, densify_limit=50, ctx=ctx).bound is None


def test_errors(ctx):
    x, u = _problem(40, m=50, n=30, l=5)
    with pytest.raises(lp.DimensionError, match="rows but X has"):
        lp.reconstruction_error(x, u[:40], QR, 3, 5, ctx=ctx)
    with pytest.raises(lp.DimensionError, match="columns but l = 6"):
        lp.reconstruction_error(x, u, QR, 3, 6, ctx=ctx)
    dup = np.hstack([u, u[:, :1]])  # rank deficient: the lazy route's Cholesky fails at pivot 5
    with pytest.raises(lp.RankDeficiencyError) as e:
        lp.reconstruction_error(x, dup, LAZY, 3, 6, ctx=ctx)
    assert e.value.index() == 5


def test_row_space_and_spectral_norm_vs_reference(ctx, ref):
    x, _ = _problem(50)
    v, _ = np.linalg.qr(np.random.default_rng(51).standard_normal((120, 7)))
    for xin in (x, lp.SparseMatrix.from_dense(x)):
        rep = lp.row_space_reconstruction_error(xin, v, ctx=ctx)
        spec, frob = ref.row_space_reconstruction_error(x, v)
        assert rep.frobenius_error == pytest.approx(frob, rel=1e-11)
        assert rep.spectral_error == pytest.approx(spec, rel=1e-7)
        assert lp.spectral_norm(xin, ctx=ctx) == pytest.approx(ref.spectral_norm(x), rel=1e-7)
    with pytest.raises(lp.InvalidArgumentError, match="orthonormal"):
        lp.row_space_reconstruction_error(x, v * 2.0, ctx=ctx)


def test_fit_then_reconstruction_error_on_a_device_sketch(ctx):
    """The metric on a fit's own sketch, with X and U as CUDA tensors."""
    import torch
    m, n, r, l = 20000, 512, 40, 48
    x = torch.empty((m, n), dtype=torch.float32, device="cuda")
    lp.synth_lowrank(x, 0, r, 0.9, 0.01, 1000, ctx=ctx)
    omega = torch.randn((n, l), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    u = x.double() @ omega
    torch.cuda.synchronize()
    rep = lp.reconstruction_error(x, u, LAZY, 32, l, ctx=ctx)
    xd = x.double()
    q, _ = torch.linalg.qr(u)
    res = xd - q @ (q.T @ xd)
    assert rep.frobenius_error == pytest.approx(torch.linalg.norm(res).item(), rel=1e-6)
    assert rep.spectral_error == pytest.approx(torch.linalg.matrix_norm(res, 2).item(), rel=1e-5)
