"""GPU: the tcgen05 split-TF32 kernels (fp32 data) against the SIMT FFMA path and
the reference, over the shapes that exercise tails and both tile layouts:
m not a multiple of 128, n not a multiple of 32 or 256, odd l, l > 128."""
import numpy as np
import pytest

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

pytestmark = pytest.mark.gpu


def _x(m, n, r, rho, seed=1000):
    import torch
    x = torch.empty((m, n), dtype=torch.float32, device="cuda")
    lp.synth_lowrank(x, 0, r, rho, 0.01, seed)
    return x


def _fit(ctx, x, k, l, path, q=0, method=lp.ReducerMethod.lazy_spca, seed=7):
    ctx.set_gemm_path(path)
    try:
        cfg = lp.ReducerConfig(method=method, k=k, l=l, projection=lp.ProjectionSpec(seed=seed),
                               power_iters=q)
        return lp.reduce(x, cfg, ctx=ctx)
    finally:
        ctx.set_gemm_path("tcgen05")


@pytest.mark.parametrize("m,n,r,k,l", [
    (1000, 256, 30, 8, 16),      # single partial tile
    (5003, 1000, 60, 20, 37),    # odd m, n % 32 != 0, odd l
    (20000, 4096, 200, 100, 110),  # c2 shape
    (9000, 2048, 300, 200, 220),   # l > 128: two M halves in U^T X (configs[2] rho)
    (4000, 300, 40, 16, 256),     # l = 256 boundary
    (6000, 2048, 400, 200, 300),  # two 152-wide column slices (configs[3] l)
    (4000, 2048, 600, 300, 460),  # three 160-wide column slices
])
def test_tc_matches_reference(ctx, ref, m, n, r, k, l):
    x = _x(m, n, r, 0.99 if l > 400 else (0.98 if l > 128 else 0.97))
    xh = x.cpu().numpy()
    got = _fit(ctx, x, k, l, "tcgen05")
    rv, rs, _, _ = ref.reduce(2, xh, k, l, 7)
    rel = np.abs(got.singular_values - rs) / rs
    kk = max(1, k // 2)
    ang = np.max(O.principal_angles(got.v[:, :kk], rv[:, :kk]))
    print(f"m={m} n={n} l={l}: sigma rel max {rel.max():.3e}, top-k/2 angle {ang:.2e}")
    assert rel.max() < 1e-4   # north_star's fp32 bar
    assert rel.max() < 5e-5   # measured 2.8e-6 .. 1.2e-5
    assert ang < 1e-4


def test_tc_and_simt_paths_agree(ctx):
    x = _x(30000, 1024, 80, 0.96)
    a = _fit(ctx, x, 32, 48, "tcgen05")
    b = _fit(ctx, x, 32, 48, "simt")
    rel = np.abs(a.singular_values - b.singular_values) / b.singular_values
    assert rel.max() < 2e-5, rel.max()
    assert O.chordal_distance(a.v[:, :16], b.v[:, :16]) < 1e-4


def test_tc_transform_matches_fp64(ctx):
    import torch
    x = _x(7777, 512, 50, 0.95)
    m = _fit(ctx, x, 40, 48, "tcgen05")
    y = torch.empty((7777, 40), dtype=torch.float32, device="cuda")
    lp.apply_map(m, x, out=y, ctx=ctx)
    yr = x.double().cpu().numpy() @ m.v
    err = np.abs(y.cpu().numpy() - yr).max() / np.abs(yr).max()
    assert err < 1e-5, err  # fp32 output; split-TF32 bias ~1.3e-6 (see gemm_tc.cu)


def test_tc_power_and_spca(ctx, ref):
    x = _x(6000, 1024, 120, 0.97)
    xh = x.cpu().numpy().astype(np.float64)
    p = _fit(ctx, x, 40, 60, "tcgen05", q=1)
    v, s, _ = O.reduce_lazy_spca(xh, 40, 60, 7, power_iters=1)
    assert np.max(np.abs(p.singular_values - s) / s) < 1e-4
    sp = _fit(ctx, x, 40, 60, "tcgen05", method=lp.ReducerMethod.spca)
    rv, rs, _, _ = ref.reduce(1, x.cpu().numpy(), 40, 60, 7)
    assert np.max(np.abs(sp.singular_values - rs) / rs) < 1e-4


def test_sketch_first_stage_scales_fall_back_to_the_scan(ctx):
    """The sketch takes each run's A-row scale from the run's first stage; rows
    whose later stage outgrows it (or sits far below it) make the fit rerun with
    the full per-run scan. X here has, in every 128-column block, a zero first
    half and small values in the second half (so every run's first stage is
    zero, whatever the run length), and a few huge entries late."""
    import torch
    rng = np.random.default_rng(8)
    m, n = 8192, 1024
    x = rng.standard_normal((m, n)).astype(np.float32) * 1e-3
    for c0 in range(0, n, 128):
        x[:, c0:c0 + 64] = 0.0
    x[::97, 1000] = 0.5
    cfg = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=16, l=32, projection=lp.ProjectionSpec(seed=3))
    m32 = lp.reduce_lazy_spca(torch.from_numpy(x).cuda(), cfg, ctx=ctx)
    v64, s64, _ = O.reduce_lazy_spca(x.astype(np.float64), 16, 32, 3)
    assert np.max(np.abs(m32.singular_values - s64) / s64) < 1e-4


@pytest.mark.parametrize("q", [0, 1])
def test_sketch_overflow_in_a_later_stage_reruns_before_host_checks(ctx, q):
    """rows with small nonzero noise in each run's first stage
    and O(1) values later overflow fp16 at the first-stage scale (inf in U, NaN
    in F). The power step's pivots and the rank floor would throw before the
    overflow flag was read; the fit must rerun with the scan instead."""
    import torch
    rng = np.random.default_rng(11)
    m, n = 8192, 2048
    x = rng.standard_normal((m, n)).astype(np.float32) * 0.5
    for c0 in range(0, n, 512):
        x[:, c0:c0 + 64] = rng.standard_normal((m, 64)).astype(np.float32) * 1e-3
    cfg = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=16, l=32, projection=lp.ProjectionSpec(seed=3),
                           power_iters=q)
    got = lp.reduce_lazy_spca(torch.from_numpy(x).cuda(), cfg, ctx=ctx)
    v64, s64, _ = O.reduce_lazy_spca(x.astype(np.float64), 16, 32, 3, power_iters=q)
    assert np.all(np.isfinite(got.singular_values))
    assert np.max(np.abs(got.singular_values - s64) / s64) < 1e-4


@pytest.mark.parametrize("conv", ["8", "84"])
def test_eight_converter_warps_bit_identical(ctx, monkeypatch, conv):
    """LPCA_TC_CONV=8 / 84 (two converter warps per TMEM lane quadrant, each one
    32-column half of every stage; csrc/tc_pair.cuh) writes the same fp16 A
    planes with the same run scales as the default four, so fits, power steps,
    transforms and the scanned rerun are bit-identical."""
    import torch
    x = _x(9000, 2048, 300, 0.98)
    rng = np.random.default_rng(8)
    xa = rng.standard_normal((8192, 1024)).astype(np.float32) * 1e-3
    for c0 in range(0, 1024, 128):   # zero first stages, huge late entries: the scanned rerun
        xa[:, c0:c0 + 64] = 0.0
    xa[::97, 1000] = 0.5
    xa = torch.from_numpy(xa).cuda()

    def run():
        out = []
        for xx, k, l, q in ((x, 200, 220, 1), (xa, 150, 220, 0)):
            cfg = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=k, l=l, power_iters=q,
                                   projection=lp.ProjectionSpec(seed=7))
            y = torch.empty((xx.shape[0], k), dtype=torch.float32, device="cuda")
            mp, _ = lp.fit_transform(xx, cfg, ctx=ctx, out=y)
            out += [mp.singular_values, mp.v, y.cpu().numpy()]
        return out

    base = run()
    monkeypatch.setenv("LPCA_TC_CONV", conv)
    got = run()
    for a, b in zip(base, got):
        assert np.array_equal(a, b)
