"""GPU: BASELINE configs[3] and configs[4] shapes at reduced row counts.

* c4: fp32 X, n = 16,384, very sparse Omega (density 1/sqrt(n)), k = 256,
  l = 300 (two column slices on the tensor cores), q = 2 — against the library's
  fp64 reference-order path on the same fp32-rounded X (parity for q >= 1 is
  unpinned by the reference).
* c5: fp64 X, l = 512, q = 1 — SPCA and Lazy SPCA give the same subspace at
  k = l and the same reduced pairwise distances (the reference's acceptance
  criterion 2, proj/tests/acceptance.cpp:154-207), on rows sampled like
  distance_preservation (metrics.cpp:327-334)."""
import numpy as np
import pytest
import torch

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

pytestmark = pytest.mark.gpu


def test_c4_shape_very_sparse_omega_power2(ctx):
    m, n, r, k, l = 20000, 16384, 400, 256, 300
    x32 = torch.empty((m, n), dtype=torch.float32, device="cuda")
    lp.synth_lowrank(x32, 0, r, 0.98, 0.01, 1000, ctx=ctx)
    spec = lp.ProjectionSpec(kind=lp.ProjectionKind.very_sparse, density=1.0 / 128, seed=7)
    cfg = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=k, l=l, projection=spec, power_iters=2)
    m32 = lp.reduce_lazy_spca(x32, cfg, ctx=ctx)
    y32 = torch.empty((m, k), dtype=torch.float32, device="cuda")
    lp.apply_map(m32, x32, out=y32, ctx=ctx)  # the tensor-core transform
    x64 = x32.double()
    torch.cuda.synchronize()
    ref_ctx = lp.Context(0)
    ref_ctx.set_gemm_path("simt")
    m64 = lp.reduce_lazy_spca(x64, cfg, ctx=ref_ctx)
    y64 = torch.empty((m, k), dtype=torch.float64, device="cuda")
    lp.apply_map(m64, x64, out=y64, ctx=ref_ctx)
    s32, s64 = m32.singular_values, m64.singular_values
    assert np.max(np.abs(s32 - s64) / s64) < 1e-4
    assert np.max(O.principal_angles(m32.v[:, :k // 2], m64.v[:, :k // 2])) < 2e-5  # measured ~4e-7
    dy = y32.double() - y64
    assert (dy.norm() / y64.norm()).item() < 5e-5  # measured ~2e-6
    del m64
    ref_ctx.close()


def test_c5_shape_fp64_spca_equals_lazy_at_k_eq_l(ctx):
    m, n, r, k = 20000, 2048, 500, 256
    x = torch.empty((m, n), dtype=torch.float64, device="cuda")
    lp.synth_lowrank(x, 0, r, 0.99, 0.01, 1000, ctx=ctx)
    base = dict(k=k, l=k, projection=lp.ProjectionSpec(seed=7), power_iters=1)
    ms = lp.reduce_spca(x, lp.ReducerConfig(method=lp.ReducerMethod.spca, **base), ctx=ctx)
    ml = lp.reduce_lazy_spca(x, lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, **base), ctx=ctx)
    assert O.chordal_distance(ms.v, ml.v) <= 1e-8
    ys, yl = lp.apply_map(ms, x, ctx=ctx), lp.apply_map(ml, x, ctx=ctx)
    pairs = np.array(O.pair_sample(m, 1000, 7))
    ys, yl = np.asarray(ys), np.asarray(yl)
    ds = np.linalg.norm(ys[pairs[:, 0]] - ys[pairs[:, 1]], axis=1)
    dl = np.linalg.norm(yl[pairs[:, 0]] - yl[pairs[:, 1]], axis=1)
    assert np.max(np.abs(ds - dl)) <= 1e-9 * max(1.0, ds.max())
