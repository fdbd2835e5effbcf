"""GPU: lpca_fit_transform (one call; on the device the transform is queued
behind the fit's spectral step) gives the same map and the same Y as
reduce + apply_map, bitwise, for every reducer and input path."""
import numpy as np
import pytest
import torch

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

pytestmark = pytest.mark.gpu


def _cfg(method, k=12, l=20, **kw):
    return lp.ReducerConfig(method=method, k=k, l=l, projection=lp.ProjectionSpec(seed=7), **kw)


@pytest.mark.parametrize("method", [lp.ReducerMethod.lazy_spca, lp.ReducerMethod.spca, lp.ReducerMethod.rp])
def test_device_fused_equals_separate_calls_f32(ctx, method):
    m, n = 40000, 768
    x = torch.empty((m, n), dtype=torch.float32, device="cuda")
    lp.synth_lowrank(x, 0, 60, 0.95, 0.01, 11, ctx=ctx)
    cfg = _cfg(method, k=20 if method == lp.ReducerMethod.rp else 12, l=20)
    y1 = torch.empty((m, cfg.k), dtype=torch.float32, device="cuda")
    y2 = torch.empty_like(y1)
    mp1 = lp.reduce(x, cfg, ctx=ctx)
    lp.apply_map(mp1, x, out=y1, ctx=ctx)
    mp2, _ = lp.fit_transform(x, cfg, ctx=ctx, out=y2)
    torch.cuda.synchronize()
    assert np.array_equal(mp1.v, mp2.v)
    assert np.array_equal(mp1.singular_values, mp2.singular_values)
    assert torch.equal(y1, y2)


def test_host_fused_f64_sparse_and_streaming(ctx):
    x = O.synth_lowrank(0, 3000, 200, 20, 0.9, 0.01, 4)
    for xin in (x, lp.SparseMatrix.from_dense(x * (np.abs(x) > 1.0))):
        for cfg in (_cfg(lp.ReducerMethod.lazy_spca), _cfg(lp.ReducerMethod.lazy_spca, block_rows=700)):
            mp1 = lp.reduce(xin, cfg, ctx=ctx)
            y1 = lp.apply_map(mp1, xin, layout="row", ctx=ctx)
            mp2, y2 = lp.fit_transform(xin, cfg, ctx=ctx)
            assert np.array_equal(mp1.v, mp2.v)
            assert np.array_equal(y1, y2)


def test_fused_timings_are_filled(ctx):
    m, n = 20000, 512
    x = torch.empty((m, n), dtype=torch.float32, device="cuda")
    lp.synth_lowrank(x, 0, 40, 0.9, 0.01, 3, ctx=ctx)
    y = torch.empty((m, 10), dtype=torch.float32, device="cuda")
    tm = lp.ReducerTimings()
    lp.fit_transform(x, _cfg(lp.ReducerMethod.lazy_spca, k=10, l=16), timings=tm, ctx=ctx, out=y)
    assert tm.sketch > 0 and tm.f_form > 0 and tm.svd > 0 and tm.transform > 0 and tm.transform_pass > 0
