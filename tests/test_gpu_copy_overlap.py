"""GPU: a host X crosses PCIe in row chunks while the sketch runs on the chunks
already landed, and Y comes back chunk by chunk behind the transform
(csrc/lpca.cu stage_x_arriving, xw_pass, transform_dev). The results must be
bit-identical to one whole copy (LPCA_H2D_CHUNKS=0) and to the device-resident
call, for every method, dtype and a ragged last chunk."""
import numpy as np
import pytest
import torch

import paper_1709_07175_b200 as lp

pytestmark = pytest.mark.gpu

M = lp.ReducerMethod


def _x(m, n, dtype):
    x = torch.empty((m, n), dtype=dtype, device="cuda")
    lp.synth_lowrank(x, 0, 60, 0.95, 0.01, 1000)
    return x


def _run(x_host, cfg, ctx, y_dtype):
    mp, y = lp.fit_transform(x_host, cfg, y_dtype=y_dtype, ctx=ctx)
    return mp.singular_values if cfg.method != M.rp else np.zeros(1), mp.v, y


@pytest.mark.parametrize("dtype,method,q,n,sparse", [
    (torch.float32, M.lazy_spca, 0, 1000, False),
    (torch.float32, M.lazy_spca, 1, 1000, False),
    (torch.float32, M.spca, 0, 1000, False),
    (torch.float32, M.rp, 0, 1000, False),
    (torch.float64, M.lazy_spca, 0, 1000, False),
    (torch.float32, M.lazy_spca, 1, 9000, True),   # very sparse Omega, long rows: the row gather per chunk
])
def test_chunked_copies_bit_identical(ctx, monkeypatch, dtype, method, q, n, sparse):
    m, k, l = 20_011, 12, 12 if method == M.rp else 30   # ragged last chunk
    x = _x(m, n, dtype)
    xh = x.cpu().numpy()
    spec = (lp.ProjectionSpec(kind=lp.ProjectionKind.very_sparse, density=1 / 64, seed=5) if sparse
            else lp.ProjectionSpec(seed=5))
    cfg = lp.ReducerConfig(method=method, k=k, l=l, power_iters=q, projection=spec)
    y_dt = np.float32 if dtype == torch.float32 else np.float64
    monkeypatch.setenv("LPCA_H2D_CHUNK_MB", "1")   # 512-row chunks: ~40 of them (n = 1000)
    chunked = _run(xh, cfg, ctx, y_dt)
    monkeypatch.setenv("LPCA_H2D_CHUNKS", "0")
    whole = _run(xh, cfg, ctx, y_dt)
    monkeypatch.delenv("LPCA_H2D_CHUNKS")
    for a, b in zip(chunked, whole):
        assert np.array_equal(a, b)
    # the device-resident call (no copies at all) agrees bit for bit too
    out = torch.empty((m, k), dtype=dtype, device="cuda")
    mp, _ = lp.fit_transform(x, cfg, ctx=ctx, out=out)
    assert np.array_equal(mp.v, chunked[1])
    assert np.array_equal(out.cpu().numpy(), chunked[2])


def test_chunked_fit_only_and_timings(ctx, monkeypatch):
    m, n = 30_000, 512
    x = _x(m, n, torch.float32)
    xh = x.cpu().numpy()
    cfg = lp.ReducerConfig(method=M.lazy_spca, k=10, l=20, projection=lp.ProjectionSpec(seed=3))
    monkeypatch.setenv("LPCA_H2D_CHUNK_MB", "2")
    t = lp.ReducerTimings()
    a = lp.reduce(xh, cfg, timings=t, ctx=ctx)
    assert t.h2d > 0.0 and t.sketch_pass > 0.0
    # RP reads no X: its timings still wait for the upload's last chunk
    t_rp = lp.ReducerTimings()
    lp.reduce(xh, lp.ReducerConfig(method=M.rp, k=10, l=10), timings=t_rp, ctx=ctx)
    assert t_rp.h2d > 0.0
    monkeypatch.setenv("LPCA_H2D_CHUNKS", "0")
    b = lp.reduce(xh, cfg, ctx=ctx)
    assert np.array_equal(a.v, b.v) and np.array_equal(a.singular_values, b.singular_values)


def test_chunked_copy_error_leaves_context_usable(ctx, monkeypatch):
    """An error raised after the copies were queued (k > l) returns with no copy
    still reading the caller's buffer, and the next call works."""
    xh = _x(20_000, 600, torch.float32).cpu().numpy()
    monkeypatch.setenv("LPCA_H2D_CHUNK_MB", "1")
    with pytest.raises(lp.InvalidArgumentError):
        lp.reduce(xh, lp.ReducerConfig(method=M.lazy_spca, k=40, l=20), ctx=ctx)
    del xh
    xh2 = _x(20_000, 600, torch.float32).cpu().numpy()
    mp = lp.reduce(xh2, lp.ReducerConfig(method=M.lazy_spca, k=10, l=20), ctx=ctx)
    assert np.all(np.isfinite(mp.singular_values))
