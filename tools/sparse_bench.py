"""Sparse-X timing: Lazy SPCA fit + transform of a CSC X
shaped like the paper's malware data (98,450 mostly binary
features, mean density 0.0244, very sparse Omega at the aggressive density
log(k)/k, l = k), on this library's sparse path (csrc/sparse.cu: CSR/CSC
gathers in the reference's order) against the reference compiled from its
sources (oracle/_ref, all host threads) on a row sample of the same data.

The data are synthetic (the dataset is private): column j holds
Binomial(m, 0.0244) distinct rows drawn uniformly, values 1.0 (binary
features), built on the GPU and handed to both sides as the reference's
canonical CSC, ours in pinned host memory. Our timing is the whole library
call from host CSC to host Y (upload, the device checks and CSR build, the
passes, the Y download), wall clock, mean of --steps after one warm-up; the
phase split comes from ReducerTimings.

usage: python tools/sparse_bench.py [--rows 500000] [--k 100] [--ref-rows 20000]"""
import argparse
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1709_07175_b200 as lp  # noqa: E402

N_FEATURES, DENSITY = 98_450, 0.0244


def gen_csc(m: int, n: int, density: float, seed: int):
    """Canonical CSC (sorted, distinct rows per column) built on the GPU."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    counts = torch.binomial(torch.full((n,), float(m), device="cuda"),
                            torch.full((n,), density, device="cuda"), generator=g).long()
    cols = torch.repeat_interleave(torch.arange(n, device="cuda"), counts)
    rows = torch.randint(0, m, (cols.numel(),), device="cuda", generator=g)
    keys = torch.unique(cols * m + rows)  # sorted: column-major, rows ascending, duplicates merged
    cols, rows = keys // m, keys % m
    del keys
    col_ptr = torch.zeros(n + 1, dtype=torch.long, device="cuda")
    col_ptr[1:] = torch.cumsum(torch.bincount(cols, minlength=n), 0)
    return col_ptr, rows, cols


def _pinned(t: torch.Tensor) -> np.ndarray:
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


def to_sparse(m, n, col_ptr, rows):
    """The CSC arrays in pinned host memory (as a caller feeding the GPU would
    hold them), so the library's uploads run at the PCIe rate."""
    vals = torch.ones(rows.numel(), dtype=torch.float64, device="cuda")
    return lp.SparseMatrix(m, n, col_ptr.cpu().numpy(), _pinned(rows), _pinned(vals))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=500_000)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--ref-rows", type=int, default=20_000)
    ap.add_argument("--seed", type=int, default=460)
    args = ap.parse_args()
    m, n, k = args.rows, N_FEATURES, args.k
    dens_omega = math.log(k) / k  # aggressive
    col_ptr, rows, cols = gen_csc(m, n, DENSITY, args.seed)
    nnz = rows.numel()
    x = to_sparse(m, n, col_ptr, rows)
    ctx = lp.Context(0)
    cfg = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=k, l=k,
                           projection=lp.ProjectionSpec(kind=lp.ProjectionKind.very_sparse, density=dens_omega,
                                                        seed=7))
    lp.fit_transform(x, cfg, ctx=ctx)  # warm-up
    launches0 = ctx.launch_count()
    tm = lp.ReducerTimings()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        mp, y = lp.fit_transform(x, cfg, ctx=ctx, timings=tm)
    ours = (time.perf_counter() - t0) / args.steps
    launches = (ctx.launch_count() - launches0) // args.steps
    phases = {p: getattr(tm, p) / args.steps * 1e3 for p in ("sketch", "power", "f_form", "svd", "transform")}

    # the reference on the first ref-rows rows (the same columns' entries with row < ref_rows)
    ref_line = None
    try:
        from oracle import refbind as R
        if not R.available():
            raise RuntimeError("oracle/_ref not built")
        R.use_native(True)
        threads = len(os.sched_getaffinity(0))
        R.set_threads(threads)
        keep = rows < args.ref_rows
        rs, cs = rows[keep], cols[keep]
        cp = torch.zeros(n + 1, dtype=torch.long, device="cuda")
        cp[1:] = torch.cumsum(torch.bincount(cs, minlength=n), 0)
        secs = []
        for _ in range(2):
            _, _, sig_ref, s = R.fit_transform_csc(2, args.ref_rows, n, cp.cpu().numpy(), rs.cpu().numpy(),
                                                   np.ones(rs.numel()), k, k, 7, kind=1, density=dens_omega,
                                                   want_y=True)
            secs.append(s)
        # parity on the sample: our sparse path on the same CSC
        sample = lp.SparseMatrix(args.ref_rows, n, cp.cpu().numpy(), rs.cpu().numpy(), np.ones(rs.numel()))
        mine, _ = lp.fit_transform(sample, cfg, ctx=ctx)
        sig_err = float(np.max(np.abs(mine.singular_values - sig_ref) / sig_ref))
        ref_line = {"value": args.ref_rows / secs[-1], "unit": "samples/s", "cores": threads,
                    "sigma_rel_err_vs_ours_on_sample": sig_err,
                    "sample": f"{args.ref_rows} rows x {n}, nnz {int(rs.numel())}, reduce(lazy_spca) + apply_map "
                              f"on the reference's CSC, reference built {R.build_flags()}"}
    except Exception as e:  # noqa: BLE001 - reported, not fatal
        ref_line = {"unavailable": str(e)}

    bytes_x = nnz * (8 + 8)  # CSC as handed over: int64 row index + fp64 value
    print(json.dumps({
        "metric": "Lazy SPCA fit+transform samples/sec, sparse X (host CSC in, host Y out)",
        "value": m / ours, "unit": "samples/s", "seconds_per_call": ours,
        "config": {"rows": m, "features": n, "density": DENSITY, "nnz": int(nnz), "k": k, "l": k,
                   "omega": f"very sparse, density log(k)/k = {dens_omega:.4f}", "values": "1.0 (binary)",
                   "host_csc_gb": bytes_x / 1e9},
        "phases_ms": phases, "gpu_launches_per_call": launches,
        "cpu_reference": ref_line,
        "sigma_head": [float(s) for s in mp.singular_values[:3]],
    }))


if __name__ == "__main__":
    main()
