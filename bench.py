"""Lazy SPCA fit+transform throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c3|c1] [--gemm tcgen05|simt] [--no-e2e] [--no-cpu]

A step is one Lazy SPCA fit (Omega regeneration, sketch U = X Omega, F = U^T X,
the l x l step) plus the transform Y = X V over one rank's resident rows.
N > 1: launched by torch.distributed.run, one process per GPU; each rank holds
its own row shard (weak scaling) and the F exchange is one NCCL allreduce
inside the library. Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# BASELINE.json configs; the bench line is configs[1] ("c2") unless --config.
CONFIGS = {
    "c1": dict(m=10_000, n=1_000, r=50, rho=0.9, k=10, l=20, q=0, dtype="f64",
               name="configs[0]: X fp64 10,000x1,000, r=50, rho=0.9, k=10, l=20, q=0"),
    "c2": dict(m=1_000_000, n=4_096, r=200, rho=0.97, k=100, l=110, q=0, dtype="f32",
               name="configs[1]: X fp32 1,000,000x4,096, r=200, rho=0.97, k=100, l=110, q=0"),
    "c3": dict(m=4_600_000, n=4_096, r=300, rho=0.98, k=200, l=220, q=1, dtype="f32",
               name="configs[2]: X fp32 4,600,000x4,096, r=300, rho=0.98, k=200, l=220, q=1"),
    "c4": dict(m=2_000_000, n=16_384, r=400, rho=0.98, k=256, l=300, q=2, dtype="f32",
               kind="very_sparse", density=1.0 / 128,
               name="configs[3]: X fp32 2,000,000x16,384, r=400, rho=0.98, very sparse Omega "
                    "(density 1/sqrt(n)), k=256, l=300, q=2"),
    "c5": dict(m=1_000_000, n=2_048, r=500, rho=0.99, k=256, l=512, q=1, dtype="f64",
               name="configs[4] per GPU: X fp64 1,000,000x2,048 (8e6 rows over 8 GPUs), r=500, "
                    "rho=0.99, k=256, l=512, q=1"),
}


def projection(cfg, lp):
    kind = lp.ProjectionKind.very_sparse if cfg.get("kind") == "very_sparse" else lp.ProjectionKind.gaussian
    return lp.ProjectionSpec(kind=kind, density=cfg.get("density", 1.0), seed=SEED_OMEGA)
SEED_X, SEED_OMEGA = 1000, 7
METRIC = "Lazy SPCA fit+transform samples/sec"
FP64_TFLOPS = 37.0  # B200 datasheet dense fp64 (tensor) rate; the fp64 configs' roofline peak


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML during the timed region."""

    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
             0x100: "display_clock_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.NAMES.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons)}


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_reference(cfg: dict, sample_rows: int, threads: int, steps: int = 1, warmup: int = 0):
    """The reference's own CPU implementation (oracle/_ref: proj/core compiled
    unmodified) on a bounded row sample of the same workload. Returns
    (samples/s, kind, cores, sample description)."""
    import numpy as np
    from oracle import lazypca_oracle as O
    from oracle import refbind as R
    dt = np.float32 if cfg["dtype"] == "f32" else np.float64
    x = O.synth_lowrank(0, sample_rows, cfg["n"], cfg["r"], cfg["rho"], 0.01, SEED_X, dtype=dt,
                        exact_log=False)
    R.set_threads(threads)
    if cfg["q"] > 0:
        kind = "port"  # q >= 1 has no reference implementation
        times = []
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            v, s, _ = O.reduce_lazy_spca(x.astype(np.float64), cfg["k"], cfg["l"], SEED_OMEGA,
                                         kind=cfg.get("kind", "gaussian"), density=cfg.get("density", 1.0),
                                         power_iters=cfg["q"])
            O.apply_map(x, v)
            if i >= warmup:
                times.append(time.perf_counter() - t0)
    else:
        kind = "reference"
        times = []
        for i in range(warmup + steps):
            _, _, _, secs = R.fit_transform(2, x, cfg["k"], cfg["l"], SEED_OMEGA,
                                            kind=1 if cfg.get("kind") == "very_sparse" else 0,
                                            density=cfg.get("density", 1.0), want_y=True)
            if i >= warmup:
                times.append(secs)
    per = sum(times) / len(times)
    desc = (f"{sample_rows} rows x {cfg['n']} of the same generator, dense stored as the reference's "
            f"CSC; reduce(lazy_spca)+apply_map, {threads} threads, {len(times)} timed reps")
    return sample_rows / per, kind, threads, desc, per


def run_reference(args, cfg):
    rank, world, _ = _dist()
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    rows = int(args.ref_rows)
    value, kind, cores, desc, per = cpu_reference(cfg, rows, threads, steps=args.steps,
                                                  warmup=args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (BASELINE low-rank generator, seeded)",
        "config": {"workload": cfg["name"], "sample_rows": rows, "method": "lazy_spca"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": kind,
                         "sample": desc},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, cfg):
    import torch
    import paper_1709_07175_b200 as lp

    rank, world, local = _dist()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [lp.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = lp.Context(local, rank, world, obj[0])
    else:
        dist = None
        ctx = lp.Context(local)
    if args.gemm:
        ctx.set_gemm_path(args.gemm)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)

    m, n, k, l = cfg["m"], cfg["n"], cfg["k"], cfg["l"]
    tdt = torch.float32 if cfg["dtype"] == "f32" else torch.float64
    esz = 4 if cfg["dtype"] == "f32" else 8
    x = torch.empty((m, n), dtype=tdt, device="cuda")
    lp.synth_lowrank(x, rank * m, cfg["r"], cfg["rho"], 0.01, SEED_X, ctx=ctx)
    y = torch.empty((m, k), dtype=tdt, device="cuda")
    conf = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=k, l=l,
                            projection=projection(cfg, lp), power_iters=cfg["q"])
    torch.cuda.synchronize()

    def step(tm=None):
        # fit + transform of the resident X in one library call (lpca_fit_transform:
        # the same kernels as reduce_lazy_spca + apply_map, the transform queued
        # behind the fit's spectral step instead of after its host checks)
        mp, _ = lp.fit_transform(x, conf, timings=tm, ctx=ctx, out=y)
        return mp

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches0 = ctx.launch_count()
    tm = lp.ReducerTimings()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            mp = step(tm)
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = ctx.launch_count() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * m / (ms * 1e-3)

    # dominant kernel: the sketch pass U = X Omega, timed alone by the library's
    # device events around its launch on this stream (lpca_timings.sketch_pass)
    sketch_s = tm.sketch_pass / args.steps
    f_s = tm.f_pass / args.steps
    tr_s = tm.transform_pass / args.steps
    x_bytes = m * n * esz
    npad = (l + 15) // 16 * 16
    if esz == 4:  # fp16 hi/lo planes: W^T in, U^T out (+ its 256-row block scales)
        sk_bytes = x_bytes + 4 * npad * n + 4 * npad * m + 4 * npad * ((m + 255) // 256)
    else:
        sk_bytes = x_bytes + n * l * 8 + m * l * 8
    hbm, peak_kind = _peaks()
    achieved = sk_bytes / sketch_s / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": _traffic(args.config), "kernel": "sketch U = X Omega (tc2_kernel<XW, fp16>)",
            "peak_source": peak_kind, "algorithmic_bytes": sk_bytes, "kernel_ms": sketch_s * 1e3}
    if esz == 8:
        # fp64 X runs the DMMA kernel (xw_f64_fast_kernel), bound by the fp64
        # tensor-core rate, not HBM: 2 m n l flops per pass. No measured fp64
        # peak exists in MEASURED_PEAKS.json; the datasheet figure stands in.
        tf = 2.0 * m * n * l / sketch_s / 1e12
        roof.update({"bound": "tensor", "achieved": tf, "peak": FP64_TFLOPS, "unit": "TFLOP/s",
                     "frac": tf / FP64_TFLOPS, "traffic": None,
                     "kernel": ("sketch U = X Omega (xw_f64_fast_kernel, DMMA m8n8k4)" if l > 64 and n > 64
                                else "sketch U = X Omega (xw_simt_kernel, DFMA)"),
                     "peak_source": "B200 datasheet fp64 tensor 37 TFLOP/s (not measured)",
                     "hbm_GBps": achieved, "algorithmic_flops": 2.0 * m * n * l})
    roof.update({
            "phases_ms": {"sketch": tm.sketch / args.steps * 1e3, "power": tm.power / args.steps * 1e3,
                          "f_form": tm.f_form / args.steps * 1e3, "svd": tm.svd / args.steps * 1e3,
                          "transform": tm.transform / args.steps * 1e3},
            "pass_ms": {"sketch": sketch_s * 1e3, "f": f_s * 1e3, "transform": tr_s * 1e3},
            "f_pass_GBps": (x_bytes + 4 * npad * m) / f_s / 1e9 if f_s > 0 else None,
            "transform_pass_GBps": (x_bytes + m * k * esz) / tr_s / 1e9 if tr_s > 0 else None})

    e2e = None
    if not args.no_e2e:
        e2e = _e2e(args, cfg, ctx, x, conf, world, dist, lp, torch)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, kind, cores, desc, _ = cpu_reference(cfg, int(args.cpu_rows), len(os.sched_getaffinity(0)))
        cpu = {"value": v, "unit": "samples/s", "cores": cores, "kind": kind, "sample": desc}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": cfg["dtype"], "data": "synthetic (BASELINE low-rank generator, seeded, generated on device)",
            "config": {"workload": cfg["name"], "rows_per_gpu": m, "global_rows": world * m,
                       "method": "lazy_spca", "gemm_path": (args.gemm or "tcgen05") if cfg["dtype"] != "f64" else "dmma (fp64 X)",
                       "parallelism": f"dp{world} (row shards, NCCL allreduce of F)",
                       "l2": "inputs larger than L2 (X is %.1f GB per GPU)" % (x_bytes / 1e9)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    del mp
    ctx.close()
    if dist:
        dist.destroy_process_group()


def _traffic(config):
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(config)
        except Exception:
            return None
    return None


def _e2e(args, cfg, ctx, x, conf, world, dist, lp, torch):
    """Same metric through the public C ABI with host buffers: every step copies
    X from pinned host memory to the device and Y back (lpca_fit_transform)."""
    import ctypes as C
    from paper_1709_07175_b200 import _lib as L
    m, n, k = cfg["m"], cfg["n"], cfg["k"]
    xh = torch.empty((m, n), dtype=x.dtype, pin_memory=True)
    xh.copy_(x)
    yh = torch.empty((m, k), dtype=x.dtype, pin_memory=True)
    vw = lp.api._View(xh)  # host row-major view
    cfgc = conf._c()
    dt = L.LPCA_F32 if x.dtype == torch.float32 else L.LPCA_F64
    steps = max(1, min(args.steps, args.e2e_steps))

    def one():
        h = C.c_void_p()
        t = L.Timings()
        lp.api._check(ctx.lib.lpca_fit_transform(ctx.h, C.byref(cfgc), C.byref(vw.view), C.byref(h),
                                                 C.c_void_p(yh.data_ptr()), dt, L.LPCA_ROW_MAJOR,
                                                 L.LPCA_HOST, 0, C.byref(t)))
        ctx.lib.lpca_map_destroy(h)

    for _ in range(max(1, args.warmup)):
        one()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    sec = (time.perf_counter() - t0) / steps
    if dist:
        t = torch.tensor([sec], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    esz = x.element_size()
    return {"value": world * m / sec, "unit": "samples/s", "h2d_bytes_per_step": m * n * esz,
            "d2h_bytes_per_step": m * k * esz, "ms_per_step": sec * 1e3, "steps": steps,
            "path": "lpca_fit_transform (C ABI), pinned host X in, host Y out"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--gemm", default=None, choices=["tcgen05", "simt"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-rows", type=int, default=40_000)
    ap.add_argument("--ref-rows", type=int, default=16_384)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
