"""Lazy SPCA fit+transform throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c3|c2|c1|c4|c5] [--gemm tcgen05|simt] [--no-e2e] [--no-cpu]

The bench line is BASELINE configs[2] ("c3", the north-star workload: X fp32
4.6M x 4096, l = 220, q = 1) unless --config says otherwise.

A step is one Lazy SPCA fit (Omega regeneration, sketch U = X Omega, the power
step Z = X^T U, Z <- orth(Z), U = X Z, F = U^T X, the l x l step) plus the
transform Y = X V over this rank's resident rows, through one
lpca_fit_transform call.

Multi-GPU: --gpus N > 1 re-launches this script under torch.distributed.run
(one process per GPU) unless it already runs under it. The global row count is
fixed and row-sharded (strong scaling: rank r holds rows
[r * ceil(m / N), ...)); each rank generates its own shard on its GPU, and the
F and Z exchanges are NCCL allreduces inside the library. Rank 0 prints one
JSON line; time is the max over ranks of the device-event time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# BASELINE.json configs. m is the GLOBAL row count (sharded over ranks).
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
    "c5": dict(m=8_000_000, n=2_048, r=500, rho=0.99, k=256, l=512, q=1, dtype="f64",
               name="configs[4]: X fp64 8,000,000x2,048, r=500, rho=0.99, k=256, l=512, q=1"),
}
# Not a BASELINE config: SURVEY 8(f1), sparse X shaped like the paper's malware
# data (98,450 mostly binary features at density 0.0244, very
# sparse Omega at the aggressive density log(k)/k, l = k), a 500k-row slice.
SPARSE = dict(m=500_000, n=98_450, x_density=0.0244, k=100, l=100,
              name="sparse X (SURVEY 8 f1): CSC 500,000x98,450 binary at density 0.0244, very sparse Omega "
                   "log(k)/k, k=l=100, q=0")
DEFAULT_CONFIG = "c3"
# bounded CPU samples (rows) for the reference's CPU path: ~10-30 s of work for
# cpu_baseline, a few seconds per step for --impl reference
CPU_ROWS = {"c1": 10_000, "c2": 40_000, "c3": 16_384, "c4": 4_096, "c5": 8_192}
REF_ROWS = {"c1": 10_000, "c2": 16_384, "c3": 6_144, "c4": 2_048, "c5": 4_096}

SEED_X, SEED_OMEGA = 1000, 7
METRIC = "Lazy SPCA fit+transform samples/sec"


def projection(cfg, lp):
    kind = lp.ProjectionKind.very_sparse if cfg.get("kind") == "very_sparse" else lp.ProjectionKind.gaussian
    return lp.ProjectionSpec(kind=kind, density=cfg.get("density", 1.0), seed=SEED_OMEGA)


def shard_rows(m: int, world: int, rank: int) -> tuple[int, int]:
    """(first row, row count) of rank's contiguous shard of m rows (strong scaling)."""
    per = -(-m // world)
    lo = min(m, rank * per)
    return lo, min(m, lo + per) - lo


def peaks() -> dict:
    """Roofline denominators: MEASURED_PEAKS.json (driver-written: HBM copy GB/s,
    dense bf16 TF/s burst and sustained), plus profiles/peaks_r02.json
    (tools/peaks.cu on a B200 of this pool: tcgen05 f16 / tf32, DMMA, DFMA)."""
    out = {"hbm_gbs": 6550.0, "bf16_tflops_sustained": 1408.4, "source": "fallback (B200_PROFILING.md)"}
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        out.update(hbm_gbs=float(d["hbm_gbs"]),
                   bf16_tflops_sustained=float(d.get("bf16_tflops_sustained", d.get("bf16_tflops"))),
                   source="MEASURED_PEAKS.json")
    q = ROOT / "profiles" / "peaks_r02.json"
    if q.exists():
        d = json.loads(q.read_text())
        out["dmma_f64_tflops"] = float(d["dmma_f64_tflops"])
        out["dfma_f64_tflops"] = float(d["dfma_f64_tflops"])
        out["f16_tcgen05_tflops_microbench"] = float(d["f16_tcgen05_tflops"])
        out["peaks_file"] = "profiles/peaks_r02.json"
    else:
        out["dmma_f64_tflops"] = 37.0  # datasheet stand-in until tools/peaks.py has run
    return out


def cpu_model() -> str:
    """Model name plus family/model/stepping (a virtualised host often reports a
    generic name: family 6 model 143 is Sapphire Rapids, 207 Emerald Rapids),
    the logical CPUs online and whether AVX-512 / AMX are exposed."""
    info = {}
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if ":" in line:
                k, v = (t.strip() for t in line.split(":", 1))
                info.setdefault(k, v)
    except OSError:
        return "unknown"
    flags = set(info.get("flags", "").split())
    isa = "+".join(f for f in ("avx512f", "amx_tile") if f in flags) or "no avx512"
    return (f"{info.get('model name', 'unknown')} (family {info.get('cpu family', '?')} model "
            f"{info.get('model', '?')} stepping {info.get('stepping', '?')}, {os.cpu_count()} logical CPUs, {isa})")


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML during the timed region."""

    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
             0x100: "display_clock_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.power = [], set(), []
        self.max_mhz = self.power_limit_w = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            try:
                self.power_limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1000.0
            except Exception:
                pass
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                try:
                    self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                except Exception:
                    pass
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
        out = {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
               "reasons": sorted(self.reasons)}
        if self.power:  # board power: at the enforced limit the passes are energy-bound
            out["power_w"] = round(statistics.median(self.power), 1)
            out["power_limit_w"] = self.power_limit_w
        return out


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def relaunch_if_needed(args) -> int | None:
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run
    with N processes and return its exit code. Under torchrun, --gpus must match
    WORLD_SIZE."""
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is not None:
        if int(world_env) != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}")
        return None
    if args.gpus <= 1:
        return None
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the comm_nranks lines stay visible in the log
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.run(cmd, env=env).returncode


def stub_worker(args, cfg):
    """Launcher check without a GPU (tests/test_bench_cpu.py): every rank joins a
    gloo group and reports its shard; rank 0 prints the gathered list."""
    import torch.distributed as dist
    rank, world, _ = _dist()
    dist.init_process_group("gloo")
    m = args.rows or cfg["m"]
    row0, rows = shard_rows(m, world, rank)
    got = [None] * world
    dist.all_gather_object(got, {"rank": rank, "world": world, "row0": row0, "rows": rows})
    if rank == 0:
        print(json.dumps({"stub": True, "n_gpus": args.gpus, "global_rows": m, "shards": got}), flush=True)
    dist.destroy_process_group()


# ---- the reference's CPU path ---------------------------------------------------
def cpu_reference(cfg: dict, sample_rows: int, threads: int, steps: int = 1, warmup: int = 0):
    """The reference's own CPU implementation (oracle/_ref: proj/core compiled
    from /root/reference unmodified, with its default -march=native on hosts of
    the build's ISA) on a bounded row sample of the same workload. q = 0 runs
    reduce(lazy_spca) + apply_map; q >= 1 (no reference reducer: SPEC.md:371)
    composes the reference's kernels build_sketch / gemm_t / householder_qr /
    spmm / truncated_svd_via_gram (oracle/ref_capi.cpp). Returns
    (samples/s, kind, cores, description, seconds per step)."""
    import numpy as np
    from oracle import lazypca_oracle as O
    from oracle import refbind as R
    R.use_native(True)
    dt = np.float32 if cfg["dtype"] == "f32" else np.float64
    x = O.synth_lowrank(0, sample_rows, cfg["n"], cfg["r"], cfg["rho"], 0.01, SEED_X, dtype=dt, exact_log=False)
    R.set_threads(threads)
    kind = 1 if cfg.get("kind") == "very_sparse" else 0
    times = []
    for i in range(warmup + steps):
        if cfg["q"] > 0:
            _, _, _, secs = R.lazy_power_fit_transform(x, cfg["k"], cfg["l"], SEED_OMEGA, cfg["q"], kind=kind,
                                                       density=cfg.get("density", 1.0))
        else:
            _, _, _, secs = R.fit_transform(2, x, cfg["k"], cfg["l"], SEED_OMEGA, kind=kind,
                                            density=cfg.get("density", 1.0), want_y=True)
        if i >= warmup:
            times.append(secs)
    per = sum(times) / len(times)
    how = ("reduce(lazy_spca) + apply_map" if cfg["q"] == 0 else
           f"Lazy SPCA with q={cfg['q']} composed from the reference's build_sketch / gemm_t / householder_qr / "
           "spmm / truncated_svd_via_gram + spmm(X, V)")
    desc = (f"{sample_rows} rows x {cfg['n']} of the same generator (dense stored as the reference's CSC, "
            f"conversion untimed); {how}; {threads} threads on {cpu_model()}; reference built "
            f"{R.build_flags()}; {len(times)} timed reps")
    return sample_rows / per, "reference", threads, desc, per


def run_reference(args, cfg):
    rank, world, _ = _dist()
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    rows = int(args.ref_rows or REF_ROWS[args.config])
    value, kind, cores, desc, per = cpu_reference(cfg, rows, threads, steps=args.steps, warmup=args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (BASELINE low-rank generator, seeded)",
        "config": {"workload": cfg["name"], "sample_rows": rows, "method": "lazy_spca"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": kind, "sample": desc},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- roofline ---------------------------------------------------------------------
def pass_roof(rows, n, w, esz, t, pk, extra_bytes=0):
    """One X pass: algorithmic bytes (X once + operand/output planes) over HBM,
    algorithmic flops 2 rows n w at the dtype's peak (fp32 data: three fp16
    products per fp32-faithful one, so bf16_sustained / 3; fp64: DMMA)."""
    byts = rows * n * esz + extra_bytes
    flops = 2.0 * rows * n * w
    p_flops = (pk["bf16_tflops_sustained"] / 3.0 if esz == 4 else pk["dmma_f64_tflops"]) * 1e12
    t_hbm = byts / (pk["hbm_gbs"] * 1e9)
    t_mma = flops / p_flops
    return {"ms": t * 1e3, "bytes": byts, "flops": flops, "t_hbm_ms": t_hbm * 1e3, "t_mma_ms": t_mma * 1e3,
            "bound": "hbm" if t_hbm >= t_mma else "tensor",
            "frac": (max(t_hbm, t_mma) / t) if t > 0 else None}


def roofline(cfg, rows, esz, tm, steps, pk, config):
    n, k, l, q = cfg["n"], cfg["k"], cfg["l"], cfg["q"]
    npad = (l + 15) // 16 * 16
    up = 4 * npad * rows if esz == 4 else rows * l * 8          # U^T fp16 hi/lo planes (or U fp64)
    # configs[3] on fp32 (n > 8192): the sketch is the row gather, an HBM-bound
    # read of X (about n l density adds per row, no tensor work); U is written
    # in fp32 and its fp16 planes made from it
    gather = cfg.get("kind") == "very_sparse" and esz == 4 and n > 8192
    sketch = (pass_roof(rows, n, 0, esz, tm.sketch_pass / steps, pk, 4 * npad * rows * 3) if gather else
              pass_roof(rows, n, l, esz, tm.sketch_pass / steps, pk, up + 4 * npad * n))
    passes = {
        "sketch": sketch,
        "f": pass_roof(rows, n, l, esz, tm.f_pass / steps, pk, up),
        "transform": pass_roof(rows, n, k, esz, tm.transform_pass / steps, pk, rows * k * esz),
    }
    if q > 0:
        pp = pass_roof(rows, n, l, esz, tm.power_pass / steps / (2 * q), pk, up)
        passes["power (per pass, 2 per step)"] = pp
    tot_t = sum(p["ms"] * (2 * q if "power" in nm else 1) for nm, p in passes.items()) / 1e3
    tot_roof = sum(max(p["t_hbm_ms"], p["t_mma_ms"]) * (2 * q if "power" in nm else 1)
                   for nm, p in passes.items()) / 1e3
    sk = passes["sketch"]
    bound = sk["bound"]
    if bound == "tensor":
        achieved, peak, unit = sk["flops"] / (sk["ms"] * 1e-3) / 1e12, sk["flops"] / (sk["t_mma_ms"] * 1e-3) / 1e12, "TFLOP/s"
    else:
        achieved, peak, unit = sk["bytes"] / (sk["ms"] * 1e-3) / 1e9, pk["hbm_gbs"], "GB/s"
    kern = ("sparse_sketch_rows_kernel (row gather, bank-conflict-free schedule)" if gather else
            "tc2_kernel<XW, fp16> (2-SM tcgen05, 3-term fp16 split)" if esz == 4
            else "xw_f64_fast_kernel (DMMA m8n8k4)")
    return {
        "bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
        "traffic": _traffic(config),
        "kernel": f"sketch U = X Omega, {kern}",
        "peak_note": ("very sparse Omega: the gather's bytes (X once, U and its planes) against HBM"
                      if gather else
                      "fp32 data: fp32-equivalent TFLOP/s (2 m n l) against bf16_tflops_sustained / 3 "
                      "(every fp32 product is three fp16 products)" if esz == 4 else
                      "fp64 data: TFLOP/s against the measured DMMA rate") + f"; peaks from {pk['source']}",
        "x_passes_frac": tot_roof / tot_t if tot_t > 0 else None,
        "x_passes_ms": tot_t * 1e3,
        "passes": passes,
        "peaks": pk,
    }


def _traffic(config):
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(config)
        except Exception:
            return None
    return None


# ---- our arm --------------------------------------------------------------------
def run_ours(args, cfg):
    import torch
    import paper_1709_07175_b200 as lp

    rank, world, local = _dist()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # comm_nranks lines stay visible in the log
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

    m_global = args.rows or cfg["m"]
    row0, m = shard_rows(m_global, world, rank)
    n, k, l = cfg["n"], cfg["k"], cfg["l"]
    tdt = torch.float32 if cfg["dtype"] == "f32" else torch.float64
    esz = 4 if cfg["dtype"] == "f32" else 8
    x = torch.empty((m, n), dtype=tdt, device="cuda")
    lp.synth_lowrank(x, row0, cfg["r"], cfg["rho"], 0.01, SEED_X, ctx=ctx)
    y = torch.empty((m, k), dtype=tdt, device="cuda")
    conf = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=k, l=l,
                            projection=projection(cfg, lp), power_iters=cfg["q"])
    torch.cuda.synchronize()

    def step(tm=None):
        # fit + transform of the resident shard in one library call
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
    value = m_global / (ms * 1e-3)
    pk = peaks()
    roof = roofline(cfg, m, esz, tm, args.steps, pk, args.config)
    roof["phases_ms"] = {"sketch": tm.sketch / args.steps * 1e3, "power": tm.power / args.steps * 1e3,
                         "f_form": tm.f_form / args.steps * 1e3, "svd": tm.svd / args.steps * 1e3,
                         "transform": tm.transform / args.steps * 1e3}

    e2e = None
    if not args.no_e2e:
        xh = _pinned_copy(x, k, torch)
        # the C-ABI call stages X on the device itself: release the resident
        # shard first (configs[3]: two 131 GB copies do not fit in HBM)
        del x, y, step
        torch.cuda.empty_cache()
        e2e = xh if isinstance(xh, dict) else _e2e(args, cfg, ctx, xh, conf, m_global, dist, lp, torch)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, kind, cores, desc, _ = cpu_reference(cfg, int(args.cpu_rows or CPU_ROWS[args.config]),
                                                len(os.sched_getaffinity(0)))
        cpu = {"value": v, "unit": "samples/s", "cores": cores, "kind": kind, "sample": desc}
    if rank == 0:
        dname = {"f32": "f32 (3-term fp16 split on tcgen05, fp32 accumulate, fp64 l x l step)",
                 "f64": "f64 (DMMA)"}[cfg["dtype"]]
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": cfg["dtype"], "dtype_detail": dname,
            "data": "synthetic (BASELINE low-rank generator, seeded, each shard generated on its GPU)",
            "config": {"workload": cfg["name"], "global_rows": m_global, "rows_per_gpu": m,
                       "method": "lazy_spca",
                       "gemm_path": (args.gemm or "tcgen05") if cfg["dtype"] != "f64" else "dmma (fp64 X)",
                       "parallelism": f"dp{world} (row shards, NCCL allreduce of Z and F)",
                       "l2": "inputs larger than L2 (X is %.1f GB per GPU)" % (m * n * esz / 1e9)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    del mp
    ctx.close()
    if dist:
        dist.destroy_process_group()


def _pinned_copy(x, k, torch):
    """This rank's X in pinned host memory (and the pinned Y buffer), or an
    "unavailable" record."""
    m, n = x.shape
    try:
        xh = torch.empty((m, n), dtype=x.dtype, pin_memory=True)
        yh = torch.empty((m, k), dtype=x.dtype, pin_memory=True)
    except RuntimeError as e:
        return {"unavailable": f"pinned host buffers of {m * n * x.element_size() / 1e9:.1f} GB: {e}"[:200]}
    xh.copy_(x)
    return xh, yh


def _e2e(args, cfg, ctx, host, conf, m_global, dist, lp, torch):
    """Same metric through the public C ABI with host buffers: every step copies
    this rank's X from pinned host memory to the device and Y back
    (lpca_fit_transform with LPCA_HOST views)."""
    import ctypes as C
    from paper_1709_07175_b200 import _lib as L
    xh, yh = host
    x = xh
    m, n, k = x.shape[0], cfg["n"], cfg["k"]
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
    return {"value": m_global / sec, "unit": "samples/s", "h2d_bytes_per_step": m * n * esz,
            "d2h_bytes_per_step": m * k * esz, "ms_per_step": sec * 1e3, "steps": steps,
            "path": "lpca_fit_transform (C ABI), pinned host X in, host Y out (per rank)"}


# ---- sparse X (not a BASELINE config) -----------------------------------------------
def _sparse_csc(m: int, n: int, density: float, seed: int, torch):
    """Canonical CSC built on the GPU: column j holds Binomial(m, density)
    distinct uniformly drawn rows, values 1.0 (binary features)."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    counts = torch.binomial(torch.full((n,), float(m), device="cuda"),
                            torch.full((n,), density, device="cuda"), generator=g).long()
    cols = torch.repeat_interleave(torch.arange(n, device="cuda"), counts)
    rows = torch.randint(0, m, (cols.numel(),), device="cuda", generator=g)
    keys = torch.unique(cols * m + rows)  # sorted column-major, duplicates merged
    cols, rows = keys // m, keys % m
    del keys
    return cols, rows


def _csc_arrays(m, n, cols, rows, torch, pinned):
    """(col_ptr, row_idx, values) as host numpy arrays (row_idx / values pinned
    when asked: the uploads then run at the PCIe rate)."""
    col_ptr = torch.zeros(n + 1, dtype=torch.long, device="cuda")
    col_ptr[1:] = torch.cumsum(torch.bincount(cols, minlength=n), 0)
    vals = torch.ones(rows.numel(), dtype=torch.float64, device="cuda")

    def host(t):
        if not pinned:
            return t.cpu().numpy()
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h.numpy()
    return col_ptr.cpu().numpy(), host(rows), host(vals)


def _sparse_reference(cfg, sample_rows, threads, cols, rows, steps, warmup, torch):
    """The reference's reduce(lazy_spca) + apply_map on the first sample_rows
    rows of the same CSC (oracle/_ref, all host threads)."""
    from oracle import refbind as R
    R.use_native(True)
    R.set_threads(threads)
    keep = rows < sample_rows
    cp, ri, va = _csc_arrays(sample_rows, cfg["n"], cols[keep], rows[keep], torch, pinned=False)
    dens = math.log(cfg["k"]) / cfg["k"]
    secs = []
    for i in range(warmup + steps):
        _, _, _, sec = R.fit_transform_csc(2, sample_rows, cfg["n"], cp, ri, va, cfg["k"], cfg["l"], SEED_OMEGA,
                                           kind=1, density=dens, want_y=True)
        if i >= warmup:
            secs.append(sec)
    per = sum(secs) / len(secs)
    desc = (f"{sample_rows} rows x {cfg['n']} of the same CSC (nnz {int(keep.sum())}); reduce(lazy_spca) + "
            f"apply_map on the reference's SparseMatrix; {threads} threads on {cpu_model()}; reference built "
            f"{R.build_flags()}; {len(secs)} timed reps")
    return sample_rows / per, threads, desc, per


def run_sparse(args):
    """Sparse X on one GPU: every step is one lpca_fit_transform of a host CSC
    (pinned) into a host Y — the upload, the device checks and CSR build, the
    sketch (very sparse Omega as sign masks), F, the l x l step, the transform
    and the Y download, wall clock. value and e2e are the same number here (a
    CSC input always crosses PCIe); the phase split comes from ReducerTimings."""
    import torch
    import paper_1709_07175_b200 as lp
    cfg = dict(SPARSE)
    m = args.rows or cfg["m"]
    torch.cuda.set_device(0)
    cols, rows = _sparse_csc(m, cfg["n"], cfg["x_density"], 460, torch)
    threads = len(os.sched_getaffinity(0))
    if args.impl == "reference":
        sr = args.ref_rows or 20_000
        v, cores, desc, per = _sparse_reference(cfg, sr, threads, cols, rows, args.steps, args.warmup, torch)
        print(json.dumps({"impl": "reference", "metric": METRIC + " (sparse X)", "value": v, "unit": "samples/s",
                          "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic (binary CSC, seeded)",
                          "config": {"workload": cfg["name"], "sample_rows": sr, "method": "lazy_spca"},
                          "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "reference",
                                           "sample": desc},
                          "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return
    cp, ri, va = _csc_arrays(m, cfg["n"], cols, rows, torch, pinned=True)
    x = lp.SparseMatrix(m, cfg["n"], cp, ri, va)
    ctx = lp.Context(0)
    conf = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=cfg["k"], l=cfg["l"],
                            projection=lp.ProjectionSpec(kind=lp.ProjectionKind.very_sparse,
                                                         density=math.log(cfg["k"]) / cfg["k"], seed=SEED_OMEGA))
    for _ in range(args.warmup):
        lp.fit_transform(x, conf, ctx=ctx)
    launches0 = ctx.launch_count()
    tm = lp.ReducerTimings()
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            lp.fit_transform(x, conf, ctx=ctx, timings=tm)
        torch.cuda.synchronize()
        sec = (time.perf_counter() - t0) / args.steps
    nnz = int(ri.size)
    cpu = None
    if not args.no_cpu:
        v, cores, desc, _ = _sparse_reference(cfg, int(args.cpu_rows or 20_000), threads, cols, rows, 1, 1, torch)
        cpu = {"value": v, "unit": "samples/s", "cores": cores, "kind": "reference", "sample": desc}
    h2d = nnz * 16 + (cfg["n"] + 1) * 8
    print(json.dumps({
        "metric": METRIC + " (sparse X)", "value": m / sec, "unit": "samples/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "dtype_detail": "f64 values, CSR/CSC gathers in the reference's summation order",
        "data": "synthetic (binary CSC at the paper's density, seeded)",
        "config": {"workload": cfg["name"], "rows": m, "nnz": nnz, "method": "lazy_spca",
                   "parallelism": "dp1", "l2": "inputs larger than L2 (CSC %.1f GB)" % (h2d / 1e9)},
        "phases_ms": {p: getattr(tm, p) / args.steps * 1e3 for p in ("sketch", "f_form", "svd", "transform")},
        "roofline": None, "cpu_baseline": cpu,
        "e2e": {"value": m / sec, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": m * cfg["k"] * 8, "ms_per_step": sec * 1e3,
                "path": "lpca_fit_transform (C ABI) on a pinned host CSC, host Y out"},
        "gpu_launches": ctx.launch_count() - launches0, "clocks": clk.summary(),
    }), flush=True)
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS) + ["sparse"])
    ap.add_argument("--rows", type=int, default=0, help="override the global row count (experiments only)")
    ap.add_argument("--gemm", default=None, choices=["tcgen05", "simt"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-rows", type=int, default=0)
    ap.add_argument("--ref-rows", type=int, default=0)
    ap.add_argument("--stub-worker", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.config == "sparse":
        return run_sparse(args)
    cfg = CONFIGS[args.config]
    rc = relaunch_if_needed(args)
    if rc is not None:
        sys.exit(rc)
    if args.stub_worker:
        stub_worker(args, cfg)
    elif args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
