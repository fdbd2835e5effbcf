"""Command line: `python -m paper_1709_07175_b200 {reduce,compare,bench} ...`.

The reference CLI's reduce / compare / bench (proj/tools/lazypca_cli.cpp:162-452)
over this library: the same options and defaults, the same JSON records
(timings; comparison_record_json, metrics.cpp:354-371), the same exit codes
(ParseError / InvalidArgument 2, RankDeficiency 3, Dimension 4, other 1,
lazypca_cli.cpp:618-635) and `--manifest` defaults for reduce / compare
(load_manifest / fill_from, lazypca_cli.cpp:47-69, 580-613), plus `--device N`
(the GPU to run on). gen-synthetic (the reference's sparse synthetic generator)
is out of scope.
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from . import api as lp


def _fmt(v: float) -> str:
    for prec in range(1, 18):  # format_double: the shortest %g form that round-trips
        s = "%.*g" % (prec, v)
        if float(s) == v:
            return s
    return "%.17g" % v


def _timings_json(t: lp.ReducerTimings) -> str:
    return ('{"sketch":%s,"qr":%s,"f_form":%s,"svd":%s,"total":%s}'
            % (_fmt(t.sketch), _fmt(t.qr), _fmt(t.f_form), _fmt(t.svd), _fmt(t.total)))


def _check_format(fmt: str) -> None:
    if fmt not in ("mm", "csv"):
        raise lp.InvalidArgumentError(f'format must be "mm" or "csv", got "{fmt}"')


def _load(path: str, fmt: str):
    _check_format(fmt)
    return lp.read_sparse_matrix_market(path) if fmt == "mm" else lp.read_dense_csv(path)


def _config(a) -> lp.ReducerConfig:
    kind = lp.projection_kind_from_string(a.projection)
    spec = lp.ProjectionSpec(kind=kind, seed=int(a.seed))
    if kind == lp.ProjectionKind.very_sparse:
        spec.density = lp.density_for(lp.DensityPolicy.parse(a.density_policy), a.l if a.l > 0 else a.k)
    return lp.ReducerConfig(method=lp.reducer_method_from_string(a.method), k=a.k, l=a.l, projection=spec,
                            block_rows=a.block_rows, streaming=bool(a.streaming or a.block_rows > 0))


def run_reduce(a, ctx) -> int:
    if not a.input:
        raise lp.InvalidArgumentError("reduce: no input given")
    if a.report != "json":
        raise lp.InvalidArgumentError("reduce: only the json report format exists")
    cfg = _config(a)
    t = lp.ReducerTimings()
    if cfg.streaming:
        _check_format(a.format)
        opener = lp.MatrixMarketRowBlockStream if a.format == "mm" else lp.CsvRowBlockStream
        if cfg.method == lp.ReducerMethod.rp:
            # the map is the scaled projection: only the column count is needed
            x = _load(a.input, a.format)
            mp = lp.reduce(x, lp.ReducerConfig(method=cfg.method, k=cfg.k, l=cfg.l, projection=cfg.projection),
                           timings=t, ctx=ctx)
        elif cfg.method == lp.ReducerMethod.spca:
            mp = lp.reduce_spca_streaming(opener(a.input, cfg.block_rows), cfg, timings=t, ctx=ctx)
        else:
            mp = lp.reduce_lazy_spca_streaming(opener(a.input, cfg.block_rows), cfg, timings=t, ctx=ctx)
        if a.out_reduced:  # block by block, like write_reduced_streaming
            st = opener(a.input, cfg.block_rows)
            with open(a.out_reduced, "w") as out:
                while (b := st.next()) is not None:
                    y = lp.apply_map(mp, b.block, ctx=ctx)
                    for row in y:
                        out.write(",".join(_fmt(float(v)) for v in row) + "\n")
    else:
        x = _load(a.input, a.format)
        mp = lp.reduce(x, cfg, timings=t, ctx=ctx)
        if a.out_reduced:
            lp.write_dense_csv(lp.apply_map(mp, x, ctx=ctx), a.out_reduced)
    if a.out_map:
        lp.save_map_file(mp, a.out_map)
    print(_timings_json(t))
    return 0


def _basis(mp) -> np.ndarray:
    # orthonormal basis of the map's column span (rp maps are not orthonormal)
    return np.linalg.qr(mp.v)[0] if mp.method == "rp" else mp.v


def _method_error(x, mp, cfg, ctx):
    rows, cols = (x.rows(), x.cols()) if isinstance(x, lp.SparseMatrix) else x.shape
    densify_limit = 300
    with_bound = cfg.l >= cfg.k + 2 and max(rows, cols) <= densify_limit
    if mp.method == "rp":
        return lp.row_space_reconstruction_error(x, _basis(mp), ctx=ctx)
    omega = lp.regenerate(cfg.projection, ctx=ctx)
    u = lp.build_sketch(x, omega, ctx=ctx).u
    route = lp.ResidualRoute.qr if mp.method == "spca" else lp.ResidualRoute.lazy
    return lp.reconstruction_error(x, u, route, cfg.k, cfg.l, with_bound, densify_limit, ctx=ctx)


def run_compare(a, ctx) -> int:
    ia, ib = a.input_a or a.input, a.input_b or a.input
    if not ia or not ib:
        raise lp.InvalidArgumentError("compare: no input given")
    xa = _load(ia, a.format)
    xb = xa if ib == ia else _load(ib, a.format)
    sa = (xa.rows(), xa.cols()) if isinstance(xa, lp.SparseMatrix) else xa.shape
    sb = (xb.rows(), xb.cols()) if isinstance(xb, lp.SparseMatrix) else xb.shape
    if sa != sb:
        raise lp.DimensionError(f"compare: inputs are {sa[0]}x{sa[1]} and {sb[0]}x{sb[1]}; dimensions must match")
    a.method = a.method_a
    ca = _config(a).resolved(sa[1])
    a.method = a.method_b
    cb = _config(a).resolved(sb[1])
    ma, mb = lp.reduce(xa, ca, ctx=ctx), lp.reduce(xb, cb, ctx=ctx)
    chordal = lp.chordal_distance(_basis(ma), _basis(mb), ctx=ctx)
    ea, eb = _method_error(xa, ma, ca, ctx), _method_error(xb, mb, cb, ctx)
    dp = lp.distance_preservation(xa, ma, mb, max_pairs=a.max_pairs, seed=a.seed, ctx=ctx)
    rec = {"method_a": ma.method, "method_b": mb.method, "k": ca.k, "l": ca.l, "seed": int(a.seed),
           "chordal": chordal, "spectral_error": ea.spectral_error, "frobenius_error": ea.frobenius_error,
           "bound": ea.bound, "max_contraction_violation": dp.max_contraction_violation,
           "max_map_discrepancy": dp.max_map_discrepancy, "spectral_error_b": eb.spectral_error,
           "frobenius_error_b": eb.frobenius_error}
    line = json.dumps(rec, separators=(",", ":"))
    print(line)
    if a.out_report:
        with open(a.out_report, "a") as out:
            out.write(line + "\n")
    if {ma.method, mb.method} != {"spca", "lazy_spca"}:
        return 0
    scale = 1.0 + max(ea.spectral_error, eb.spectral_error, ea.frobenius_error, eb.frobenius_error)
    ok = (rec["max_contraction_violation"] <= 1e-12
          and abs(ea.spectral_error - eb.spectral_error) <= 1e-9 * scale
          and abs(ea.frobenius_error - eb.frobenius_error) <= 1e-9 * scale)
    if rec["k"] == rec["l"]:
        ok = ok and chordal <= 1e-8 and rec["max_map_discrepancy"] <= 1e-9
    if not ok:
        print("compare: spca/lazy_spca agreement tolerances violated", file=sys.stderr)
    return 0 if ok else 1


def run_bench(a, ctx) -> int:
    ks = [int(v) for v in a.k_list.split(",") if v]
    if not ks:
        return 0
    if a.input:
        x = _load(a.input, a.format)
    else:
        rng = np.random.default_rng(a.seed)
        d = rng.standard_normal((a.m, a.n)) * (rng.uniform(0, 1, (a.m, a.n)) < a.density)
        x = lp.SparseMatrix.from_dense(d)
    out = open(a.out, "w") if a.out else sys.stdout
    out.write("method,k,l,seconds,rows_per_second\n")
    rows = x.rows() if isinstance(x, lp.SparseMatrix) else x.shape[0]
    for method in [m for m in a.methods.split(",") if m]:
        for k in ks:
            ns = argparse.Namespace(method=method, k=k, l=0, projection=a.projection, density_policy=a.density_policy,
                                    seed=a.seed, block_rows=a.block_rows, streaming=a.block_rows > 0)
            cfg = _config(ns)
            best = None
            for _ in range(max(1, a.repeats)):
                t0 = time.perf_counter()
                lp.reduce(x, cfg, ctx=ctx)
                dt = time.perf_counter() - t0
                best = dt if best is None else min(best, dt)
            out.write(f"{method},{k},{cfg.l or k},{_fmt(best)},{_fmt(rows / best)}\n")
    if a.out:
        out.close()
    return 0


def _load_manifest(path: str) -> dict:
    """load_manifest (lazypca_cli.cpp:47-58): a JSON object, else ParseError."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise lp.ParseError("manifest: cannot open " + path) from None
    try:
        j = json.loads(text)
    except ValueError as e:
        raise lp.ParseError(f"manifest: {e}") from None
    if not isinstance(j, dict):
        raise lp.ParseError("manifest: top level must be a JSON object")
    return j


def _given(argv, flag: str) -> bool:
    return any(v == flag or v.startswith(flag + "=") for v in argv)


def _fill_from(a, argv, flag: str, j: dict, key: str, attr: str, kind) -> None:
    """fill_from (lazypca_cli.cpp:60-69): the manifest's value unless the flag
    was given on the command line; a value of the wrong JSON type is a
    ParseError naming the key (nlohmann's get<T>: numbers convert between
    integer and floating point, strings and booleans do not)."""
    if _given(argv, flag) or key not in j:
        return
    v = j[key]
    ok = (isinstance(v, str) if kind is str else isinstance(v, bool) if kind is bool
          else isinstance(v, (int, float)) and not isinstance(v, bool))
    if not ok:
        raise lp.ParseError(f'manifest: bad value for "{key}": type must be {kind.__name__}, '
                            f"but is {type(v).__name__}")
    if kind is int:
        v = int(v)
        if attr == "seed" and v < 0:
            v &= (1 << 64) - 1
    setattr(a, attr, v)


_FIT_KEYS = [("--input", "input", "input", str), ("--format", "format", "format", str),
             ("--k", "k", "k", int), ("--l", "l", "l", int), ("--projection", "projection", "projection", str),
             ("--density-policy", "density_policy", "density_policy", str), ("--seed", "seed", "seed", int)]
_REDUCE_KEYS = [("--method", "method", "method", str), ("--block-rows", "block_rows", "block_rows", int),
                ("--streaming", "streaming", "streaming", bool),
                ("--deterministic", "deterministic", "deterministic", bool),
                ("--out-map", "out_map", "out_map", str), ("--out-reduced", "out_reduced", "out_reduced", str)]
_COMPARE_KEYS = [("--method-a", "method_a", "method_a", str), ("--method-b", "method_b", "method_b", str)]


def _apply_manifest(a, argv) -> None:
    if not getattr(a, "manifest", ""):
        return
    j = _load_manifest(a.manifest)
    keys = _FIT_KEYS + (_REDUCE_KEYS if a.cmd == "reduce" else _COMPARE_KEYS)
    for flag, key, attr, kind in keys:
        _fill_from(a, argv, flag, j, key, attr, kind)


def _fit_args(p, method_default="spca"):
    p.add_argument("--input", default="")
    p.add_argument("--format", default="mm")
    p.add_argument("--k", type=int, default=0)
    p.add_argument("--l", type=int, default=0)
    p.add_argument("--projection", default="gaussian")
    p.add_argument("--density-policy", dest="density_policy", default="conservative")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--block-rows", dest="block_rows", type=int, default=0)
    p.add_argument("--streaming", action="store_true")
    p.add_argument("--deterministic", action="store_true")  # accepted: runs are deterministic
    p.add_argument("--method", default=method_default)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1709_07175_b200")
    ap.add_argument("--device", type=int, default=0, help="CUDA device")
    ap.add_argument("--threads", type=int, default=0, help="accepted for compatibility (no host pool)")
    sub = ap.add_subparsers(dest="cmd")
    r = sub.add_parser("reduce", help="fit a reduction map and apply it")
    _fit_args(r)
    r.add_argument("--out-map", dest="out_map", default="")
    r.add_argument("--out-reduced", dest="out_reduced", default="")
    r.add_argument("--report", default="json")
    r.add_argument("--manifest", default="", help="JSON manifest with defaults for the above")
    c = sub.add_parser("compare", help="run two methods on the same data and report agreement")
    _fit_args(c)
    c.add_argument("--input-a", dest="input_a", default="")
    c.add_argument("--input-b", dest="input_b", default="")
    c.add_argument("--method-a", dest="method_a", default="spca")
    c.add_argument("--method-b", dest="method_b", default="lazy_spca")
    c.add_argument("--max-pairs", dest="max_pairs", type=int, default=10000)
    c.add_argument("--out-report", dest="out_report", default="")
    c.add_argument("--manifest", default="", help="JSON manifest with defaults for the above")
    b = sub.add_parser("bench", help="time the reducers over a list of target dims")
    b.add_argument("--input", default="")
    b.add_argument("--format", default="mm")
    b.add_argument("--m", type=int, default=0)
    b.add_argument("--n", type=int, default=0)
    b.add_argument("--density", type=float, default=0.01)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--k-list", dest="k_list", default="")
    b.add_argument("--repeats", type=int, default=1)
    b.add_argument("--methods", default="spca,lazy_spca")
    b.add_argument("--block-rows", dest="block_rows", type=int, default=25000)
    b.add_argument("--projection", default="very_sparse")
    b.add_argument("--density-policy", dest="density_policy", default="aggressive")
    b.add_argument("--out", default="")
    argv = sys.argv[1:] if argv is None else list(argv)
    a = ap.parse_args(argv)
    if not a.cmd:
        ap.print_help()
        return 0
    try:
        _apply_manifest(a, argv)
        ctx = lp.Context(a.device)
        return {"reduce": run_reduce, "compare": run_compare, "bench": run_bench}[a.cmd](a, ctx)
    except lp.ParseError as e:
        line = f" (line {e.line()})" if e.line() > 0 else ""
        print(f"error: {e}{line}", file=sys.stderr)
        return 2
    except lp.InvalidArgumentError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except lp.RankDeficiencyError as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    except lp.DimensionError as e:
        print(f"error: {e}", file=sys.stderr)
        return 4
    except Exception as e:  # noqa: BLE001 — the reference maps everything else to 1
        print(f"error: {e}", file=sys.stderr)
        return 1
