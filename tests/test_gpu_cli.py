"""GPU: the command line (python -m paper_1709_07175_b200, the reference CLI's
reduce / compare / bench, lazypca_cli.cpp:162-452): outputs, records and exit
codes."""
import json
import subprocess
import sys

import numpy as np
import pytest

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

pytestmark = pytest.mark.gpu


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1709_07175_b200", *args], capture_output=True, text=True,
                          timeout=300)


@pytest.fixture
def data(tmp_path):
    x = O.synth_lowrank(0, 600, 90, 10, 0.85, 0.05, 7)
    mtx, csv = tmp_path / "x.mtx", tmp_path / "x.csv"
    lp.write_sparse_matrix_market(lp.SparseMatrix.from_dense(x), str(mtx))
    lp.write_dense_csv(x, str(csv))
    return x, mtx, csv, tmp_path


def test_reduce_writes_map_and_reduced(data, ctx):
    x, mtx, csv, tmp = data
    for fmt, path, extra in (("mm", mtx, []), ("csv", csv, ["--block-rows", "200"])):
        mp, red = tmp / f"m_{fmt}.map", tmp / f"y_{fmt}.csv"
        r = _cli("reduce", "--input", str(path), "--format", fmt, "--method", "lazy_spca", "--k", "5", "--l", "8",
                 "--seed", "3", "--out-map", str(mp), "--out-reduced", str(red), *extra)
        assert r.returncode == 0, r.stderr
        t = json.loads(r.stdout.strip().splitlines()[-1])
        assert set(t) == {"sketch", "qr", "f_form", "svd", "total"}
        m = lp.load_map_file(str(mp), ctx=ctx)
        want = lp.reduce_lazy_spca(x, lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=5, l=8,
                                                       projection=lp.ProjectionSpec(seed=3)), ctx=ctx)
        assert np.max(O.principal_angles(m.v, want.v)) < 1e-8
        y = lp.read_dense_csv(str(red))
        assert y.shape == (600, 5)
        assert np.allclose(y, x @ m.v, rtol=1e-9, atol=1e-9)


def test_reduce_manifest_matches_flags(data):
    """--manifest supplies the flags not given (lazypca_cli.cpp:580-598): the
    map equals the one from the same settings as flags."""
    _, mtx, _, tmp = data
    man = tmp / "m.json"
    man.write_text(json.dumps({"input": str(mtx), "method": "lazy_spca", "k": 5, "l": 9, "seed": 4,
                               "out_map": str(tmp / "from_manifest.map")}))
    r = _cli("reduce", "--manifest", str(man), "--k", "6")
    assert r.returncode == 0, r.stderr
    r2 = _cli("reduce", "--input", str(mtx), "--method", "lazy_spca", "--k", "6", "--l", "9", "--seed", "4",
              "--out-map", str(tmp / "from_flags.map"))
    assert r2.returncode == 0, r2.stderr
    assert (tmp / "from_manifest.map").read_bytes() == (tmp / "from_flags.map").read_bytes()


def test_compare_spca_lazy_record_and_exit(data):
    _, mtx, _, tmp = data
    rep = tmp / "r.jsonl"
    r = _cli("compare", "--input", str(mtx), "--k", "6", "--l", "6", "--seed", "2", "--max-pairs", "500",
             "--out-report", str(rep))
    assert r.returncode == 0, r.stderr
    rec = json.loads(r.stdout.strip())
    assert list(rec)[:6] == ["method_a", "method_b", "k", "l", "seed", "chordal"]
    assert rec["method_a"] == "spca" and rec["method_b"] == "lazy_spca" and rec["chordal"] <= 1e-8
    assert rec["bound"] is None  # max(600, 90) is above the compare command's densify limit (300)
    assert json.loads(rep.read_text().strip()) == rec


def test_bench_csv(data):
    _, mtx, _, tmp = data
    out = tmp / "b.csv"
    r = _cli("bench", "--input", str(mtx), "--k-list", "4,8", "--methods", "lazy_spca", "--block-rows", "0",
             "--projection", "gaussian", "--out", str(out))
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "method,k,l,seconds,rows_per_second" and len(lines) == 3


def test_exit_codes(data):
    _, mtx, _, tmp = data
    bad = tmp / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate real general\n3 3 1\n4 1 1\n")
    r = _cli("reduce", "--input", str(bad), "--k", "2")
    assert r.returncode == 2 and "(line 3)" in r.stderr
    assert _cli("reduce", "--k", "2").returncode == 2
    assert _cli("reduce", "--input", str(mtx), "--format", "xml", "--k", "2").returncode == 2
    low = tmp / "low.mtx"
    lp.write_sparse_matrix_market(lp.SparseMatrix.from_dense(np.outer(np.arange(1, 41.0), np.arange(1, 31.0))),
                                  str(low))
    r = _cli("reduce", "--input", str(low), "--method", "lazy_spca", "--k", "5", "--l", "8")
    assert r.returncode == 3, r.stderr
