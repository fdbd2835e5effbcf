"""CPU: the command line's manifest handling (load_manifest / fill_from,
lazypca_cli.cpp:47-69, 580-613) — the manifest is read before any device work,
so its errors exit with the ParseError code 2 without a GPU."""
import argparse
import json
import subprocess
import sys

import pytest

from paper_1709_07175_b200 import api as lp
from paper_1709_07175_b200 import cli


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1709_07175_b200", *args], capture_output=True, text=True,
                          timeout=300)


@pytest.mark.parametrize("content,needle", [
    (None, "manifest: cannot open"),
    ("[1, 2]", "manifest: top level must be a JSON object"),
    ("{not json", "manifest: "),
    ('{"k": "five"}', 'manifest: bad value for "k"'),
    ('{"streaming": 1}', 'manifest: bad value for "streaming"'),
    ('{"method": 3}', 'manifest: bad value for "method"'),
])
def test_manifest_errors_exit_2(tmp_path, content, needle):
    path = tmp_path / "m.json"
    if content is not None:
        path.write_text(content)
    r = _cli("reduce", "--manifest", str(path))
    assert r.returncode == 2, r.stderr
    assert r.stderr.startswith("error: " + needle), r.stderr


def _ns(**kw):
    base = dict(cmd="reduce", input="", format="mm", k=0, l=0, projection="gaussian", density_policy="conservative",
                seed=0, block_rows=0, streaming=False, deterministic=False, method="spca", out_map="",
                out_reduced="", manifest="")
    base.update(kw)
    return argparse.Namespace(**base)


def test_manifest_fills_unset_flags_only(tmp_path):
    path = tmp_path / "m.json"
    path.write_text(json.dumps({"input": "x.mtx", "k": 7, "l": 12.0, "method": "lazy_spca", "seed": 5,
                                "streaming": True, "block_rows": 100, "out_map": "a.map", "unknown": 1}))
    a = _ns(manifest=str(path), k=3)
    cli._apply_manifest(a, ["reduce", "--manifest", str(path), "--k", "3"])
    assert (a.input, a.k, a.l, a.method, a.seed, a.streaming, a.block_rows, a.out_map) == \
        ("x.mtx", 3, 12, "lazy_spca", 5, True, 100, "a.map")
    b = _ns(cmd="compare", manifest=str(path), method_a="spca", method_b="lazy_spca")
    path.write_text(json.dumps({"method_a": "rp", "method_b": "spca", "k": 4, "out_map": "ignored"}))
    cli._apply_manifest(b, ["compare", "--manifest", str(path), "--method-b=lazy_spca"])
    assert (b.method_a, b.method_b, b.k, b.out_map) == ("rp", "lazy_spca", 4, "")


def test_manifest_error_class():
    with pytest.raises(lp.ParseError):
        cli._load_manifest("/nonexistent/manifest.json")
