"""CPU: bench.py's multi-GPU launcher and strong-scaling row split (VERDICT r1:
`--gpus N` must start N ranks itself and shard a fixed global row count)."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def test_shard_rows_cover_the_global_rows_once():
    for m, world in ((4_600_000, 1), (4_600_000, 2), (4_600_000, 8), (10, 4), (3, 8), (0, 2)):
        shards = [bench.shard_rows(m, world, r) for r in range(world)]
        assert sum(c for _, c in shards) == m
        nxt = 0
        for lo, c in shards:
            assert c >= 0 and (c == 0 or lo == nxt)
            nxt = lo + c
        assert max(c for _, c in shards) == -(-m // world) if m else True


def test_gpus_flag_launches_ranks_with_the_row_split():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--stub-worker", "--config", "c3"],
                       capture_output=True, text=True, timeout=240, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [json.loads(s) for s in r.stdout.splitlines() if s.startswith("{")]
    assert len(line) == 1, r.stdout
    d = line[0]
    assert d["n_gpus"] == 2 and d["global_rows"] == 4_600_000
    assert [s["rank"] for s in d["shards"]] == [0, 1]
    assert all(s["world"] == 2 for s in d["shards"])
    assert [(s["row0"], s["rows"]) for s in d["shards"]] == [(0, 2_300_000), (2_300_000, 2_300_000)]


def test_gpus_must_match_an_existing_world(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "4")

    class A:
        gpus = 2
    try:
        bench.relaunch_if_needed(A())
    except SystemExit as e:
        assert "WORLD_SIZE=4" in str(e)
    else:
        raise AssertionError("mismatch accepted")


def test_default_workload_is_the_north_star():
    assert bench.DEFAULT_CONFIG == "c3"
    c = bench.CONFIGS["c3"]
    assert (c["m"], c["n"], c["l"], c["k"], c["q"], c["dtype"]) == (4_600_000, 4096, 220, 200, 1, "f32")
