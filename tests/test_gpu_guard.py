"""GPU: no kernel writes outside its buffers (compute-
sanitizer is closed on the pool, so pattern bands stand in for memcheck):
ragged shapes of every kernel family, fp32 and fp64, with a guard band after
every library workspace (LPCA_WS_GUARD=1, lpca_debug_check_guards) and
sentinels around the caller's Y."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_no_out_of_bounds_writes():
    env = dict(os.environ, LPCA_WS_GUARD="1")
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "helpers" / "guard_run.py")], capture_output=True,
                       text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["bad_workspaces"] == 0, d["names"]
    assert d["bad_y"] == []
