"""Runs tools/peaks (built from tools/peaks.cu here) on the GPU box and writes
profiles/peaks_r02.json: the measured tcgen05 f16 / tf32, DMMA and DFMA rates
bench.py uses as roofline denominators next to MEASURED_PEAKS.json.
Usage: python tools/peaks.py [out.json]"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
out = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "peaks_r02.json"
r = subprocess.run([str(ROOT / "tools" / "peaks")], capture_output=True, text=True, timeout=120)
print(r.stdout, r.stderr)
d = json.loads(r.stdout.strip().splitlines()[-1])
d["how"] = ("tools/peaks.cu: every SM issues back-to-back dense MMAs (tcgen05 cta_group::2 M=256 N=256, A in "
            "TMEM; mma.sync m8n8k4 f64) or DFMA chains for ~2 s per unit, CUDA-event timed; sm_mhz from clock64")
out.write_text(json.dumps(d, indent=1) + "\n")
