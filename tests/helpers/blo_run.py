"""Fits a very sparse Omega through the dense X W pass (the default
for fp32 X) and writes sigma and V to argv[1]
(tests/test_gpu_sparse_omega.py compares runs with LPCA_BLO_SKIP on and off)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_1709_07175_b200 as lp  # noqa: E402

ctx = lp.Context(0)
out = {}
for name, (m, n, l, k, d, q) in {"c4ish": (6000, 16384, 300, 100, 1.0 / 128, 0),
                                  "ragged": (3001, 1000, 37, 12, 0.05, 1)}.items():
    x = torch.empty((m, n), dtype=torch.float32, device="cuda")
    lp.synth_lowrank(x, 0, min(n, 3 * l), 0.98, 0.01, 1000, ctx=ctx)
    c = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=k, l=l, power_iters=q,
                         projection=lp.ProjectionSpec(kind=lp.ProjectionKind.very_sparse, density=d, seed=11))
    r = lp.reduce_lazy_spca(x, c, ctx=ctx)
    out[name + "_s"] = r.singular_values
    out[name + "_v"] = r.v
np.savez(sys.argv[1], **out)
