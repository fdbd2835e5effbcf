"""GPU: BASELINE configs[1] at FULL size (X fp32 1,000,000 x 4,096, l = 110,
k = 100) through the bench's call (fit_transform), against the compiled
reference's streaming Lazy SPCA on the same X (tests/golden/c2_full.npz, made
on a GPU box's host cores by tests/golden/make_c2_fixture.py from the device
generator's X; VERDICT r1 missing #5)."""
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

pytestmark = pytest.mark.gpu
FIX = Path(__file__).resolve().parent / "golden" / "c2_full.npz"


@pytest.mark.skipif(not FIX.exists(), reason="tests/golden/c2_full.npz not generated")
def test_c2_full_size_matches_the_reference_streaming_fit(ctx):
    f = np.load(FIX)
    m, n, k, l = int(f["m"]), int(f["n"]), int(f["k"]), int(f["l"])
    x = torch.empty((m, n), dtype=torch.float32, device="cuda")
    lp.synth_lowrank(x, 0, 200, 0.97, 0.01, int(f["seed_x"]), ctx=ctx)
    cfg = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=k, l=l,
                           projection=lp.ProjectionSpec(seed=int(f["seed_omega"])))
    y = torch.empty((m, k), dtype=torch.float32, device="cuda")
    mp, _ = lp.fit_transform(x, cfg, ctx=ctx, out=y)
    s = f["sigma"]
    rel = np.abs(mp.singular_values - s) / s
    ang = O.principal_angles(mp.v[:, :10], f["v10"]).max()
    print(f"c2 full: sigma rel max {rel.max():.2e} normwise {np.abs(mp.singular_values - s).max() / s[0]:.2e}, "
          f"top-10 angle {ang:.2e}")
    assert rel.max() < 1e-4   # north_star's fp32 bar
    assert rel.max() < 3e-5   # measured 3.3e-6
    assert ang < 5e-5  # measured 4.6e-6
