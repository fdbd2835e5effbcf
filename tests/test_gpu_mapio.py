"""GPU: a fitted device map through a map file (save_map_file / load_map_file,
proj/core/src/reducer.cpp:355-412) — byte-identical to the reference's file for
the same map, and the reloaded map transforms identically."""
import numpy as np
import pytest

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

pytestmark = pytest.mark.gpu


def test_fit_save_load_transform(ctx, ref, tmp_path):
    x = O.synth_lowrank(0, 2000, 120, 20, 0.9, 0.01, 4)
    cfg = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=6, l=12, projection=lp.ProjectionSpec(seed=21))
    m = lp.reduce_lazy_spca(x, cfg, ctx=ctx)
    ours = tmp_path / "fit.map"
    lp.save_map_file(m, str(ours))
    theirs = tmp_path / "ref.map"
    ref.save_map_file(str(theirs), 2, 6, 12, 120, 21, 1.0, np.sqrt(12.0), m.v, m.singular_values)
    assert ours.read_bytes() == theirs.read_bytes()
    back = lp.load_map_file(str(ours), ctx=ctx)
    assert np.array_equal(back.v, m.v) and np.array_equal(back.singular_values, m.singular_values)
    assert np.array_equal(lp.apply_map(back, x, ctx=ctx), lp.apply_map(m, x, ctx=ctx))
    # the reference reads it back too
    r = ref.load_map_file(str(ours))
    assert np.array_equal(r["v"], m.v)
