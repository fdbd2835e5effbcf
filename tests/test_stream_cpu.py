"""CPU: the numpy restatement of the streaming reducers (Algorithms 3 and 4,
proj/core/src/reducer.cpp:236-335) against the compiled reference's own
streaming path (reduce() with block_rows, reducer.cpp:340-346)."""
import numpy as np
import pytest

from oracle import lazypca_oracle as O
from oracle import refbind


@pytest.fixture(scope="module")
def ref():
    if not refbind.available():
        pytest.skip("compiled reference unavailable")
    return refbind


@pytest.mark.parametrize("method,code", [("lazy", 2), ("spca", 1)])
def test_streaming_oracle_matches_reference(ref, method, code):
    x = O.synth_lowrank(0, 700, 60, 12, 0.85, 0.01, 3)
    k, l, br = 5, 10, 160
    v_ref, s_ref, _, _ = ref.reduce(code, x, k, l, 11, block_rows=br)
    blocks = [x[i:i + br] for i in range(0, x.shape[0], br)]
    v, s, _ = O.reduce_streaming(blocks, method, k, l, 11)
    assert np.max(np.abs(s - s_ref) / s_ref) < 1e-11
    assert np.max(O.principal_angles(v, v_ref)) < 1e-9
    # one pass over blocks gives the in-core subspace (Algorithm 4 == 2; 3 == 1 in exact arithmetic)
    v_in, s_in, _ = (O.reduce_lazy_spca if method == "lazy" else O.reduce_spca)(x, k, l, 11)
    assert np.max(np.abs(s - s_in) / s_in) < 1e-10
