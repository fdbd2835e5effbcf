"""GPU: the streaming reducers (lpca_fit_stream; reduce_{lazy_spca,spca}_streaming,
proj/core/src/reducer.cpp:236-335) and reduce() with block_rows (:340-346),
against the compiled reference's streaming path and the in-core fit."""
import numpy as np
import pytest
import torch

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

pytestmark = pytest.mark.gpu


def _cfg(method, k, l, seed=11, block_rows=0):
    return lp.ReducerConfig(method=method, k=k, l=l, projection=lp.ProjectionSpec(seed=seed),
                            block_rows=block_rows)


class _ListStream(lp.RowBlockStream):
    def __init__(self, blocks, slices=None):
        self.blocks = list(blocks)
        self.slices = list(slices) if slices is not None else list(range(len(self.blocks)))
        self.i = 0

    def next(self):
        if self.i >= len(self.blocks):
            return None
        b = lp.RowBlock(self.slices[self.i], self.blocks[self.i])
        self.i += 1
        return b


@pytest.mark.parametrize("method,code", [(lp.ReducerMethod.lazy_spca, 2), (lp.ReducerMethod.spca, 1)])
def test_stream_fp64_matches_reference_streaming(ctx, ref, method, code):
    x = O.synth_lowrank(0, 3000, 200, 30, 0.9, 0.01, 5)
    k, l, br = 10, 20, 700
    v_ref, s_ref, _, _ = ref.reduce(code, x, k, l, 11, block_rows=br)
    stream = lp.SliceRowBlockStream(x, br)
    fn = lp.reduce_lazy_spca_streaming if method == lp.ReducerMethod.lazy_spca else lp.reduce_spca_streaming
    m = fn(stream, _cfg(method, k, l), ctx=ctx)
    assert np.max(np.abs(m.singular_values - s_ref) / s_ref) < 1e-10
    assert np.max(O.principal_angles(m.v, v_ref)) < 1e-8
    # reduce() with block_rows takes the same route through lpca_fit
    m2 = lp.reduce(x, _cfg(method, k, l, block_rows=br), ctx=ctx)
    assert np.max(np.abs(m2.singular_values - s_ref) / s_ref) < 1e-10


def test_single_block_stream_is_bitwise_in_core(ctx):
    x = O.synth_lowrank(0, 2000, 150, 20, 0.9, 0.01, 6)
    cfg = _cfg(lp.ReducerMethod.lazy_spca, 8, 16)
    m_in = lp.reduce_lazy_spca(x, cfg, ctx=ctx)
    m_st = lp.reduce_lazy_spca_streaming(_ListStream([x]), cfg, ctx=ctx)
    assert np.array_equal(m_in.v, m_st.v)
    assert np.array_equal(m_in.singular_values, m_st.singular_values)


@pytest.mark.parametrize("where", ["host", "device"])
def test_stream_fp32_tensor_core_blocks(ctx, where):
    x = O.synth_lowrank(0, 60000, 1024, 60, 0.95, 0.01, 7).astype(np.float32)
    k, l, br = 40, 48, 16384
    cfg = _cfg(lp.ReducerMethod.lazy_spca, k, l)
    xin = torch.from_numpy(x).cuda() if where == "device" else x
    m_in = lp.reduce_lazy_spca(xin, cfg, ctx=ctx)
    blocks = [xin[i:i + br] for i in range(0, x.shape[0], br)]  # last block is ragged
    m_st = lp.reduce_lazy_spca_streaming(_ListStream(blocks), cfg, ctx=ctx)
    s0 = m_in.singular_values
    assert np.max(np.abs(m_st.singular_values - s0) / s0) < 1e-5
    assert np.max(O.principal_angles(m_st.v[:, :k // 2], m_in.v[:, :k // 2])) < 1e-4
    v64, s64, _ = O.reduce_streaming([x[i:i + br] for i in range(0, x.shape[0], br)], "lazy", k, l, 11)
    assert np.max(np.abs(m_st.singular_values - s64) / s64) < 1e-4


def test_stream_errors_match_reference(ctx):
    x = O.synth_lowrank(0, 400, 50, 10, 0.9, 0.01, 8)
    cfg = _cfg(lp.ReducerMethod.lazy_spca, 4, 8)
    with pytest.raises(lp.InvalidArgumentError, match="empty"):
        lp.reduce_lazy_spca_streaming(_ListStream([]), cfg, ctx=ctx)
    with pytest.raises(lp.InvalidArgumentError, match="first slice index must be 0"):
        lp.reduce_lazy_spca_streaming(_ListStream([x[:200]], [1]), cfg, ctx=ctx)
    with pytest.raises(lp.InvalidArgumentError, match="expected slice 1, got 2"):
        lp.reduce_lazy_spca_streaming(_ListStream([x[:200], x[200:]], [0, 2]), cfg, ctx=ctx)
    with pytest.raises(lp.DimensionError, match="columns"):
        lp.reduce_lazy_spca_streaming(_ListStream([x[:200], x[200:, :40]]), cfg, ctx=ctx)
    with pytest.raises(lp.DimensionError, match="at least l"):
        lp.reduce_spca_streaming(_ListStream([x[:5], x[5:]]), _cfg(lp.ReducerMethod.spca, 4, 8), ctx=ctx)

    class Boom(lp.RowBlockStream):
        def next(self):
            raise KeyError("disk gone")

    with pytest.raises(KeyError):
        lp.reduce_lazy_spca_streaming(Boom(), cfg, ctx=ctx)
    # the context stays usable after a failed stream
    m = lp.reduce_lazy_spca(x, cfg, ctx=ctx)
    assert m.singular_values[0] > 0


def test_stream_rp_reads_only_the_width(ctx):
    x = O.synth_lowrank(0, 300, 40, 8, 0.9, 0.01, 9)
    cfg = _cfg(lp.ReducerMethod.rp, 6, 6)
    s = _ListStream([x[:100], x[100:]])
    m = lp.api._fit_stream(s, cfg, None, ctx)
    v_ref, _ = O.reduce_rp(40, 6, 11)
    assert np.array_equal(m.v, v_ref)


def test_cpp_shim_streaming_end_to_end(tmp_path):
    """A reference caller's C++ (tests/cpp/shim_stream.cpp) relinked against the library."""
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    lib = root / "paper_1709_07175_b200"
    exe = tmp_path / "s"
    r = subprocess.run(["g++", "-std=c++17", "-O1", f"-I{root / 'include'}", str(root / "tests" / "cpp" / "shim_stream.cpp"),
                        "-o", str(exe), f"-L{lib}", "-llazypca_b200", f"-Wl,-rpath,{lib}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
