"""CPU: the C-ABI library loads, exports every symbol include/*.h declares, and
its pure-host entry points (config resolution, density policy) behave like the
reference. No compute call runs here (there is no GPU); creating a context must
fail loudly rather than fall back to the CPU."""
import re
from pathlib import Path

import pytest

from paper_1709_07175_b200 import _lib as L
from paper_1709_07175_b200 import api

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "lazypca_b200.h"


def _declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lpca_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = L.load()
    declared = _declared_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in {HEADER.name} but not exported"
    assert set(declared) == set(L.SIGNATURES), "ctypes signature table out of sync with the header"


def test_abi_version():
    assert L.load().lpca_abi_version() == 1


def test_library_has_sm100a_code_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(L.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_context_creation_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(api.CudaError):
        api.Context(0)


def test_config_resolution_mirrors_reference():
    # test_reducer.cpp "config resolution fills defaults and rejects contradictions"
    def cfg(method, k, l, seed=1):
        return api.ReducerConfig(method=method, k=k, l=l, projection=api.ProjectionSpec(seed=seed))

    r = cfg(api.ReducerMethod.spca, 4, 0).resolved(30)
    assert r.l == 4 and r.projection.n == 30 and r.projection.l == 4
    with pytest.raises(api.InvalidArgumentError):
        cfg(api.ReducerMethod.spca, 0, 0).resolved(30)
    with pytest.raises(api.InvalidArgumentError):
        cfg(api.ReducerMethod.spca, 6, 4).resolved(30)
    with pytest.raises(api.InvalidArgumentError):
        cfg(api.ReducerMethod.rp, 3, 5).resolved(30)
    with pytest.raises(api.InvalidArgumentError):
        cfg(api.ReducerMethod.spca, 4, 40).resolved(30)
    s = cfg(api.ReducerMethod.spca, 4, 6)
    s.streaming = True
    with pytest.raises(api.InvalidArgumentError):
        s.resolved(30)
    d = cfg(api.ReducerMethod.lazy_spca, 4, 6)
    d.projection.n = 31
    with pytest.raises(api.DimensionError):
        d.resolved(30)
    d = cfg(api.ReducerMethod.lazy_spca, 4, 6)
    d.projection.density = 0.0
    with pytest.raises(api.InvalidArgumentError):
        d.resolved(30)
    b = cfg(api.ReducerMethod.lazy_spca, 4, 6)
    b.block_rows = 10
    assert b.resolved(30).streaming


def test_density_policy_matches_reference(golden):
    assert api.density_for(api.DensityPolicy.aggressive(), 100) == float(golden.kat["density_aggr_100"])
    assert api.density_for(api.DensityPolicy.conservative(), 100) == float(golden.kat["density_cons_100"])
    assert api.density_for(api.DensityPolicy.explicit_value(0.25), 50) == 0.25
    with pytest.raises(api.InvalidArgumentError):
        api.density_for(api.DensityPolicy.aggressive(), 1)
    with pytest.raises(api.InvalidArgumentError):
        api.density_for(api.DensityPolicy.explicit_value(0.0), 10)
    assert api.DensityPolicy.parse("value:0.125").value == 0.125
    with pytest.raises(api.InvalidArgumentError):
        api.DensityPolicy.parse("sometimes")


def test_method_names_round_trip():
    for m in api.ReducerMethod:
        assert api.reducer_method_from_string(api.to_string(m)) == m
    with pytest.raises(api.InvalidArgumentError):
        api.reducer_method_from_string("pca")


def test_shim_header_compiles_against_abi(tmp_path):
    """include/lazypca_b200.hpp (the reference-shaped C++ shim) compiles and links."""
    import subprocess
    src = tmp_path / "t.cpp"
    src.write_text('#include "lazypca_b200.hpp"\nint main(){ lazypca::ReducerConfig c; c.k = 3;'
                   ' return lazypca::ReducerConfig(c).resolved(10).l == 3 ? 0 : 1; }\n')
    exe = tmp_path / "t"
    r = subprocess.run(["g++", "-std=c++17", f"-I{ROOT / 'include'}", str(src), "-o", str(exe),
                        f"-L{L.LIB_PATH.parent}", "-llazypca_b200", f"-Wl,-rpath,{L.LIB_PATH.parent}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([str(exe)]).returncode == 0
    # the streaming half of the shim (RowBlockStream, reduce_*_streaming) compiles too
    r = subprocess.run(["g++", "-std=c++17", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "shim_stream.cpp"),
                        "-o", str(tmp_path / "s"), f"-L{L.LIB_PATH.parent}", "-llazypca_b200",
                        f"-Wl,-rpath,{L.LIB_PATH.parent}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
