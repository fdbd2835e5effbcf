"""Builds the product library liblazypca_b200.so in-tree with nvcc for sm_100a.

The library is self-contained C ABI (include/lazypca_b200.h): static cudart,
NCCL from the system (same soname as torch's bundled copy), no torch types.
Usage: python -m paper_1709_07175_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
# LPCA_BUILD_TAG / LPCA_EXTRA_NVCC_FLAGS: a side build for experiments (e.g. the
# role timers, -DLPCA_PAIR_PROF) into _build_<tag>/ and liblazypca_b200_<tag>.so,
# loaded through LPCA_LIB_PATH; the product build ignores both.
_TAG = os.environ.get("LPCA_BUILD_TAG", "")
BUILD = PKG / ("_build" + (f"_{_TAG}" if _TAG else ""))
LIB = PKG / ("liblazypca_b200" + (f"_{_TAG}" if _TAG else "") + ".so")
EXTRA = os.environ.get("LPCA_EXTRA_NVCC_FLAGS", "").split() if _TAG else []
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", str(ROOT / "include"), "-I", str(CSRC)]
SOURCES = ["lpca.cu", "omega.cu", "gemm_simt.cu", "gemm_tc.cu", "small.cu", "eigh.cu", "sparse.cu", "metrics.cu",
           "spectral.cu", "sparse_omega.cu"]
HOST_SOURCES = ["textio.cpp"]  # host-only C++ (g++)
CXX = os.environ.get("CXX", "g++")


def _json_include() -> str:
    """Directory holding nlohmann/json.hpp (3.11.x), the reference's map-header
    serialiser: the copy vendored with cudnn_frontend in this image."""
    cands = [os.environ.get("LPCA_JSON_INCLUDE", "")]
    try:
        import site
        for sp in site.getsitepackages():
            cands.append(os.path.join(sp, "include", "cudnn_frontend", "thirdparty"))
    except Exception:
        pass
    cands.append(os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}",
                              "site-packages", "include", "cudnn_frontend", "thirdparty"))
    for c in cands:
        if c and os.path.exists(os.path.join(c, "nlohmann", "json.hpp")):
            return c
    raise RuntimeError("nlohmann/json.hpp not found (set LPCA_JSON_INCLUDE)")


def _obj(src: str) -> Path:
    return BUILD / (Path(src).stem + ".o")


def _needs(src: Path, obj: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src, *CSRC.glob("*.cuh"), ROOT / "include" / "lazypca_b200.h"]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)


def _compile(src: str, verbose: bool) -> None:
    obj = _obj(src)
    if src in HOST_SOURCES:
        cmd = [CXX, "-O2", "-std=c++17", "-fPIC", "-I", str(ROOT / "include"), "-I", str(CSRC),
               "-I", "/usr/local/cuda/include", "-I", _json_include(), "-c", str(CSRC / src), "-o", str(obj)]
    else:
        cmd = [NVCC, *ARCH, *FLAGS, *EXTRA, "-c", str(CSRC / src), "-o", str(obj)]
    if verbose and src not in HOST_SOURCES:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr)


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    todo = [s for s in SOURCES + HOST_SOURCES if force or _needs(CSRC / s, _obj(s))]
    with ThreadPoolExecutor(max_workers=min(8, max(1, len(todo)))) as ex:
        list(ex.map(lambda s: _compile(s, verbose), todo))
    objs = [str(_obj(s)) for s in SOURCES + HOST_SOURCES]
    if todo or not LIB.exists() or force:
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *objs, "-Xlinker", "-z,defs",
               "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
