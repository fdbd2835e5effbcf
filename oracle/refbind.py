"""TEST INFRASTRUCTURE ONLY — ctypes binding of oracle/_ref/liblazypca_ref.so.

That library is the unmodified reference core (/root/reference/proj/core/src,
built by oracle/Makefile) behind the flat wrapper oracle/ref_capi.cpp. Only
tests/, __graft_entry__.smoke() and bench.py's CPU legs use it, as the checker
or the timed reference; the product never loads it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "liblazypca_ref.so"
# the reference's own default build (-march=native) for the timed CPU baseline
LIB_NATIVE = HERE / "_ref" / "liblazypca_ref_native.so"
_NATIVE_ISA = ("avx512f", "avx512bw", "avx512vl", "avx512_fp16", "amx_tile")
REF_SRC = Path("/root/reference/proj/core")

_lib = None


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str, index: int):
        super().__init__(msg)
        self.code, self.index = code, index


def build_if_possible() -> bool:
    """Builds _ref from the reference sources when they are present (here, not on the GPU box)."""
    if REF_SRC.exists():
        r = subprocess.run(["make", "-s", "-j8", "-C", str(HERE)], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"oracle/_ref build failed:\n{r.stdout}\n{r.stderr}")
    return LIB.exists()


def available() -> bool:
    return LIB.exists()


_use_native = False


def native_supported() -> bool:
    """True when the -march=sapphirerapids build exists and this CPU has that ISA."""
    try:
        flags = Path("/proc/cpuinfo").read_text().split()
    except OSError:
        return False
    return LIB_NATIVE.exists() and all(f in flags for f in _NATIVE_ISA)


def use_native(on: bool = True) -> bool:
    """Selects the native build (before the first call). Returns whether it is used."""
    global _use_native
    if _lib is not None:
        raise RuntimeError("refbind: select the build before the first call")
    _use_native = bool(on) and native_supported()
    return _use_native


def build_flags() -> str:
    return "-O3 -march=sapphirerapids (reference default -march=native)" if _use_native else "-O3 -march=x86-64-v2"


def load():
    global _lib
    if _lib is None:
        path = LIB_NATIVE if _use_native else LIB
        if not path.exists():
            raise RuntimeError(f"{path} missing; build it with `make -C oracle` where /root/reference exists")
        lib = C.CDLL(str(path))
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_last_error_index.restype = C.c_int64
        _lib = lib
    return _lib


def _chk(code: int) -> None:
    if code != 0:
        lib = load()
        raise RefError(code, lib.ref_last_error().decode(), int(lib.ref_last_error_index()))


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else None


def set_threads(n: int) -> None:
    load().ref_set_thread_count(C.c_int(n))


def regenerate(kind: int, n: int, l: int, density: float, seed: int):
    out = np.zeros((n, l), order="F")
    sc = C.c_double()
    _chk(load().ref_regenerate(C.c_int(kind), C.c_int64(n), C.c_int64(l), C.c_double(density),
                               C.c_uint64(seed), _p(out), C.byref(sc)))
    return out, sc.value


def density_for(mode: int, k: int, value: float = 0.0) -> float:
    out = C.c_double()
    _chk(load().ref_density_for(C.c_int(mode), C.c_int64(k), C.c_double(value), C.byref(out)))
    return out.value


def _x(x: np.ndarray):
    x = np.ascontiguousarray(x)
    dt = 4 if x.dtype == np.float32 else 8
    if x.dtype not in (np.float32, np.float64):
        x = x.astype(np.float64)
    return x, dt


def reduce(method: int, x: np.ndarray, k: int, l: int, seed: int, kind: int = 0, density: float = 1.0,
           block_rows: int = 0):
    """reduce() on dense row-major X. Returns (V n x k, sigma, scale, timings[5])."""
    x, dt = _x(x)
    m, n = x.shape
    v = np.zeros((n, k), order="F")
    sig = np.zeros(k)
    sc = C.c_double()
    t = np.zeros(5)
    _chk(load().ref_reduce(C.c_int(method), _p(x), C.c_int(dt), C.c_int64(m), C.c_int64(n), C.c_int64(k),
                           C.c_int64(l), C.c_uint64(seed), C.c_int(kind), C.c_double(density),
                           C.c_int64(block_rows), _p(v), _p(sig), C.byref(sc), _p(t)))
    return v, sig, sc.value, t


def fit_transform(method: int, x: np.ndarray, k: int, l: int, seed: int, kind: int = 0,
                  density: float = 1.0, want_y: bool = True):
    """reduce + apply_map, timed inside the reference call (CSC build excluded)."""
    x, dt = _x(x)
    m, n = x.shape
    y = np.zeros((m, k), order="F") if want_y else None
    v = np.zeros((n, k), order="F")
    sig = np.zeros(k)
    secs = C.c_double()
    _chk(load().ref_fit_transform(C.c_int(method), _p(x), C.c_int(dt), C.c_int64(m), C.c_int64(n),
                                  C.c_int64(k), C.c_int64(l), C.c_uint64(seed), C.c_int(kind),
                                  C.c_double(density), _p(y), _p(v), _p(sig), C.byref(secs)))
    return y, v, sig, secs.value


def fit_transform_csc(method: int, m: int, n: int, col_ptr, row_idx, values, k: int, l: int, seed: int,
                     kind: int = 0, density: float = 1.0, want_y: bool = True):
    """reduce + apply_map on a canonical CSC X (int64 col_ptr / row_idx, fp64
    values); returns (Y, V, sigma, seconds of reduce + apply_map)."""
    cp = np.ascontiguousarray(col_ptr, dtype=np.int64)
    ri = np.ascontiguousarray(row_idx, dtype=np.int64)
    va = np.ascontiguousarray(values, dtype=np.float64)
    y = np.zeros((m, k), order="F") if want_y else None
    v = np.zeros((n, k), order="F")
    sig = np.zeros(k)
    secs = C.c_double()
    _chk(load().ref_fit_transform_csc(C.c_int(method), C.c_int64(m), C.c_int64(n), _p(cp), _p(ri), _p(va),
                                      C.c_int64(k), C.c_int64(l), C.c_uint64(seed), C.c_int(kind),
                                      C.c_double(density), _p(y), _p(v), _p(sig), C.byref(secs)))
    return y, v, sig, secs.value


def lazy_power_fit_transform(x: np.ndarray, k: int, l: int, seed: int, q: int, kind: int = 0,
                             density: float = 1.0, want_y: bool = True):
    """Lazy SPCA with q power steps composed from the reference's kernels
    (build_sketch, gemm_t, householder_qr, spmm, truncated_svd_via_gram) + the
    transform; returns (Y, V, sigma, seconds). See ref_capi.cpp."""
    x, dt = _x(x)
    m, n = x.shape
    y = np.zeros((m, k), order="F") if want_y else None
    v = np.zeros((n, k), order="F")
    sig = np.zeros(k)
    secs = C.c_double()
    _chk(load().ref_lazy_power_fit_transform(_p(x), C.c_int(dt), C.c_int64(m), C.c_int64(n), C.c_int64(k),
                                             C.c_int64(l), C.c_uint64(seed), C.c_int(kind), C.c_double(density),
                                             C.c_int(q), _p(y), _p(v), _p(sig), C.byref(secs)))
    return y, v, sig, secs.value


def apply_map(x: np.ndarray, v: np.ndarray):
    x, dt = _x(x)
    v = np.asfortranarray(v, dtype=np.float64)
    m, n = x.shape
    y = np.zeros((m, v.shape[1]), order="F")
    _chk(load().ref_apply_map(_p(x), C.c_int(dt), C.c_int64(m), C.c_int64(n), _p(v), C.c_int64(v.shape[1]),
                              _p(y)))
    return y


def spmm(x: np.ndarray, w: np.ndarray):
    x, dt = _x(x)
    w = np.asfortranarray(w, dtype=np.float64)
    m, n = x.shape
    out = np.zeros((m, w.shape[1]), order="F")
    _chk(load().ref_spmm(_p(x), C.c_int(dt), C.c_int64(m), C.c_int64(n), _p(w), C.c_int64(w.shape[1]),
                         _p(out)))
    return out


def gemm_t(u: np.ndarray, x: np.ndarray):
    x, dt = _x(x)
    u = np.asfortranarray(u, dtype=np.float64)
    m, l = u.shape
    n = x.shape[1]
    out = np.zeros((l, n), order="F")
    _chk(load().ref_gemm_t(_p(u), C.c_int64(m), C.c_int64(l), _p(x), C.c_int(dt), C.c_int64(n), _p(out)))
    return out


def dense_aat(f: np.ndarray):
    f = np.asfortranarray(f, dtype=np.float64)
    l, n = f.shape
    out = np.zeros((l, l), order="F")
    _chk(load().ref_dense_aat(_p(f), C.c_int64(l), C.c_int64(n), _p(out)))
    return out


def eigh(a: np.ndarray, which: str = "tridiag"):
    a = np.asfortranarray(a, dtype=np.float64)
    l = a.shape[0]
    ev = np.zeros(l)
    vec = np.zeros((l, l), order="F")
    _chk(load().ref_eigh(C.c_int(0 if which == "tridiag" else 1), _p(a), C.c_int64(l), _p(ev), _p(vec)))
    return ev, vec


def truncated_svd(f: np.ndarray, k: int):
    f = np.asfortranarray(f, dtype=np.float64)
    l, n = f.shape
    sig = np.zeros(k)
    v = np.zeros((n, k), order="F")
    ut = np.zeros((l, k), order="F")
    _chk(load().ref_truncated_svd(_p(f), C.c_int64(l), C.c_int64(n), C.c_int64(k), _p(sig), _p(v), _p(ut)))
    return sig, v, ut


def householder_qr(a: np.ndarray):
    a = np.asfortranarray(a, dtype=np.float64)
    m, l = a.shape
    q = np.zeros((m, l), order="F")
    r = np.zeros((l, l), order="F")
    _chk(load().ref_householder_qr(_p(a), C.c_int64(m), C.c_int64(l), _p(q), _p(r)))
    return q, r


def chordal(v1: np.ndarray, v2: np.ndarray) -> float:
    v1 = np.asfortranarray(v1, dtype=np.float64)
    v2 = np.asfortranarray(v2, dtype=np.float64)
    out = C.c_double()
    _chk(load().ref_chordal(_p(v1), _p(v2), C.c_int64(v1.shape[0]), C.c_int64(v1.shape[1]), C.byref(out)))
    return out.value


def reconstruction_error(route: int, x: np.ndarray, u: np.ndarray, k: int, l: int, with_bound: bool = False,
                         densify_limit: int = 2000):
    """(spectral, frobenius, sigma_{k+1} or None, bound or None); route 0 = qr, 1 = lazy."""
    x, dt = _x(x)
    u = np.asfortranarray(u, dtype=np.float64)
    out = np.zeros(4)
    flags = np.zeros(2, dtype=np.int32)
    _chk(load().ref_reconstruction_error(C.c_int(route), _p(x), C.c_int(dt), C.c_int64(x.shape[0]),
                                         C.c_int64(x.shape[1]), _p(u), C.c_int64(l), C.c_int64(k),
                                         C.c_int(int(with_bound)), C.c_int64(densify_limit), _p(out), _p(flags)))
    return out[0], out[1], (out[2] if flags[0] else None), (out[3] if flags[1] else None)


def row_space_reconstruction_error(x: np.ndarray, v: np.ndarray):
    x, dt = _x(x)
    v = np.asfortranarray(v, dtype=np.float64)
    out = np.zeros(2)
    _chk(load().ref_row_space_reconstruction_error(_p(x), C.c_int(dt), C.c_int64(x.shape[0]), C.c_int64(x.shape[1]),
                                                   _p(v), C.c_int64(v.shape[1]), _p(out)))
    return out[0], out[1]


def spectral_norm(x: np.ndarray) -> float:
    x, dt = _x(x)
    out = C.c_double()
    _chk(load().ref_spectral_norm(_p(x), C.c_int(dt), C.c_int64(x.shape[0]), C.c_int64(x.shape[1]), C.byref(out)))
    return out.value


def read_matrix_file(kind: int, path: str):
    """kind 0 sparse MatrixMarket -> (rows, cols, ptr, idx, val); 1 dense MatrixMarket, 2 CSV -> array."""
    r, c, z = C.c_int64(), C.c_int64(), C.c_int64()
    lib = load()
    _chk(lib.ref_read_matrix_file(C.c_int(kind), path.encode(), C.byref(r), C.byref(c), C.byref(z), None, None, None))
    if kind == 0:
        ptr = np.zeros(c.value + 1, dtype=np.int64)
        idx = np.zeros(max(z.value, 1), dtype=np.int64)
        val = np.zeros(max(z.value, 1))
        _chk(lib.ref_read_matrix_file(C.c_int(kind), path.encode(), C.byref(r), C.byref(c), C.byref(z), _p(ptr),
                                      _p(idx), _p(val)))
        return r.value, c.value, ptr, idx[:z.value], val[:z.value]
    a = np.zeros((r.value, c.value), order="F")
    _chk(lib.ref_read_matrix_file(C.c_int(kind), path.encode(), C.byref(r), C.byref(c), C.byref(z), None, None,
                                  _p(a)))
    return a


def write_matrix_file(kind: int, path: str, rows: int, cols: int, ptr=None, idx=None, val=None) -> None:
    v = np.asfortranarray(val, dtype=np.float64)  # kept alive across the call
    _chk(load().ref_write_matrix_file(C.c_int(kind), path.encode(), C.c_int64(rows), C.c_int64(cols),
                                      _p(ptr), _p(idx), _p(v)))


def stream_blocks(kind: int, path: str, block_rows: int):
    """All blocks of the reference's MatrixMarket (0) / CSV (1) row-block stream as CSC tuples."""
    lib = load()
    out = []
    b = 0
    while True:
        cnt, r, c, z = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64(-1)
        _chk(lib.ref_stream_block(C.c_int(kind), path.encode(), C.c_int64(block_rows), C.c_int64(b), C.byref(cnt),
                                  C.byref(r), C.byref(c), C.byref(z), None, None, None))
        if b >= cnt.value:
            return out
        ptr = np.zeros(c.value + 1, dtype=np.int64)
        idx = np.zeros(max(z.value, 1), dtype=np.int64)
        val = np.zeros(max(z.value, 1))
        _chk(lib.ref_stream_block(C.c_int(kind), path.encode(), C.c_int64(block_rows), C.c_int64(b), C.byref(cnt),
                                  C.byref(r), C.byref(c), C.byref(z), _p(ptr), _p(idx), _p(val)))
        out.append((r.value, c.value, ptr, idx[:z.value], val[:z.value]))
        b += 1


def cpu_threads() -> int:
    return len(os.sched_getaffinity(0))


def save_map_file(path: str, method: int, k: int, l: int, n: int, seed: int, density: float, scale: float,
                  v: np.ndarray, sigma=None) -> None:
    """save_map_file (reducer.cpp:355-373) with V n x k."""
    v = np.asfortranarray(v, dtype=np.float64)
    s = None if sigma is None else np.ascontiguousarray(sigma, dtype=np.float64)
    _chk(load().ref_save_map_file(C.c_int(method), C.c_int64(k), C.c_int64(l), C.c_int64(n), C.c_uint64(seed),
                                  C.c_double(density), C.c_double(scale), _p(v), _p(s) if s is not None else None,
                                  path.encode()))


def load_map_file(path: str) -> dict:
    """load_map_file (reducer.cpp:375-412)."""
    k, l, n, seed = C.c_int64(), C.c_int64(), C.c_int64(), C.c_uint64()
    dens, sc, hs = C.c_double(), C.c_double(), C.c_int()
    args = [C.byref(k), C.byref(l), C.byref(n), C.byref(seed), C.byref(dens), C.byref(sc), C.byref(hs)]
    _chk(load().ref_load_map_file(path.encode(), *args, None, None))
    v = np.zeros((n.value, k.value), order="F")
    sig = np.zeros(k.value)
    _chk(load().ref_load_map_file(path.encode(), *args, _p(v), _p(sig)))
    return dict(k=k.value, l=l.value, n=n.value, seed=seed.value, density=dens.value, scale=sc.value,
                v=v, sigma=sig if hs.value else None)
