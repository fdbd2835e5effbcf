"""Python mirror of the reference `lazypca` API over the lazypca_b200 C ABI.

Names, argument meaning and error behaviour follow the reference headers
(proj/core/include/lazypca/{reducer,projection,kernels,truncated_svd,error}.hpp)
so the parity tests read like the reference's own doctest suites. Every compute
call goes through liblazypca_b200.so on the GPU; nothing here computes.

Matrix arguments may be numpy arrays (host; row-major or Fortran-ordered),
torch CUDA tensors (device, row-major), or SparseMatrix (the reference's CSC).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L


# ---- errors (proj/core/include/lazypca/error.hpp:10-58) ----------------------
class Error(RuntimeError):
    pass


class DimensionError(Error):
    pass


class InvalidArgumentError(Error):
    pass


class RankDeficiencyError(Error):
    def __init__(self, what: str, index: int = -1):
        super().__init__(what)
        self._index = index

    def index(self) -> int:
        return self._index


class ConvergenceError(Error):
    def __init__(self, what: str, last_gap: float = 0.0):
        super().__init__(what)
        self._gap = last_gap

    def last_gap(self) -> float:
        return self._gap


class ParseError(Error):
    def __init__(self, what: str, line: int = 0):
        super().__init__(what)
        self._line = line

    def line(self) -> int:
        return self._line


class CudaError(Error):
    """Device/driver failure (no reference analogue)."""


class NcclError(Error):
    """Collective failure (no reference analogue)."""


def _check(status: int) -> None:
    if status == 0:
        return
    lib = L.load()
    msg = (lib.lpca_last_error() or b"").decode(errors="replace")
    idx = int(lib.lpca_last_error_index())
    if status == 1:
        raise DimensionError(msg)
    if status == 2:
        raise InvalidArgumentError(msg)
    if status == 3:
        raise RankDeficiencyError(msg, idx)
    if status == 4:
        raise ConvergenceError(msg, float(lib.lpca_last_error_gap()))
    if status == 5:
        raise ParseError(msg, idx)
    if status == 6:
        raise CudaError(msg)
    if status == 7:
        raise NcclError(msg)
    raise Error(msg)


# ---- configuration ------------------------------------------------------------
class ReducerMethod(enum.IntEnum):
    rp = 0
    spca = 1
    lazy_spca = 2


def to_string(m) -> str:
    if isinstance(m, ReducerMethod):
        return m.name
    if isinstance(m, ProjectionKind):
        return m.name
    raise InvalidArgumentError(f"cannot name {m!r}")


def reducer_method_from_string(text: str) -> ReducerMethod:
    try:
        return ReducerMethod[text]
    except KeyError:
        raise InvalidArgumentError(
            f"unknown method '{text}' (expected rp, spca, or lazy_spca)") from None


class ProjectionKind(enum.IntEnum):
    gaussian = 0
    very_sparse = 1


def projection_kind_from_string(text: str) -> ProjectionKind:
    try:
        return ProjectionKind[text]
    except KeyError:
        raise InvalidArgumentError(f"unknown projection kind '{text}'") from None


@dataclass
class DensityPolicy:
    """proj/core/include/lazypca/projection.hpp:17-31."""
    mode: str = "conservative"
    value: float = 0.0

    @staticmethod
    def aggressive() -> "DensityPolicy":
        return DensityPolicy("aggressive")

    @staticmethod
    def conservative() -> "DensityPolicy":
        return DensityPolicy("conservative")

    @staticmethod
    def explicit_value(v: float) -> "DensityPolicy":
        return DensityPolicy("explicit_value", float(v))

    @staticmethod
    def parse(text: str) -> "DensityPolicy":
        if text == "aggressive":
            return DensityPolicy.aggressive()
        if text == "conservative":
            return DensityPolicy.conservative()
        if text.startswith("value:"):
            try:
                v = float(text[6:])
            except ValueError:
                raise InvalidArgumentError(f"density policy: cannot parse value in '{text}'") from None
            if not (v > 0.0) or v > 1.0:
                raise InvalidArgumentError(f"density policy: explicit value must lie in (0, 1], got {text[6:]}")
            return DensityPolicy.explicit_value(v)
        raise InvalidArgumentError("density policy: expected 'aggressive', 'conservative', or "
                                   f"'value:<float>', got '{text}'")

    def to_string(self) -> str:
        return self.mode if self.mode != "explicit_value" else f"value:{self.value:f}"


_MODE = {"aggressive": 0, "conservative": 1, "explicit_value": 2}


def density_for(policy: DensityPolicy, k: int) -> float:
    out = C.c_double()
    _check(L.load().lpca_density_for(_MODE[policy.mode], int(k), float(policy.value), C.byref(out)))
    return out.value


@dataclass
class ProjectionSpec:
    kind: ProjectionKind = ProjectionKind.gaussian
    n: int = 0
    l: int = 0
    density: float = 1.0
    seed: int = 0


@dataclass
class ReducerConfig:
    """proj/core/include/lazypca/reducer.hpp:20-33 (+ power_iters, an extension)."""
    method: ReducerMethod = ReducerMethod.spca
    k: int = 0
    l: int = 0
    projection: ProjectionSpec = field(default_factory=ProjectionSpec)
    block_rows: int = 0
    streaming: bool = False
    deterministic: bool = True
    power_iters: int = 0

    def _c(self) -> L.Config:
        c = L.Config()
        c.method = int(self.method)
        c.projection_kind = int(self.projection.kind)
        c.k, c.l = int(self.k), int(self.l)
        c.proj_n, c.proj_l = int(self.projection.n), int(self.projection.l)
        c.density = float(self.projection.density)
        c.seed = int(self.projection.seed) & 0xFFFFFFFFFFFFFFFF
        c.block_rows = int(self.block_rows)
        c.streaming = int(bool(self.streaming))
        c.deterministic = int(bool(self.deterministic))
        c.power_iters = int(self.power_iters)
        return c

    @staticmethod
    def _from_c(c: L.Config) -> "ReducerConfig":
        return ReducerConfig(ReducerMethod(c.method), c.k, c.l,
                             ProjectionSpec(ProjectionKind(c.projection_kind), c.proj_n, c.proj_l,
                                            c.density, c.seed),
                             c.block_rows, bool(c.streaming), bool(c.deterministic), c.power_iters)

    def resolved(self, data_cols: int) -> "ReducerConfig":
        out = L.Config()
        src = self._c()
        _check(L.load().lpca_config_resolve(C.byref(src), int(data_cols), C.byref(out)))
        return ReducerConfig._from_c(out)


@dataclass
class ReducerTimings:
    sketch: float = 0.0
    qr: float = 0.0
    f_form: float = 0.0
    svd: float = 0.0
    total: float = 0.0
    power: float = 0.0
    transform: float = 0.0
    h2d: float = 0.0
    d2h: float = 0.0
    sketch_pass: float = 0.0     # the X-pass kernels alone (extension)
    f_pass: float = 0.0
    transform_pass: float = 0.0
    power_pass: float = 0.0      # both X passes of every power step (first 8 steps)


def _fill_timings(t: Optional[ReducerTimings], c: L.Timings) -> None:
    if t is None:
        return
    for f, _ in L.Timings._fields_:
        setattr(t, f, getattr(t, f) + getattr(c, f))


# ---- data ----------------------------------------------------------------------
class SparseMatrix:
    """Canonical CSC (proj/core/include/lazypca/sparse_matrix.hpp:17-49), host memory."""

    def __init__(self, rows: int, cols: int, col_ptr, row_idx, values):
        self._rows, self._cols = int(rows), int(cols)
        self.col_ptr = np.ascontiguousarray(col_ptr, dtype=np.int64)
        self.row_idx = np.ascontiguousarray(row_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=np.float64)

    @staticmethod
    def from_csc(rows, cols, col_ptr, row_idx, values) -> "SparseMatrix":
        return SparseMatrix(rows, cols, col_ptr, row_idx, values)

    @staticmethod
    def from_dense(a: np.ndarray) -> "SparseMatrix":
        a = np.asarray(a, dtype=np.float64)
        rows, cols = a.shape
        nz = a.T != 0  # column-major scan
        counts = nz.sum(axis=1)
        col_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        r_idx = np.nonzero(nz)[1].astype(np.int64)
        vals = a.T[nz]
        return SparseMatrix(rows, cols, col_ptr, r_idx, vals)

    @staticmethod
    def from_triplets(rows, cols, entries) -> "SparseMatrix":
        d = np.zeros((rows, cols))
        for (i, j, v) in entries:
            if not (0 <= i < rows and 0 <= j < cols):
                raise DimensionError(f"triplet index ({i}, {j}) outside {rows}x{cols}")
            d[i, j] += v
        return SparseMatrix.from_dense(d)

    def rows(self) -> int:
        return self._rows

    def cols(self) -> int:
        return self._cols

    def nnz(self) -> int:
        return int(self.values.size)

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self._rows, self._cols))
        for j in range(self._cols):
            s, e = self.col_ptr[j], self.col_ptr[j + 1]
            d[self.row_idx[s:e], j] = self.values[s:e]
        return d


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class _View:
    """Builds an lpca_matrix_view for any accepted matrix and keeps it alive."""

    def __init__(self, x):
        v = L.MatrixView()
        self.keep = [x]
        if isinstance(x, SparseMatrix):
            v.dtype, v.layout, v.location = L.LPCA_F64, L.LPCA_CSC, L.LPCA_HOST
            v.rows, v.cols, v.ld = x.rows(), x.cols(), 0
            v.data = x.values.ctypes.data if x.values.size else None
            v.col_ptr = x.col_ptr.ctypes.data
            v.row_idx = x.row_idx.ctypes.data if x.row_idx.size else None
            v.nnz = x.nnz()
        elif _is_torch(x):
            import torch
            if x.dim() != 2:
                raise DimensionError("expected a 2-D tensor")
            if x.dtype not in (torch.float32, torch.float64):
                raise InvalidArgumentError("tensor dtype must be float32 or float64")
            if x.stride(1) != 1:
                x = x.contiguous()
                self.keep.append(x)
            v.dtype = L.LPCA_F32 if x.dtype == torch.float32 else L.LPCA_F64
            v.layout = L.LPCA_ROW_MAJOR
            v.location = L.LPCA_DEVICE if x.is_cuda else L.LPCA_HOST
            if x.is_cuda:
                # the library runs on its context's stream: make torch's pending
                # writes to x visible first (a no-op wait when the streams are one)
                torch.cuda.current_stream(x.device).synchronize()
            v.rows, v.cols, v.ld = x.shape[0], x.shape[1], x.stride(0) if x.shape[0] > 1 else x.shape[1]
            v.data = x.data_ptr() if x.numel() else None
        else:
            a = np.asarray(x)
            if a.ndim != 2:
                raise DimensionError("expected a 2-D matrix")
            if a.dtype not in (np.float32, np.float64):
                a = a.astype(np.float64)
            if not (a.flags.c_contiguous or a.flags.f_contiguous):
                a = np.ascontiguousarray(a)
            self.keep.append(a)
            v.dtype = L.LPCA_F32 if a.dtype == np.float32 else L.LPCA_F64
            if a.flags.c_contiguous:
                v.layout, v.ld = L.LPCA_ROW_MAJOR, a.shape[1]
            else:
                v.layout, v.ld = L.LPCA_COL_MAJOR, a.shape[0]
            v.location = L.LPCA_HOST
            v.rows, v.cols = a.shape
            v.data = a.ctypes.data if a.size else None
        self.view = v


# ---- context ---------------------------------------------------------------------
class Context:
    """One GPU (and optionally one rank of a row-sharded NCCL group)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        self.lib = L.load()
        h = C.c_void_p()
        if world > 1 or nccl_id is not None:  # (world 1 + id: a one-rank NCCL communicator)
            buf = C.create_string_buffer(bytes(nccl_id), 128)
            _check(self.lib.lpca_ctx_create_dist(device, rank, world, buf, C.byref(h)))
        else:
            _check(self.lib.lpca_ctx_create(device, C.byref(h)))
        self.h = h
        self.device, self.rank, self.world = device, rank, world

    @classmethod
    def hooked(cls, device: int, rank: int, world: int, allreduce) -> "Context":
        """A rank whose exchanges go through `allreduce(data_ptr, count, stream_ptr)`
        (in-place fp64 sum over ranks of `count` values at device address
        data_ptr, ordered on the CUDA stream stream_ptr) instead of NCCL
        (lpca_ctx_create_hooked). Exceptions in the callback fail the call."""
        self = cls.__new__(cls)
        self.lib = L.load()

        def tramp(_user, data, count, stream):
            try:
                allreduce(int(data or 0), int(count), int(stream or 0))
                return 0
            except Exception:  # reported as LPCA_ERR_NCCL by the library
                import traceback
                traceback.print_exc()
                return 1

        self._hook = L.ALLREDUCE_FN(tramp)  # kept alive with the context
        h = C.c_void_p()
        _check(self.lib.lpca_ctx_create_hooked(device, rank, world, self._hook, None, C.byref(h)))
        self.h = h
        self.device, self.rank, self.world = device, rank, world
        return self

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(L.load().lpca_nccl_unique_id(buf))
        return buf.raw

    def close(self) -> None:
        if self.h:
            self.lib.lpca_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int) -> None:
        _check(self.lib.lpca_ctx_set_stream(self.h, C.c_void_p(stream_ptr)))

    def synchronize(self) -> None:
        _check(self.lib.lpca_ctx_synchronize(self.h))

    def set_gemm_path(self, path: str) -> None:
        _check(self.lib.lpca_ctx_set_gemm_path(self.h, {"tcgen05": 0, "simt": 1}[path]))

    def set_eigensolver(self, method: str) -> None:
        _check(self.lib.lpca_ctx_set_eigensolver(self.h, {"tridiag": 0, "jacobi": 1}[method]))

    def set_exact_order(self, on: bool) -> None:
        _check(self.lib.lpca_ctx_set_exact_order(self.h, int(bool(on))))

    def launch_count(self) -> int:
        return int(self.lib.lpca_ctx_launch_count(self.h))


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def set_thread_count(n: int) -> None:
    """Accepted for API compatibility (threading.hpp:15); the GPU path has no host pool."""


def thread_count() -> int:
    return 0


# ---- maps ------------------------------------------------------------------------
class ReductionMap:
    """proj/core/include/lazypca/reducer.hpp:47-57, backed by a device-resident V."""

    def __init__(self, handle: C.c_void_p, ctx: Context):
        self._h = handle
        self._ctx = ctx
        info = L.MapInfo()
        _check(ctx.lib.lpca_map_info_get(handle, C.byref(info)))
        self.method = ReducerMethod(info.method).name
        self.k, self.l, self.n = info.k, info.l, info.n
        self.seed = info.seed
        self.density = info.density
        self.scale = info.scale
        self._has_sigma = bool(info.has_singular_values)
        self._v = None
        self._sigma = None

    @staticmethod
    def from_host(v: np.ndarray, method: str = "rp", singular_values=None, l: int = 0, seed: int = 0,
                  density: float = 1.0, scale: float = 1.0, ctx: Context | None = None) -> "ReductionMap":
        ctx = ctx or default_context()
        v = np.asfortranarray(np.asarray(v, dtype=np.float64))
        info = L.MapInfo()
        info.method = int(reducer_method_from_string(method))
        info.n, info.k = v.shape
        info.l = l or v.shape[1]
        info.seed, info.density, info.scale = seed, density, scale
        sig = None
        if singular_values is not None:
            sig = np.ascontiguousarray(singular_values, dtype=np.float64)
            info.has_singular_values = 1
        h = C.c_void_p()
        _check(ctx.lib.lpca_map_create(ctx.h, C.byref(info), v.ctypes.data if v.size else None,
                                       sig.ctypes.data if sig is not None else None, C.byref(h)))
        return ReductionMap(h, ctx)

    @property
    def v(self) -> np.ndarray:
        if self._v is None:
            out = np.zeros((self.n, self.k), dtype=np.float64, order="F")
            if out.size:
                _check(self._ctx.lib.lpca_map_copy_v(self._h, out.ctypes.data, L.LPCA_HOST))
            self._v = out
        return self._v

    @property
    def singular_values(self) -> np.ndarray:
        if self._sigma is None:
            out = np.zeros(self.k if self._has_sigma else 0, dtype=np.float64)
            if out.size:
                _check(self._ctx.lib.lpca_map_copy_sigma(self._h, out.ctypes.data))
            self._sigma = out
        return self._sigma

    def handle(self) -> C.c_void_p:
        return self._h

    def __del__(self):
        try:
            if self._h:
                self._ctx.lib.lpca_map_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass


# ---- reducers ----------------------------------------------------------------------
def _cfg_with(config: ReducerConfig, method: Optional[ReducerMethod]) -> ReducerConfig:
    if method is None:
        return config
    c = ReducerConfig(**{**config.__dict__})
    c.method = method
    return c


def _fit(x, config: ReducerConfig, timings, ctx) -> ReductionMap:
    ctx = ctx or default_context()
    vw = _View(x)
    cfg = config._c()
    t = L.Timings()
    h = C.c_void_p()
    _check(ctx.lib.lpca_fit(ctx.h, C.byref(cfg), C.byref(vw.view), C.byref(h), C.byref(t)))
    _fill_timings(timings, t)
    return ReductionMap(h, ctx)


# ---- verification metrics on the device (metrics.cpp) ------------------------------
def chordal_distance(v1, v2, ctx=None) -> float:
    """chordal_distance (metrics.cpp:123-136): subspace distance of two
    orthonormal n x k bases, cancellation-free residual form."""
    ctx = ctx or default_context()
    a = np.asfortranarray(v1, dtype=np.float64)
    b = np.asfortranarray(v2, dtype=np.float64)
    out = C.c_double()
    _check(ctx.lib.lpca_chordal_distance(ctx.h, a.ctypes.data if a.size else None, a.shape[0], a.shape[1],
                                         b.ctypes.data if b.size else None, b.shape[0], b.shape[1], L.LPCA_HOST,
                                         C.byref(out)))
    return out.value


@dataclass
class DistancePreservationReport:
    """metrics.hpp:51-65: sampled (i, j) pairs with original and reduced distances."""
    pair_i: np.ndarray
    pair_j: np.ndarray
    original: np.ndarray
    reduced_a: np.ndarray
    reduced_b: np.ndarray
    max_contraction_violation: float
    max_map_discrepancy: float


def distance_preservation(x, map_a: "ReductionMap", map_b: "ReductionMap" = None, max_pairs: int = 10000,
                          seed: int = 0, ctx=None) -> DistancePreservationReport:
    """distance_preservation (metrics.cpp:311-352), distances computed on the device."""
    ctx = ctx or map_a._ctx
    vw = _View(x)
    m = vw.view.rows
    cap = int(min(max_pairs, max(0, m * (m - 1) // 2))) if m * (m - 1) // 2 <= max_pairs else int(max_pairs)
    pi = np.zeros(max(cap, 1), dtype=np.int64)
    pj = np.zeros(max(cap, 1), dtype=np.int64)
    o, ra, rb = (np.zeros(max(cap, 1)) for _ in range(3))
    npairs, viol, gap = C.c_int64(), C.c_double(), C.c_double()
    _check(ctx.lib.lpca_distance_preservation(ctx.h, C.byref(vw.view), map_a.handle(),
                                              map_b.handle() if map_b is not None else None, int(max_pairs),
                                              int(seed) & 0xFFFFFFFFFFFFFFFF, C.byref(npairs), pi.ctypes.data,
                                              pj.ctypes.data, o.ctypes.data, ra.ctypes.data, rb.ctypes.data,
                                              C.byref(viol), C.byref(gap)))
    n = npairs.value
    return DistancePreservationReport(pi[:n], pj[:n], o[:n], ra[:n], rb[:n], viol.value, gap.value)


class ResidualRoute(enum.IntEnum):
    """metrics.hpp:28: the orthonormal-basis route (Q Q^T X) or the raw sketch (U (U^T U)^{-1} U^T X)."""
    qr = 0
    lazy = 1


def _f64_operand(a):
    """(pointer, location, shape, keepalive) of a column-major fp64 operand: a host
    array (copied Fortran-order) or a CUDA tensor (its transpose must be contiguous)."""
    if hasattr(a, "is_cuda") and a.is_cuda:
        import torch
        t = a.to(torch.float64)
        if not t.t().is_contiguous():
            t = t.t().contiguous().t()
        torch.cuda.synchronize()
        return C.c_void_p(t.data_ptr()), L.LPCA_DEVICE, tuple(t.shape), t
    h = np.asfortranarray(np.asarray(a, dtype=np.float64))
    return (h.ctypes.data if h.size else None), L.LPCA_HOST, h.shape, h


@dataclass
class ReconstructionErrorReport:
    """metrics.hpp:31-36. sigma_k_plus_1 / bound are None when not computed."""
    spectral_error: float
    frobenius_error: float
    sigma_k_plus_1: float = None
    bound: float = None


def _report(r) -> ReconstructionErrorReport:
    return ReconstructionErrorReport(r.spectral_error, r.frobenius_error,
                                     r.sigma_k_plus_1 if r.has_sigma_k_plus_1 else None,
                                     r.bound if r.has_bound else None)


def reconstruction_error(x, u, route: ResidualRoute, k: int, l: int, with_bound: bool = False,
                         densify_limit: int = 2000, ctx=None) -> ReconstructionErrorReport:
    """reconstruction_error (metrics.cpp:148-259) on the device: ||X - P X|| for P
    the projector onto range(U), U the m x l sketch (host array or CUDA tensor)."""
    ctx = ctx or default_context()
    vw = _View(x)
    ub, loc, shape, _keep = _f64_operand(u)
    out = L.ReconReport()
    _check(ctx.lib.lpca_reconstruction_error(ctx.h, C.byref(vw.view), ub, shape[0], shape[1], loc, int(route), int(k),
                                             int(l), int(bool(with_bound)), int(densify_limit), C.byref(out)))
    return _report(out)


def row_space_reconstruction_error(x, v, ctx=None) -> ReconstructionErrorReport:
    """row_space_reconstruction_error (metrics.cpp:261-308): ||X - X V V^T|| for an
    orthonormal V (n x k)."""
    ctx = ctx or default_context()
    vw = _View(x)
    vb, loc, shape, _keep = _f64_operand(v)
    out = L.ReconReport()
    _check(ctx.lib.lpca_row_space_reconstruction_error(ctx.h, C.byref(vw.view), vb, shape[0], shape[1], loc,
                                                       C.byref(out)))
    return _report(out)


def spectral_norm(x, ctx=None) -> float:
    """spectral_norm (spectral_norm.cpp:23-77): largest singular value of X by the
    reference's power iteration."""
    ctx = ctx or default_context()
    vw = _View(x)
    out = C.c_double()
    _check(ctx.lib.lpca_spectral_norm(ctx.h, C.byref(vw.view), C.byref(out)))
    return out.value


def bound_value(m: int, n: int, k: int, l: int, sigma_k_plus_1: float) -> float:
    """bound_value (metrics.cpp:136-146)."""
    out = C.c_double()
    _check(L.load().lpca_bound_value(int(m), int(n), int(k), int(l), float(sigma_k_plus_1), C.byref(out)))
    return out.value


# ---- matrix files (matrix_io.cpp), the reference's formats and bytes ---------------
def _read_file(fn, path: str):
    lib = L.load()
    h = C.c_void_p()
    _check(fn(str(path).encode(), C.byref(h)))
    try:
        rows, cols, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib.lpca_matrix_file_info(h, C.byref(rows), C.byref(cols), C.byref(nnz)))
        m, n, z = rows.value, cols.value, nnz.value
        if z >= 0:
            ptr = np.zeros(n + 1, dtype=np.int64)
            idx = np.zeros(max(z, 1), dtype=np.int64)
            val = np.zeros(max(z, 1))
            _check(lib.lpca_matrix_file_copy(h, ptr.ctypes.data, idx.ctypes.data, val.ctypes.data))
            return SparseMatrix(m, n, ptr, idx[:z], val[:z])
        a = np.zeros((m, n), order="F")
        _check(lib.lpca_matrix_file_copy(h, None, None, a.ctypes.data if a.size else None))
        return a
    finally:
        lib.lpca_matrix_file_free(h)


def read_sparse_matrix_market(path: str) -> SparseMatrix:
    """read_sparse_matrix_market_file (matrix_io.cpp:143-175)."""
    return _read_file(L.load().lpca_read_sparse_matrix_market, path)


def read_dense_matrix_market(path: str) -> np.ndarray:
    """read_dense_matrix_market_file (matrix_io.cpp:194-230), column-major."""
    return _read_file(L.load().lpca_read_dense_matrix_market, path)


def read_dense_csv(path: str) -> np.ndarray:
    """read_dense_csv_file (matrix_io.cpp:245-277)."""
    return _read_file(L.load().lpca_read_dense_csv, path)


def write_sparse_matrix_market(x: SparseMatrix, path: str) -> None:
    lib = L.load()
    _check(lib.lpca_write_sparse_matrix_market(str(path).encode(), x.rows(), x.cols(), x.col_ptr.ctypes.data,
                                               x.row_idx.ctypes.data if x.nnz() else None,
                                               x.values.ctypes.data if x.nnz() else None))


def write_dense_matrix_market(a, path: str) -> None:
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    _check(L.load().lpca_write_dense_matrix_market(str(path).encode(), a.shape[0], a.shape[1],
                                                   a.ctypes.data if a.size else None))


def write_dense_csv(a, path: str) -> None:
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    _check(L.load().lpca_write_dense_csv(str(path).encode(), a.shape[0], a.shape[1], a.ctypes.data if a.size else None))


# ---- map files (reducer.cpp:355-412), byte-compatible with the reference ----------
def save_map_file(map_: "ReductionMap", path: str) -> None:
    """save_map_file: one-line JSON header + V as a dense MatrixMarket array."""
    _check(map_._ctx.lib.lpca_map_save(map_.handle(), str(path).encode()))


def load_map_file(path: str, ctx=None) -> "ReductionMap":
    """load_map_file: a device map ready for apply_map."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    _check(ctx.lib.lpca_map_load(ctx.h, str(path).encode(), C.byref(h)))
    return ReductionMap(h, ctx)


def write_map_file(path: str, method: "ReducerMethod", v: np.ndarray, singular_values=None, l: int = 0,
                   seed: int = 0, density: float = 1.0, scale: float = 1.0) -> None:
    """The same file from host arrays (no GPU needed)."""
    v = np.asfortranarray(v, dtype=np.float64)
    info = L.MapInfo()
    info.method = int(method)
    info.n, info.k = v.shape
    info.l = l or v.shape[1]
    info.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    info.density, info.scale = float(density), float(scale)
    sig = None
    if singular_values is not None:
        sig = np.ascontiguousarray(singular_values, dtype=np.float64)
        info.has_singular_values = 1
    _check(L.load().lpca_map_file_write(str(path).encode(), C.byref(info), v.ctypes.data if v.size else None,
                                        sig.ctypes.data if sig is not None and sig.size else None))


def read_map_file(path: str) -> dict:
    """Host-side read: header fields, V (n x k) and the singular values (or None)."""
    info = L.MapInfo()
    _check(L.load().lpca_map_file_read(str(path).encode(), C.byref(info), None, 0, None))
    v = np.zeros((info.n, info.k), order="F")
    sig = np.zeros(info.k)
    _check(L.load().lpca_map_file_read(str(path).encode(), C.byref(info), v.ctypes.data if v.size else None,
                                       v.size, sig.ctypes.data if sig.size else None))
    return dict(method=ReducerMethod(info.method), k=info.k, l=info.l, n=info.n, seed=info.seed,
                density=info.density, scale=info.scale, v=v,
                singular_values=sig if info.has_singular_values else None)


# ---- streaming (reducer.cpp:236-335; sparse_matrix.hpp:53-79) --------------------
@dataclass
class RowBlock:
    """One row block of a stream (lazypca::RowBlock): any matrix _View accepts."""
    slice_index: int
    block: object


class RowBlockStream:
    """Pull-model block source (lazypca::RowBlockStream): next() returns the next
    RowBlock, or None at the end."""

    def next(self) -> Optional[RowBlock]:  # pragma: no cover - interface
        raise NotImplementedError



class _FileRowBlockStream(RowBlockStream):
    """A native row-block stream over a file; the streaming reducers drive it
    from C. next() also works from Python (a copy of the block)."""

    def __init__(self, opener, path: str, block_rows: int):
        self._lib = L.load()
        self._h = C.c_void_p()
        _check(opener(str(path).encode(), int(block_rows), C.byref(self._h)))

    def next(self):
        v = L.MatrixView()
        sl = C.c_int64()
        r = self._lib.lpca_file_stream_next(self._h, C.byref(v), C.byref(sl))
        if r < 0:
            _check(-r)
        if r == 0:
            return None
        m, n = v.rows, v.cols
        if v.layout == L.LPCA_CSC:
            i64 = C.POINTER(C.c_int64)
            ptr = np.ctypeslib.as_array(C.cast(v.col_ptr, i64), shape=(n + 1,)).copy()
            z = int(v.nnz)
            idx = (np.ctypeslib.as_array(C.cast(v.row_idx, i64), shape=(max(z, 1),))[:z].copy() if z
                   else np.zeros(0, np.int64))
            val = (np.ctypeslib.as_array(C.cast(v.data, C.POINTER(C.c_double)), shape=(max(z, 1),))[:z].copy()
                   if z else np.zeros(0))
            return RowBlock(int(sl.value), SparseMatrix(m, n, ptr, idx, val))
        a = np.ctypeslib.as_array(C.cast(v.data, C.POINTER(C.c_double)), shape=(m, n)).copy()
        return RowBlock(int(sl.value), a)

    def close(self) -> None:
        if self._h:
            self._lib.lpca_file_stream_close(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MatrixMarketRowBlockStream(_FileRowBlockStream):
    """MatrixMarketRowBlockStream (matrix_io.cpp:313-377): CSC row blocks of a
    coordinate file, one block resident."""

    def __init__(self, path: str, block_rows: int):
        super().__init__(L.load().lpca_open_matrix_market_stream, path, block_rows)


class CsvRowBlockStream(_FileRowBlockStream):
    """CsvRowBlockStream (matrix_io.cpp:379-443): row blocks of a CSV file (dense)."""

    def __init__(self, path: str, block_rows: int):
        super().__init__(L.load().lpca_open_csv_stream, path, block_rows)


class SliceRowBlockStream(RowBlockStream):
    """Lazy row partition of an in-memory matrix (sparse_matrix.cpp:125-139)."""

    def __init__(self, x, block_rows: int):
        if block_rows < 1:
            raise InvalidArgumentError("block_rows must be at least 1")
        self.x, self.block_rows, self.next_slice = x, int(block_rows), 0
        rows = x.rows() if isinstance(x, SparseMatrix) else x.shape[0]
        self.rows = rows
        self.slice_count = (rows + block_rows - 1) // block_rows

    def next(self) -> Optional[RowBlock]:
        if self.next_slice >= self.slice_count:
            return None
        lo = self.next_slice * self.block_rows
        hi = min(lo + self.block_rows, self.rows)
        if isinstance(self.x, SparseMatrix):
            blk = SparseMatrix.from_dense(self.x.to_dense()[lo:hi])
        else:
            blk = self.x[lo:hi]
        out = RowBlock(self.next_slice, blk)
        self.next_slice += 1
        return out


def split_rows(x, block_rows: int) -> list:
    s = SliceRowBlockStream(x, block_rows)
    out = []
    while (b := s.next()) is not None:
        out.append(b)
    return out


def _fit_stream(stream: RowBlockStream, config: ReducerConfig, timings, ctx) -> ReductionMap:
    ctx = ctx or default_context()
    if isinstance(stream, _FileRowBlockStream):  # native: no Python in the block loop
        cfg = config._c()
        t = L.Timings()
        h = C.c_void_p()
        nxt = C.cast(ctx.lib.lpca_file_stream_next, C.c_void_p)
        _check(ctx.lib.lpca_fit_stream(ctx.h, C.byref(cfg), nxt, stream._h, C.byref(h), C.byref(t)))
        _fill_timings(timings, t)
        return ReductionMap(h, ctx)
    keep = {}
    err = []

    def cb(_user, view_ptr, slice_ptr):
        try:
            keep.pop("v", None)  # the previous block may be released now
            b = stream.next()
            if b is None:
                return 0
            vw = _View(b.block)
            keep["v"] = vw
            view_ptr[0] = vw.view
            slice_ptr[0] = int(b.slice_index)
            return 1
        except Exception as e:  # surfaced after the C call returns
            err.append(e)
            return -1

    fn = L.NEXT_BLOCK_FN(cb)
    cfg = config._c()
    t = L.Timings()
    h = C.c_void_p()
    st = ctx.lib.lpca_fit_stream(ctx.h, C.byref(cfg), C.cast(fn, C.c_void_p), None, C.byref(h), C.byref(t))
    if err:
        raise err[0]
    _check(st)
    _fill_timings(timings, t)
    return ReductionMap(h, ctx)


def reduce_lazy_spca_streaming(stream: RowBlockStream, config: ReducerConfig,
                               timings: ReducerTimings | None = None, ctx=None) -> "ReductionMap":
    return _fit_stream(stream, _cfg_with(config, ReducerMethod.lazy_spca), timings, ctx)


def reduce_spca_streaming(stream: RowBlockStream, config: ReducerConfig,
                          timings: ReducerTimings | None = None, ctx=None) -> "ReductionMap":
    return _fit_stream(stream, _cfg_with(config, ReducerMethod.spca), timings, ctx)


def reduce_rp(x, config: ReducerConfig, timings: ReducerTimings | None = None, ctx=None):
    return _fit(x, _cfg_with(config, ReducerMethod.rp), timings, ctx)


def reduce_spca(x, config: ReducerConfig, timings: ReducerTimings | None = None, ctx=None):
    return _fit(x, _cfg_with(config, ReducerMethod.spca), timings, ctx)


def reduce_lazy_spca(x, config: ReducerConfig, timings: ReducerTimings | None = None, ctx=None):
    return _fit(x, _cfg_with(config, ReducerMethod.lazy_spca), timings, ctx)


def reduce(x, config: ReducerConfig, timings: ReducerTimings | None = None, ctx=None):
    return _fit(x, config, timings, ctx)


def _check_out(out, m: int, k: int, ctx) -> int:
    """Validates a caller's Y buffer (row-major m x k torch CUDA tensor on the
    context's device, fp32/fp64) and returns its leading dimension."""
    import torch
    if not isinstance(out, torch.Tensor):
        raise InvalidArgumentError("out must be a torch tensor")
    if out.dtype not in (torch.float32, torch.float64):
        raise InvalidArgumentError(f"out must be float32 or float64, got {out.dtype}")
    if not out.is_cuda or out.device.index != ctx.device:
        raise InvalidArgumentError(f"out must live on cuda:{ctx.device}, got {out.device}")
    if out.dim() != 2 or tuple(out.shape) != (m, k):
        raise DimensionError(f"out has shape {tuple(out.shape)}, expected ({m}, {k})")
    if m > 0 and k > 0 and (out.stride(1) != 1 or out.stride(0) < k):
        raise InvalidArgumentError("out must be row-major (stride(1) == 1, stride(0) >= k)")
    return max(out.stride(0), k)


def apply_map(map_: ReductionMap, x, out=None, layout: str = "col", timings=None, ctx=None):
    """Y = X V (reducer.cpp:348-353). Returns a column-major fp64 numpy array like
    the reference, unless `out` (a torch CUDA tensor, row-major) is given."""
    ctx = ctx or map_._ctx
    vw = _View(x)
    t = L.Timings()
    m = vw.view.rows
    if out is not None:
        import torch
        ldy = _check_out(out, m, map_.k, ctx)
        dt = L.LPCA_F32 if out.dtype == torch.float32 else L.LPCA_F64
        _check(ctx.lib.lpca_transform(ctx.h, map_.handle(), C.byref(vw.view), C.c_void_p(out.data_ptr()),
                                      dt, L.LPCA_ROW_MAJOR, L.LPCA_DEVICE, ldy, C.byref(t)))
        _fill_timings(timings, t)
        return out
    if layout == "col":
        y = np.zeros((m, map_.k), dtype=np.float64, order="F")
        lay = L.LPCA_COL_MAJOR
    else:
        y = np.zeros((m, map_.k), dtype=np.float64)
        lay = L.LPCA_ROW_MAJOR
    _check(ctx.lib.lpca_transform(ctx.h, map_.handle(), C.byref(vw.view), y.ctypes.data if y.size else None,
                                  L.LPCA_F64, lay, L.LPCA_HOST, 0, C.byref(t)))
    _fill_timings(timings, t)
    return y


def fit_transform(x, config: ReducerConfig, y_dtype=np.float64, timings=None, ctx=None, out=None):
    """fit then transform of the same X in one library call (one upload of a host
    X; on the device the transform is queued right behind the fit's spectral
    step). Y is a row-major host array, or `out` (a row-major torch CUDA tensor)."""
    ctx = ctx or default_context()
    vw = _View(x)
    cfg = config._c()
    t = L.Timings()
    h = C.c_void_p()
    if out is not None:
        import torch
        ldy = _check_out(out, vw.view.rows, config.k, ctx)
        dt = L.LPCA_F32 if out.dtype == torch.float32 else L.LPCA_F64
        _check(ctx.lib.lpca_fit_transform(ctx.h, C.byref(cfg), C.byref(vw.view), C.byref(h),
                                          C.c_void_p(out.data_ptr()), dt, L.LPCA_ROW_MAJOR, L.LPCA_DEVICE,
                                          ldy, C.byref(t)))
        _fill_timings(timings, t)
        return ReductionMap(h, ctx), out
    y = np.zeros((vw.view.rows, config.k), dtype=y_dtype)
    dt = L.LPCA_F32 if y.dtype == np.float32 else L.LPCA_F64
    _check(ctx.lib.lpca_fit_transform(ctx.h, C.byref(cfg), C.byref(vw.view), C.byref(h),
                                      y.ctypes.data if y.size else None, dt, L.LPCA_ROW_MAJOR,
                                      L.LPCA_HOST, 0, C.byref(t)))
    _fill_timings(timings, t)
    return ReductionMap(h, ctx), y


# ---- projection ----------------------------------------------------------------------
@dataclass
class ProjectionMatrix:
    spec: ProjectionSpec
    scale: float
    omega: np.ndarray  # dense n x l (very sparse: {-1,0,+1})

    def is_dense(self) -> bool:
        return self.spec.kind == ProjectionKind.gaussian

    def scaled_dense(self) -> np.ndarray:
        return self.omega * (1.0 / self.scale)


def regenerate(spec: ProjectionSpec, ctx=None) -> ProjectionMatrix:
    ctx = ctx or default_context()
    out = np.zeros((spec.n, spec.l), dtype=np.float64, order="F") if spec.n > 0 and spec.l > 0 else \
        np.zeros((max(spec.n, 0), max(spec.l, 0)), order="F")
    sc = C.c_double()
    _check(ctx.lib.lpca_regenerate(ctx.h, int(spec.kind), int(spec.n), int(spec.l), float(spec.density),
                                   int(spec.seed) & 0xFFFFFFFFFFFFFFFF,
                                   out.ctypes.data if out.size else None, L.LPCA_HOST, C.byref(sc)))
    return ProjectionMatrix(spec, sc.value, out)


def gen_gaussian(spec: ProjectionSpec, ctx=None) -> ProjectionMatrix:
    s = ProjectionSpec(**{**spec.__dict__})
    s.kind = ProjectionKind.gaussian
    return regenerate(s, ctx)


def gen_very_sparse(spec: ProjectionSpec, ctx=None) -> ProjectionMatrix:
    s = ProjectionSpec(**{**spec.__dict__})
    s.kind = ProjectionKind.very_sparse
    return regenerate(s, ctx)


@dataclass
class SketchMatrix:
    u: np.ndarray


def build_sketch(x, omega: ProjectionMatrix, ctx=None) -> SketchMatrix:
    n = omega.omega.shape[0]
    cols = x.cols() if isinstance(x, SparseMatrix) else x.shape[1]
    if cols != n:
        raise DimensionError(f"sketch: data has {cols} columns but the projection has {n} rows")
    return SketchMatrix(spmm(x, omega.omega, ctx))


# ---- kernel-level ------------------------------------------------------------------------
def spmm(x, w, ctx=None) -> np.ndarray:
    """spmm(X, W) in fp64, reference summation order (kernels.cpp:30-47)."""
    ctx = ctx or default_context()
    vw = _View(x)
    w = np.asfortranarray(np.asarray(w, dtype=np.float64))
    if w.shape[0] != vw.view.cols:
        raise DimensionError(f"spmm: inner dimensions differ ({vw.view.cols} vs {w.shape[0]})")
    out = np.zeros((vw.view.rows, w.shape[1]), order="F")
    _check(ctx.lib.lpca_spmm(ctx.h, C.byref(vw.view), w.ctypes.data if w.size else None, w.shape[1],
                             L.LPCA_HOST, out.ctypes.data if out.size else None, L.LPCA_HOST))
    return out


def gemm_t(u, x, ctx=None) -> np.ndarray:
    """gemm_t(U, X) = U^T X (kernels.cpp:70-113)."""
    ctx = ctx or default_context()
    u = np.asfortranarray(np.asarray(u, dtype=np.float64))
    vw = _View(x)
    out = np.zeros((u.shape[1], vw.view.cols), order="F")
    _check(ctx.lib.lpca_gemm_t(ctx.h, u.ctypes.data if u.size else None, u.shape[0], u.shape[1],
                               L.LPCA_HOST, C.byref(vw.view), out.ctypes.data if out.size else None,
                               L.LPCA_HOST))
    return out


def dense_aat(f, ctx=None) -> np.ndarray:
    ctx = ctx or default_context()
    f = np.asfortranarray(np.asarray(f, dtype=np.float64))
    out = np.zeros((f.shape[0], f.shape[0]), order="F")
    _check(ctx.lib.lpca_dense_aat(ctx.h, f.ctypes.data if f.size else None, f.shape[0], f.shape[1],
                                  L.LPCA_HOST, out.ctypes.data if out.size else None))
    return out


@dataclass
class EigenDecomposition:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray


def eigh(a, ctx=None, method: str = "tridiag") -> EigenDecomposition:
    """tridiag_eigh (default) or jacobi_eigh on the device: eigenvalues descending."""
    ctx = ctx or default_context()
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise DimensionError(f"eigh: matrix must be square, got {a.shape}")
    lsz = a.shape[0]
    ev = np.zeros(lsz)
    vec = np.zeros((lsz, lsz), order="F")
    fn = ctx.lib.lpca_eigh if method == "tridiag" else ctx.lib.lpca_eigh_jacobi
    _check(fn(ctx.h, a.ctypes.data if a.size else None, lsz, L.LPCA_HOST,
              ev.ctypes.data if lsz else None, vec.ctypes.data if lsz else None))
    return EigenDecomposition(ev, vec)


def tridiag_eigh(a, ctx=None) -> EigenDecomposition:
    return eigh(a, ctx, "tridiag")


def jacobi_eigh(a, ctx=None) -> EigenDecomposition:
    return eigh(a, ctx, "jacobi")


@dataclass
class TruncatedSVD:
    u_tilde: np.ndarray
    singular_values: np.ndarray
    v: np.ndarray


def truncated_svd_via_gram(f, k: int, ctx=None) -> TruncatedSVD:
    ctx = ctx or default_context()
    f = np.asfortranarray(np.asarray(f, dtype=np.float64))
    lsz, n = f.shape
    kk = max(int(k), 0)
    sig = np.zeros(max(kk, 1))
    v = np.zeros((n, kk), order="F")
    ut = np.zeros((lsz, kk), order="F")
    _check(ctx.lib.lpca_truncated_svd_via_gram(ctx.h, f.ctypes.data if f.size else None, lsz, n, int(k),
                                               L.LPCA_HOST, sig.ctypes.data,
                                               v.ctypes.data if v.size else None,
                                               ut.ctypes.data if ut.size else None))
    return TruncatedSVD(ut, sig[:kk], v)


def sketch_f32(x_dev, w_dev, out_dev=None, ctx=None):
    """OUT = X W for fp32 device X on the context's GEMM path (fp32-faithful).
    w_dev: fp64 CUDA tensor n x w (any strides; made column-major). Returns fp32 m x w."""
    import torch
    ctx = ctx or default_context()
    wc = w_dev.t().contiguous().t() if not w_dev.t().is_contiguous() else w_dev
    wc = wc.to(torch.float64)
    if out_dev is None:
        out_dev = torch.empty((x_dev.shape[0], w_dev.shape[1]), dtype=torch.float32, device=x_dev.device)
    vw = _View(x_dev)
    _check(ctx.lib.lpca_sketch_f32(ctx.h, C.byref(vw.view), C.c_void_p(wc.data_ptr()), w_dev.shape[1],
                                   C.c_void_p(out_dev.data_ptr()), out_dev.stride(0)))
    return out_dev


def gemm_t_f32(u_dev, x_dev, ctx=None):
    """F = U^T X (l x n, fp64) for fp32 device U (m x l row-major) and X."""
    import torch
    ctx = ctx or default_context()
    l = u_dev.shape[1]
    ld = u_dev.stride(0)
    f = torch.empty((x_dev.shape[1], l), dtype=torch.float64, device=x_dev.device)  # F^T row-major = F col-major
    vw = _View(x_dev)
    _check(ctx.lib.lpca_gemm_t_f32(ctx.h, C.c_void_p(u_dev.data_ptr()), ld, l, C.byref(vw.view),
                                   C.c_void_p(f.data_ptr())))
    return f.t()


def synth_lowrank(x_dev, row0: int, r: int, rho: float, noise: float = 0.01, seed: int = 1000,
                  ctx=None) -> None:
    """Fills a row-major CUDA tensor with rows [row0, row0+m) of the BASELINE
    generator X = G diag(rho^t) H + noise E (t = 0..r-1)."""
    import torch
    ctx = ctx or default_context()
    dt = 4 if x_dev.dtype == torch.float32 else 8
    _check(ctx.lib.lpca_synth_lowrank(ctx.h, int(row0), x_dev.shape[0], x_dev.shape[1], int(r), float(rho),
                                      float(noise), int(seed), dt, C.c_void_p(x_dev.data_ptr()),
                                      x_dev.stride(0)))
