"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference Lazy SPCA path.

numpy restatement of the reference algorithms on the hot path, each function
citing the reference file:line it follows (paths relative to /root/reference).
It is pinned against the compiled reference (oracle/_ref, see refbind.py) and
against tests/golden/*.npz fixtures generated from it (tests/golden/make_golden.py).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import it;
the product (liblazypca_b200.so) never does.

Integer / byte work (splitmix64, xoshiro256**, the uniform mapping) is
restated bit-exactly with wrapping uint64 arrays; normal_icdf uses plain
float64 operations in the reference's order (no FMA) and C libm's log, so
Omega is bit-exact with the reference built with -ffp-contract=off. Floating
point linear algebra (GEMMs, eigensolve) is restated with numpy/LAPACK and
compared within tolerances.
"""
from __future__ import annotations

import math

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def _u(x) -> np.ndarray:
    return np.asarray(x, dtype=np.uint64)


# ---- rng.hpp:15-65 ------------------------------------------------------------
def splitmix64_next(state: np.ndarray):
    """splitmix64 (rng.hpp:16-21) on arrays: returns (new_state, output)."""
    with np.errstate(over="ignore"):
        state = _u(state) + GOLDEN
        z = state.copy()
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return state, z ^ (z >> np.uint64(31))


def mix64(z) -> np.ndarray:
    return splitmix64_next(_u(z))[1]


def _rotl(x: np.ndarray, k: int) -> np.ndarray:
    return (x << np.uint64(k)) | (x >> np.uint64(64 - k))


class Xoshiro256:
    """xoshiro256** (rng.hpp:29-56), vectorised over independent streams."""

    def __init__(self, seeds):
        sm = _u(seeds).copy()
        s = []
        for _ in range(4):
            sm, w = splitmix64_next(sm)
            s.append(w)
        self.s = s

    def next(self) -> np.ndarray:
        s0, s1, s2, s3 = self.s
        with np.errstate(over="ignore"):
            result = _rotl(s1 * np.uint64(5), 7) * np.uint64(9)
        t = s1 << np.uint64(17)
        s2 = s2 ^ s0
        s3 = s3 ^ s1
        s1 = s1 ^ s2
        s0 = s0 ^ s3
        s2 = s2 ^ t
        s3 = _rotl(s3, 45)
        self.s = [s0, s1, s2, s3]
        return result


def column_stream_seeds(seed: int, cols) -> np.ndarray:
    """column_stream (rng.hpp:61-65): derived seed for each column."""
    with np.errstate(over="ignore"):
        return mix64(mix64(_u(seed)) ^ (GOLDEN * (_u(cols) + np.uint64(1))))


def u64_to_uniform(bits: np.ndarray) -> np.ndarray:
    """Xoshiro256::uniform (rng.hpp:49-51)."""
    return ((bits >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


_A = (-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
      1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00)
_B = (-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
      6.680131188771972e+01, -1.328068155288572e+01)
_C = (-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
      -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00)
_D = (7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
      3.754408661907416e+00)
_P_LOW = 0.02425
_libm_log = np.frompyfunc(math.log, 1, 1)


def normal_icdf(p: np.ndarray, exact_log: bool = True) -> np.ndarray:
    """Acklam inverse normal CDF (rng.hpp:69-97), reference evaluation order.
    exact_log=False uses numpy's vectorised log (may differ by an ulp from libm)."""
    p = np.asarray(p, dtype=np.float64)
    out = np.empty_like(p)
    lo = p < _P_LOW
    hi = p > 1.0 - _P_LOW
    mid = ~(lo | hi)
    q = p[mid] - 0.5
    r = q * q
    num = ((((((_A[0] * r + _A[1]) * r + _A[2]) * r + _A[3]) * r + _A[4]) * r + _A[5]) * q)
    den = (((((_B[0] * r + _B[1]) * r + _B[2]) * r + _B[3]) * r + _B[4]) * r + 1.0)
    out[mid] = num / den
    for mask, arg, sign in ((lo, p[lo], 1.0), (hi, 1.0 - p[hi], -1.0)):
        if not mask.any():
            continue
        lg = _libm_log(arg).astype(np.float64) if exact_log else np.log(arg)
        q = np.sqrt(-2.0 * lg)
        num = (((((_C[0] * q + _C[1]) * q + _C[2]) * q + _C[3]) * q + _C[4]) * q + _C[5])
        den = ((((_D[0] * q + _D[1]) * q + _D[2]) * q + _D[3]) * q + 1.0)
        out[mask] = (sign * num) / den
    return out


def _column_draws(n: int, l: int, seed: int) -> np.ndarray:
    rng = Xoshiro256(column_stream_seeds(seed, np.arange(l, dtype=np.uint64)))
    bits = np.empty((n, l), dtype=np.uint64)
    for i in range(n):
        bits[i] = rng.next()
    return bits


def gen_gaussian(n: int, l: int, seed: int):
    """gen_gaussian (projection.cpp:71-84): Omega n x l, scale sqrt(l)."""
    _validate(n, l, 1.0)
    om = normal_icdf(u64_to_uniform(_column_draws(n, l, seed)))
    return np.asfortranarray(om), math.sqrt(l)


def gen_very_sparse(n: int, l: int, density: float, seed: int):
    """gen_very_sparse (projection.cpp:86-126): dense {-1,0,+1}, scale sqrt(l*d)."""
    _validate(n, l, density)
    u = u64_to_uniform(_column_draws(n, l, seed))
    half = density / 2.0
    om = np.where(u >= density, 0.0, np.where(u < half, 1.0, -1.0))
    return np.asfortranarray(om), math.sqrt(l * density)


def _validate(n, l, density):
    """ProjectionSpec::validate (projection.cpp:52-60)."""
    if l < 2:
        raise ValueError(f"projection: sketch width l must be at least 2, got {l}")
    if l > n:
        raise ValueError(f"projection: sketch width l = {l} exceeds data dimensionality n = {n}")
    if not (density > 0.0) or density > 1.0:
        raise ValueError("projection: density must lie in (0, 1]")


def density_for(mode: str, k: int, value: float = 0.0) -> float:
    """density_for (projection.cpp:38-50)."""
    if k < 2:
        raise ValueError("density policy: k must be at least 2")
    d = {"aggressive": math.log(k) / k, "conservative": 1.0 / math.sqrt(k)}.get(mode, value)
    return min(d, 1.0)


# ---- l x l step (truncated_svd.cpp:13-82) -----------------------------------------
class RankDeficiency(Exception):
    def __init__(self, safe: int):
        super().__init__(f"largest safe k = {safe}")
        self.safe = safe


def truncated_svd_via_gram(f: np.ndarray, k: int):
    """G = F F^T (dense_aat, kernels.cpp:148-172); eig descending; rank floor
    1e-12 * lambda_max; sigma = sqrt(lambda); V = F^T U~ / sigma; canonical signs."""
    lsz, n = f.shape
    if lsz > n:
        raise ValueError("F must be wide")
    g = f @ f.T
    lam, vec = np.linalg.eigh(g)
    order = np.argsort(-lam, kind="stable")
    lam, vec = lam[order], vec[:, order]
    floor = 1e-12 * max(lam[0], 0.0)
    safe = 0
    while safe < lsz and lam[safe] > floor and lam[safe] > 0.0:
        safe += 1
    if k > safe:
        raise RankDeficiency(safe)
    sig = np.sqrt(lam[:k])
    ut = vec[:, :k].copy()
    v = (f.T @ ut) / sig
    for r in range(k):  # truncated_svd.cpp:64-80
        arg = int(np.argmax(np.abs(v[:, r])))
        if v[arg, r] < 0.0:
            v[:, r] = -v[:, r]
            ut[:, r] = -ut[:, r]
    return sig, np.asfortranarray(v), ut


def orth(a: np.ndarray) -> np.ndarray:
    """householder_qr's Q with non-negative R diagonal (qr.cpp:84-132)."""
    q, r = np.linalg.qr(a)
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s


# ---- reducers (reducer.cpp:171-234) ------------------------------------------------
def omega_for(n, l, seed, kind="gaussian", density=1.0):
    if kind == "gaussian":
        return gen_gaussian(n, l, seed)
    return gen_very_sparse(n, l, density, seed)


def sketch(x: np.ndarray, om: np.ndarray, power_iters: int = 0) -> np.ndarray:
    """U = X Omega (reducer.cpp:163-169, kernels.cpp:30-47), then the builder's
    power scheme (not in the reference): Z = X^T U, Z <- orth(Z), U = X Z."""
    x = np.asarray(x, dtype=np.float64)
    u = x @ om
    for _ in range(power_iters):
        z = orth(x.T @ u)
        u = x @ z
    return u


def reduce_lazy_spca(x, k, l, seed, kind="gaussian", density=1.0, power_iters=0):
    """reduce_lazy_spca (reducer.cpp:216-234): F = U^T X, then truncated_svd_via_gram."""
    x = np.asarray(x, dtype=np.float64)
    om, scale = omega_for(x.shape[1], l, seed, kind, density)
    u = sketch(x, om, power_iters)
    f = u.T @ x
    sig, v, _ = truncated_svd_via_gram(f, k)
    return v, sig, scale


def reduce_spca(x, k, l, seed, kind="gaussian", density=1.0, power_iters=0):
    """reduce_spca (reducer.cpp:192-214): Q = qr(U), F = Q^T X."""
    x = np.asarray(x, dtype=np.float64)
    om, scale = omega_for(x.shape[1], l, seed, kind, density)
    q = orth(sketch(x, om, power_iters))
    sig, v, _ = truncated_svd_via_gram(q.T @ x, k)
    return v, sig, scale


def reduce_rp(n, k, seed, kind="gaussian", density=1.0):
    """reduce_rp (reducer.cpp:171-190): V = Omega / c."""
    om, scale = omega_for(n, k, seed, kind, density)
    return om * (1.0 / scale), scale


def apply_map(x, v):
    """apply_map (reducer.cpp:348-353)."""
    return np.asarray(x, dtype=np.float64) @ v


def reduce_lazy_spca_sharded(x_shards, k, l, seed, allreduce, power_iters=0):
    """Algorithm 4 (reducer.cpp:300-335) across ranks: each rank sketches its own
    rows, U_r^T X_r (and Z_r) partials are summed by `allreduce`, and the l x l
    step is replicated. Used by the world-size-2 gloo tests of the sharded host logic."""
    x = np.asarray(x_shards, dtype=np.float64)
    om, _ = gen_gaussian(x.shape[1], l, seed)
    u = x @ om
    for _ in range(power_iters):
        z = orth(allreduce(x.T @ u))
        u = x @ z
    f = allreduce(u.T @ x)
    sig, v, _ = truncated_svd_via_gram(f, k)
    return v, sig, u


def reduce_streaming(blocks, method, k, l, seed, kind="gaussian", density=1.0):
    """reduce_{lazy_spca,spca}_streaming (reducer.cpp:236-335): one pass over row
    blocks, F = sum_s U_s^T X_s (gemm_t_add); SPCA also keeps the stacked
    Householder R of [R; U_s] (householder_qr_r_only, qr.cpp:134-142) and ends
    with F <- R^{-T} F (solve_rt_in_place, reducer.cpp:55-73)."""
    blocks = [np.asarray(b, dtype=np.float64) for b in blocks]
    if not blocks:
        raise ValueError("streaming: the block stream is empty")
    n = blocks[0].shape[1]
    om, scale = omega_for(n, l, seed, kind, density)
    f = np.zeros((l, n))
    r = None
    for b in blocks:
        u = b @ om
        f += u.T @ b
        if method == "spca":
            stacked = u if r is None else np.vstack([r, u])
            r = np.linalg.qr(stacked, mode="r")
            sg = np.sign(np.diag(r))
            sg[sg == 0] = 1.0
            r = r * sg[:, None]
    if method == "spca":
        f = np.linalg.solve(r.T, f)
    sig, v, _ = truncated_svd_via_gram(f, k)
    return v, sig, scale


# ---- metrics used as checkers (metrics.cpp:100-136, 311-352) ------------------------
def chordal_distance(v1: np.ndarray, v2: np.ndarray) -> float:
    def res2(a, b):
        r = a - b @ (b.T @ a)
        return float((r * r).sum())
    return math.sqrt(res2(v1, v2) + res2(v2, v1))


def principal_angles(v1: np.ndarray, v2: np.ndarray) -> np.ndarray:
    """Principal angles between span(v1) and span(v2), ascending. Small angles
    come from the sines (singular values of (I - Q1 Q1^T) Q2), which keep full
    relative precision where arccos of the cosines bottoms out at sqrt(eps)."""
    q1, _ = np.linalg.qr(v1)
    q2, _ = np.linalg.qr(v2)
    cos = np.sort(np.clip(np.linalg.svd(q1.T @ q2, compute_uv=False), -1.0, 1.0))[::-1]
    sin = np.sort(np.clip(np.linalg.svd(q2 - q1 @ (q1.T @ q2), compute_uv=False), 0.0, 1.0))
    return np.where(cos > np.sqrt(0.5), np.arcsin(sin[: cos.size]), np.arccos(cos))


def pair_sample(m: int, max_pairs: int, seed: int):
    """distance_preservation's pair draw (metrics.cpp:327-334)."""
    rng = Xoshiro256(mix64(_u(seed) ^ np.uint64(0x9A17B0A155A3F2C1)).reshape(1))
    pairs = []
    while len(pairs) < max_pairs:
        i = int(rng.next()[0] % np.uint64(m))
        j = int(rng.next()[0] % np.uint64(m))
        if i == j:
            continue
        pairs.append((min(i, j), max(i, j)))
    return pairs


# ---- BASELINE synthetic generator (not in the reference) ----------------------------
def counter_normal(seed: int, idx: np.ndarray, exact_log: bool = True) -> np.ndarray:
    with np.errstate(over="ignore"):
        return normal_icdf(u64_to_uniform(mix64(_u(seed) ^ (_u(idx) * GOLDEN))), exact_log)


def synth_lowrank(row0: int, m: int, n: int, r: int, rho: float, noise: float, seed: int,
                  dtype=np.float64, exact_log: bool = True) -> np.ndarray:
    """X = G diag(rho^t) H + noise E, t = 0..r-1, counter-based N(0,1) factors
    keyed exactly like the device generator (csrc/omega.cu). Summation order is
    numpy's, so the result agrees with the device to rounding, not bitwise."""
    sig = np.empty(r)
    s = 1.0
    for t in range(r):
        sig[t] = s
        s *= rho
    rows = np.arange(row0, row0 + m, dtype=np.uint64)
    gi = rows[:, None] * np.uint64(r) + np.arange(r, dtype=np.uint64)[None, :]
    g = counter_normal(seed + 1001, gi, exact_log) * sig[None, :]
    h = counter_normal(seed + 1002, np.arange(r * n, dtype=np.uint64), exact_log).reshape(r, n)
    out = np.empty((m, n), dtype=dtype)
    for b0 in range(0, m, 4096):  # bounded temporaries
        b1 = min(m, b0 + 4096)
        ei = rows[b0:b1, None] * np.uint64(n) + np.arange(n, dtype=np.uint64)[None, :]
        out[b0:b1] = g[b0:b1] @ h + noise * counter_normal(seed + 1003, ei, exact_log)
    return out
