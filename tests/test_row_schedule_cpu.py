"""CPU: the row gather's entry schedule (csrc/sparse_omega.cu build_row_schedule,
exported as lpca_debug_row_schedule). For a very sparse Omega pattern, every
warp's schedule must (a) hand each lane (Omega column) each of its nonzeros
exactly once with its sign, (b) read 32 distinct shared-memory banks at every
step (one wavefront), (c) send idle lanes to zero words, and (d) take exactly
the maximum degree of the warp's lane x bank multigraph steps (Koenig)."""
import ctypes as C

import numpy as np
import pytest

from paper_1709_07175_b200 import _lib as L


def _pattern(n, l, density, seed):
    rng = np.random.default_rng(seed)
    u = rng.random((l, n))
    sign = np.where(u < density / 2, -1, np.where(u < density, 1, 0))
    return sign  # [column][j] in {-1, 0, 1}


def _schedule(sign, cap=193):
    l, n = sign.shape
    cnt = np.zeros(l, dtype=np.int32)
    cols = np.zeros((l, cap), dtype=np.uint32)
    for c in range(l):
        js = np.nonzero(sign[c])[0]
        cnt[c] = len(js)
        k = min(len(js), cap)
        cols[c, :k] = js[:k].astype(np.uint32) | np.where(sign[c, js[:k]] < 0, 0x80000000, 0).astype(np.uint32)
    warps = 2 * ((l + 31) // 32)
    out = np.zeros(warps * 96 * 32, dtype=np.uint32)
    smax, splits = C.c_int32(), C.c_int32()
    steps = L.load().lpca_debug_row_schedule(cnt.ctypes.data, cols.ctypes.data, cap, n, l, out.ctypes.data,
                                             out.size, C.byref(smax), C.byref(splits))
    return steps, smax.value, splits.value, out, cnt


@pytest.mark.parametrize("n,l,density,seed", [
    (16384, 300, 1 / 128, 1),   # configs[3]
    (4096, 110, 1 / 64, 2),
    (1000, 37, 0.05, 3),        # ragged warps, n not a multiple of 32
    (2048, 64, 1 / 45, 4),
])
def test_schedule_is_complete_conflict_free_and_optimal(n, l, density, seed):
    sign = _pattern(n, l, density, seed)
    steps, smax, splits, out, cnt = _schedule(sign)
    assert steps > 0 and smax in (64, 96, 128, 192) and splits in (1, 2) and steps <= smax
    npad = (n + 31) // 32 * 32
    half = ((n + 1) // 2 + 31) // 32 * 32   # split point of a row's entries (splits == 2)
    wps = (l + 31) // 32
    warps = wps * splits
    words = out[:warps * (smax // 2) * 32].reshape(warps, smax // 2, 32)
    codes = np.empty((warps, smax, 32), dtype=np.uint32)   # [warp][step][lane]
    codes[:, 0::2, :] = words & 0xFFFF
    codes[:, 1::2, :] = words >> 16
    worst = 0
    for w in range(warps):
        part, g = divmod(w, wps)
        idx = codes[w] & 0x7FFF
        sg = codes[w] >> 15
        for s in range(smax):
            assert len(set((idx[s] % 32).tolist())) == 32   # one wavefront per step
        banks = np.zeros(32, dtype=int)
        degs = []
        for lane in range(32):
            c = 32 * g + lane
            real = idx[:, lane] < npad
            assert np.all(idx[~real, lane] < npad + 32) and np.all(sg[~real, lane] == 0)
            got = sorted(zip(idx[real, lane].tolist(), sg[real, lane].tolist()))
            if c < l:
                js = np.nonzero(sign[c])[0]
                if splits == 2:
                    js = js[(js < half) if part == 0 else (js >= half)]
                want = sorted(zip(js.tolist(), (sign[c, js] < 0).astype(int).tolist()))
                banks += np.bincount(js % 32, minlength=32)
                degs.append(len(js))
            else:
                want = []
            assert got == want
        delta = max(max(degs, default=0), int(banks.max()))
        worst = max(worst, delta)
    assert steps == worst


def test_schedule_infeasible_when_a_column_is_too_long():
    sign = _pattern(4096, 40, 0.2, 5)   # ~820 entries per column
    steps, smax, splits, _, _ = _schedule(sign)
    assert steps == -1 and smax == 0 and splits == 0
