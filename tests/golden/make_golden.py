"""Generates tests/golden/*.npz from the compiled reference (oracle/_ref).

Run here, where /root/reference exists:  python tests/golden/make_golden.py
The fixtures are small, committed, and travel to the GPU box, which has no
reference sources. Every array below comes out of the unmodified reference
core through oracle/ref_capi.cpp; inputs are seeded and regenerated
deterministically from the numpy restatement's counter-based generator.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import lazypca_oracle as O  # noqa: E402
from oracle import refbind as R  # noqa: E402

OUT = Path(__file__).resolve().parent


def main() -> None:
    R.build_if_possible()
    # Omega bit patterns (projection.cpp:71-126)
    omega = {}
    for (kind, n, l, d, seed) in [(0, 1000, 20, 1.0, 7), (0, 4096, 8, 1.0, 123456789),
                                  (0, 257, 5, 1.0, 0), (1, 16384, 4, 1.0 / 128, 7),
                                  (1, 500, 30, 0.1, 99)]:
        om, sc = R.regenerate(kind, n, l, d, seed)
        omega[f"k{kind}_n{n}_l{l}_s{seed}"] = om
        omega[f"k{kind}_n{n}_l{l}_s{seed}_scale"] = np.array(sc)
        omega[f"k{kind}_n{n}_l{l}_s{seed}_density"] = np.array(d)
    np.savez_compressed(OUT / "omega.npz", **omega)

    # Reducers on a small c1-shaped problem (reducer.cpp:171-234, 348-353)
    x = O.synth_lowrank(0, 600, 120, 12, 0.9, 0.01, 1000)
    red = {"x": x}
    for method, name in [(0, "rp"), (1, "spca"), (2, "lazy_spca")]:
        k, l = (8, 8) if method == 0 else (6, 10)
        v, sig, sc, _ = R.reduce(method, x, k, l, 7)
        red[f"{name}_v"] = v
        red[f"{name}_sigma"] = sig
        red[f"{name}_scale"] = np.array(sc)
        red[f"{name}_y"] = R.apply_map(x, v)
    # kernel level (kernels.cpp): spmm, gemm_t, dense_aat
    om, _ = R.regenerate(0, 120, 10, 1.0, 7)
    u = R.spmm(x, om)
    red["u"] = u
    red["f"] = R.gemm_t(u, x)
    red["g"] = R.dense_aat(red["f"])
    sig, v, ut = R.truncated_svd(red["f"], 6)
    red["tsvd_sigma"], red["tsvd_v"], red["tsvd_ut"] = sig, v, ut
    np.savez_compressed(OUT / "reducers.npz", **red)

    # Known-answer tests restated from the reference's doctest suites
    kat = {}
    # test_reducer.cpp:118-135: diag(5,4,3,2,1), exact sketch -> sigma (5, 4), v = e1, e2
    xd = np.diag([5.0, 4.0, 3.0, 2.0, 1.0])
    om = np.zeros((5, 2))
    om[0, 0] = om[1, 1] = 1.0
    q, _ = R.householder_qr(R.spmm(xd, om))
    sig, v, _ = R.truncated_svd(R.gemm_t(q, xd), 2)
    kat["diag_sigma"], kat["diag_v"] = sig, v
    # test_linalg.cpp:177-208 style: eigenvalues 4, 2, -1 and a repeated pair 3, 3
    rng = np.random.default_rng(5)
    qq, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    a = qq @ np.diag([4.0, 2.0, -1.0]) @ qq.T
    a = (a + a.T) / 2
    ev, vec = R.eigh(a)
    kat["eig3_a"], kat["eig3_ev"] = a, ev
    qq, _ = np.linalg.qr(rng.standard_normal((4, 4)))
    b = qq @ np.diag([3.0, 3.0, 1.0, -2.0]) @ qq.T
    b = (b + b.T) / 2
    kat["eig4_a"], kat["eig4_ev"] = b, R.eigh(b)[0]
    kat["density_aggr_100"] = np.array(R.density_for(0, 100))
    kat["density_cons_100"] = np.array(R.density_for(1, 100))
    np.savez_compressed(OUT / "kat.npz", **kat)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
