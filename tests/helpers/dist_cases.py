"""Cases of the world-size-2 library test (tests/test_gpu_dist.py), shared by
the rank processes and the single-process reference run."""
import numpy as np

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

M = lp.ReducerMethod
CASES = {
    # fp64 data: the fit on 2 ranks must equal the single-process fit to 1e-12
    "lazy_q0": dict(method=M.lazy_spca, k=8, l=16, m=3000, n=300, dtype="f64"),
    "lazy_q1": dict(method=M.lazy_spca, k=8, l=16, q=1, m=3000, n=300, dtype="f64"),
    "spca": dict(method=M.spca, k=8, l=16, m=3000, n=300, dtype="f64"),
    # rank 1 holds no rows at all
    "lazy_empty_shard": dict(method=M.lazy_spca, k=8, l=16, m=3000, n=300, dtype="f64", split="all_on_0"),
    # fp32 data on the tensor-core path, built to trip the sketch's overflow rerun
    "lazy_f32_rerun": dict(method=M.lazy_spca, k=16, l=32, m=8192, n=2048, dtype="f32", overflow=True),
    # fp32, a very sparse Omega on long rows: the row gather on each rank
    "lazy_f32_row_gather": dict(method=M.lazy_spca, k=16, l=40, q=1, m=4096, n=9000, dtype="f32",
                                very_sparse=1.0 / 90),
    # sparse X (CSC, the device-staged CSR/CSC path) on each rank; the second
    # with a very sparse Omega (the sign-mask sketch)
    "sparse_lazy_q1": dict(method=M.lazy_spca, k=8, l=16, q=1, m=3000, n=300, dtype="f64", sparse=0.05),
    "sparse_lazy_vs_omega": dict(method=M.lazy_spca, k=8, l=16, m=3000, n=300, dtype="f64", sparse=0.05,
                                 very_sparse=1.0 / 17),
    # streaming reducers (Algorithms 4 and 3) over each rank's blocks
    "stream_lazy": dict(method=M.lazy_spca, k=8, l=16, m=3000, n=300, dtype="f64", stream=True, block_rows=700),
    "stream_spca": dict(method=M.spca, k=8, l=16, m=3000, n=300, dtype="f64", stream=True, block_rows=700),
    "stream_spca_empty": dict(method=M.spca, k=8, l=16, m=3000, n=300, dtype="f64", stream=True, block_rows=700,
                              split="all_on_0"),
    # rank 1's shard has one column fewer: both ranks raise DimensionError (no rank left waiting)
    "n_mismatch": dict(method=M.lazy_spca, k=8, l=16, m=3000, n=300, dtype="f64", drop_col_on=1, error="DimensionError"),
    "stream_n_mismatch": dict(method=M.spca, k=8, l=16, m=3000, n=300, dtype="f64", stream=True, block_rows=700,
                              drop_col_on=1, error="DimensionError"),
}


def case_data(name):
    c = CASES[name]
    if c.get("overflow"):
        rng = np.random.default_rng(11)
        x = rng.standard_normal((c["m"], c["n"])).astype(np.float32) * 0.5
        for c0 in range(0, c["n"], 512):
            x[:, c0:c0 + 64] = rng.standard_normal((c["m"], 64)).astype(np.float32) * 1e-3
        return x
    dt = np.float32 if c["dtype"] == "f32" else np.float64
    x = O.synth_lowrank(0, c["m"], c["n"], 30, 0.93, 0.01, 17, dtype=dt)
    if c.get("sparse"):
        x = x * (np.random.default_rng(19).random(x.shape) < c["sparse"])
    return x


def as_input(c, x):
    """The case's X as the reducers take it: a CSC SparseMatrix for sparse cases."""
    return lp.SparseMatrix.from_dense(x) if c.get("sparse") else x


def shard(c, m, world, rank):
    if c.get("split") == "all_on_0":
        return (0, m) if rank == 0 else (m, m)
    per = -(-m // world)
    lo = min(m, rank * per)
    return lo, min(m, lo + per)


def projection(c):
    """The case's Omega: Gaussian, or very sparse at the case's density."""
    if c.get("very_sparse"):
        return lp.ProjectionSpec(kind=lp.ProjectionKind.very_sparse, density=c["very_sparse"], seed=5)
    return lp.ProjectionSpec(seed=5)
