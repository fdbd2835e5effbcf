"""GPU: row-permutation invariance, the reference's reducer property
(proj/tests/test_reducer.cpp:234-260). Lazy SPCA, SPCA and the power step sum
over rows (Algorithm 4, reducer.cpp:300-335), so permuting X's rows permutes U
and Y and leaves F, sigma and V unchanged up to the summation order. fp64
(DMMA / SIMT passes): 1e-12. fp32 on the tensor-core passes, where a
permutation also changes which rows share a 512-row U^T scale block and a
2-SM pair tile: sigma within 5e-7 (measured 3e-8), V within 2e-6 rad
(1.3e-7), and Y's rows follow the permutation (5e-6 of max|Y|, 4.7e-7)."""
import numpy as np
import pytest
import torch

import paper_1709_07175_b200 as lp
from oracle import lazypca_oracle as O

pytestmark = pytest.mark.gpu


def _cfg(method, k, l, q=0):
    return lp.ReducerConfig(method=method, k=k, l=l, projection=lp.ProjectionSpec(seed=4), power_iters=q)


@pytest.mark.parametrize("method,q", [(lp.ReducerMethod.lazy_spca, 0), (lp.ReducerMethod.lazy_spca, 1),
                                      (lp.ReducerMethod.spca, 0)])
def test_fp64_fit_is_row_permutation_invariant(ctx, method, q):
    x = O.synth_lowrank(0, 4000, 300, 40, 0.93, 0.01, 8)
    perm = np.random.default_rng(2).permutation(x.shape[0])
    k, l = 10, 24
    a = lp.reduce(x, _cfg(method, k, l, q), ctx=ctx)
    b = lp.reduce(np.ascontiguousarray(x[perm]), _cfg(method, k, l, q), ctx=ctx)
    assert np.max(np.abs(a.singular_values - b.singular_values) / a.singular_values) < 1e-12
    assert np.max(O.principal_angles(a.v[:, :k // 2], b.v[:, :k // 2])) < 1e-10


def test_fp32_tensor_core_fit_transform_is_row_permutation_invariant(ctx):
    m, n, k, l = 20000, 1024, 16, 24
    x = torch.empty((m, n), dtype=torch.float32, device="cuda")
    lp.synth_lowrank(x, 0, 60, 0.95, 0.01, 77, ctx=ctx)
    perm = torch.from_numpy(np.random.default_rng(3).permutation(m)).cuda()
    cfg = _cfg(lp.ReducerMethod.lazy_spca, k, l, q=1)
    a, ya = lp.fit_transform(x, cfg, ctx=ctx)
    b, yb = lp.fit_transform(x[perm].contiguous(), cfg, ctx=ctx)
    rel = np.max(np.abs(a.singular_values - b.singular_values) / a.singular_values)
    ang = np.max(O.principal_angles(a.v[:, :k // 2], b.v[:, :k // 2]))
    print(f"fp32 permutation: sigma {rel:.1e}, angles {ang:.1e}")
    assert rel < 5e-7, rel  # measured 3.2e-8
    assert ang < 2e-6, ang  # measured 1.3e-7
    # Y's rows follow the permutation (up to V's own difference and fp32 rounding)
    ya, yb = torch.as_tensor(ya).cpu().numpy(), torch.as_tensor(yb).cpu().numpy()
    s = np.sign(np.sum(a.v[:, :k // 2] * b.v[:, :k // 2], axis=0))  # canonical signs agree
    assert np.all(s == 1.0)
    diff = np.abs(yb[:, :k // 2] - ya[perm.cpu().numpy(), :k // 2]).max()
    print(f"fp32 permutation: Y {diff / np.abs(ya[:, :k // 2]).max():.1e}")
    assert diff < 5e-6 * np.abs(ya[:, :k // 2]).max(), diff  # measured 4.7e-7
