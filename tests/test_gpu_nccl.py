"""GPU: the library's NCCL path on one GPU. lpca_ctx_create_dist with world == 1
and an id builds a one-rank communicator, so every exchange of the fit (the Z
and F sums of Algorithm 4, reducer.cpp:300-335; SPCA's Grams; the streaming
stacks) still runs through ncclAllReduce on the library's stream: libnccl is
resolved next to torch's bundled copy, the communicator is created and
destroyed, and the collectives are ordered with the library's kernels. A
one-rank sum is the identity, so the maps and Y must equal the plain context's
bitwise. (The pool has one GPU: NCCL refuses two ranks on one device, so the
two-rank sequence runs through the caller-collective hook, test_gpu_dist.py.)"""
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_1709_07175_b200 as lp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests" / "helpers"))
from dist_cases import CASES, as_input, case_data, projection  # noqa: E402

pytestmark = pytest.mark.gpu

NAMES = sorted(n for n, c in CASES.items() if "error" not in c and "split" not in c)


@pytest.fixture(scope="module")
def nccl_ctx():
    c = lp.Context(0, 0, 1, lp.Context.nccl_unique_id())
    yield c
    c.close()


def _fit(ctx, name):
    c = CASES[name]
    x = case_data(name)
    cfg = lp.ReducerConfig(method=c["method"], k=c["k"], l=c["l"], projection=projection(c),
                           power_iters=c.get("q", 0))
    if c.get("stream"):
        fn = lp.reduce_spca_streaming if c["method"] == lp.ReducerMethod.spca else lp.reduce_lazy_spca_streaming
        return fn(lp.SliceRowBlockStream(x, c["block_rows"]), cfg, ctx=ctx), None
    if c.get("sparse"):
        return lp.fit_transform(as_input(c, x), cfg, ctx=ctx)
    mp, y = lp.fit_transform(torch.from_numpy(x).cuda(), cfg, ctx=ctx)
    return mp, y


@pytest.mark.parametrize("name", NAMES)
def test_one_rank_nccl_fit_equals_the_plain_context(ctx, nccl_ctx, name):
    a, ya = _fit(ctx, name)
    b, yb = _fit(nccl_ctx, name)
    assert np.array_equal(a.v, b.v), name
    assert np.array_equal(a.singular_values, b.singular_values), name
    if ya is not None:
        assert torch.equal(torch.as_tensor(ya).cpu(), torch.as_tensor(yb).cpu()), name

