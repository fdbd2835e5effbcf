"""Small invocations of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck): the fp32 tensor-core passes (sketch with the overflow
rerun, power step, F, transform), fp64 DMMA and SIMT passes, SPCA's
CholeskyQR3, the streaming reducer, the eigensolvers and the sparse path.
Usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1709_07175_b200 as lp  # noqa: E402

ctx = lp.Context(0)
M = lp.ReducerMethod


def cfg(method, k, l, q=0, **kw):
    return lp.ReducerConfig(method=method, k=k, l=l, power_iters=q, projection=lp.ProjectionSpec(seed=5, **kw))


# fp32, tensor-core pair kernels: l = 40 (two full A slots) and l = 220 (quarter slots), q = 1
for m, n, k, l in ((1000, 512, 16, 40), (600, 1024, 100, 220)):
    x = torch.empty((m, n), dtype=torch.float32, device="cuda")
    lp.synth_lowrank(x, 0, 30, 0.95, 0.01, 1000, ctx=ctx)
    y = torch.empty((m, k), dtype=torch.float32, device="cuda")
    lp.fit_transform(x, cfg(M.lazy_spca, k, l, q=1), ctx=ctx, out=y)
    lp.reduce_spca(x, cfg(M.spca, k, l), ctx=ctx)
# the overflow rerun
rng = np.random.default_rng(1)
xo = rng.standard_normal((512, 1024)).astype(np.float32) * 0.5
xo[:, :64] *= 1e-3
lp.reduce_lazy_spca(torch.from_numpy(xo).cuda(), cfg(M.lazy_spca, 8, 16), ctx=ctx)
# fp64: DMMA (l > 64) and SIMT passes, streaming SPCA
x64 = torch.empty((700, 300), dtype=torch.float64, device="cuda")
lp.synth_lowrank(x64, 0, 30, 0.95, 0.01, 1000, ctx=ctx)
lp.fit_transform(x64, cfg(M.lazy_spca, 40, 80, q=1), ctx=ctx)
lp.fit_transform(x64, cfg(M.lazy_spca, 8, 16), ctx=ctx)
lp.reduce_spca_streaming(lp.SliceRowBlockStream(x64.cpu().numpy(), 200), cfg(M.spca, 8, 16), ctx=ctx)
# eigensolvers at a cluster size (l > 128)
g = np.random.default_rng(2).standard_normal((160, 160))
lp.eigh(g + g.T, ctx=ctx)
lp.eigh(g + g.T, ctx=ctx, method="jacobi")
# sparse X (CSR / CSC gathers) and very sparse Omega
xs = lp.SparseMatrix.from_dense(np.where(rng.random((400, 300)) < 0.05, rng.standard_normal((400, 300)), 0.0))
lp.reduce_lazy_spca(xs, cfg(M.lazy_spca, 8, 16, kind=lp.ProjectionKind.very_sparse, density=0.1), ctx=ctx)
torch.cuda.synchronize()
print("sanitize run ok, kernels launched", ctx.launch_count())
