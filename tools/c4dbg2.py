import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_1709_07175_b200 as lp
ctx = lp.Context(0)
import os
m, n, r = 20000, int(os.environ.get('N', '4096')), 300
x32 = torch.empty((m, n), dtype=torch.float32, device="cuda")
lp.synth_lowrank(x32, 0, r, 0.98, 0.01, 1000, ctx=ctx)
out = []
for (k, l, q) in [(int(a), int(b), int(c)) for a, b, c in (s.split(",") for s in sys.argv[1:])]:
    cfg = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=k, l=l, projection=lp.ProjectionSpec(kind=lp.ProjectionKind.very_sparse if os.environ.get('VS') else lp.ProjectionKind.gaussian, density=1/128, seed=7), power_iters=q)
    try:
        m32 = lp.reduce_lazy_spca(x32, cfg, ctx=ctx)
        out.append("k%d l%d q%d %.4e" % (k, l, q, m32.singular_values[0]))
        del m32
    except Exception as e:
        out.append("ERR " + str(e)[:40])
print(" | ".join(out), flush=True)
