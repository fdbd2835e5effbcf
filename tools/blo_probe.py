"""Times the dense X W sketch of a very sparse Omega (LPCA_SPARSE_OMEGA=0) at a
configs[3]-shaped slice; LPCA_VERBOSE=1 reports whether W's lo plane is zero."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1709_07175_b200 as lp  # noqa: E402

ctx = lp.Context(0)
m, n, l, k = int(os.environ.get("ROWS", 200_000)), 16384, 300, 256
x = torch.empty((m, n), dtype=torch.float32, device="cuda")
lp.synth_lowrank(x, 0, 400, 0.98, 0.01, 1000, ctx=ctx)
c = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=k, l=l, power_iters=0,
                     projection=lp.ProjectionSpec(kind=lp.ProjectionKind.very_sparse, density=1 / 128, seed=11))
for i in range(3):
    t = lp.ReducerTimings()
    lp.reduce_lazy_spca(x, c, timings=t, ctx=ctx)
    print(f"sketch_pass {t.sketch_pass * 1e3:.2f} ms  f_pass {t.f_pass * 1e3:.2f} ms", flush=True)
