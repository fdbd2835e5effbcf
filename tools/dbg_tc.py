"""Debug: tcgen05 sketch / gemm_t on small shapes vs float64 numpy."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1709_07175_b200 as lp

ctx = lp.Context(0)
torch.manual_seed(0)
for (m, n, w) in [(128, 32, 16), (256, 64, 16), (300, 100, 37), (1000, 256, 112)]:
    x = torch.randn(m, n, device="cuda", dtype=torch.float32)
    W = torch.randn(n, w, device="cuda", dtype=torch.float64)
    for path in ("simt", "tcgen05"):
        ctx.set_gemm_path(path)
        out = lp.sketch_f32(x, W, ctx=ctx)
        ref = x.double() @ W
        err = (out.double() - ref).abs()
        print(f"sketch m={m} n={n} w={w} {path}: max err {err.max().item():.3e} ref max {ref.abs().max().item():.2f}")
        if err.max() > 1e-3:
            bad = (err > 1e-3).nonzero()
            print("  bad rows", bad[:, 0].unique()[:20].tolist(), "cols", bad[:, 1].unique()[:20].tolist())
            print("  out[0,:8]", out[0, :8].tolist()); print("  ref[0,:8]", ref[0, :8].tolist())
    for l in (16, 37, 112, 200):
        u = torch.randn(m, (l + 15) // 16 * 16, device="cuda", dtype=torch.float32)
        u[:, l:] = 0
        for path in ("simt", "tcgen05"):
            ctx.set_gemm_path(path)
            try:
                f = lp.gemm_t_f32(u[:, :], x, ctx=ctx) if False else None
                fl = torch.empty(0)
                f = lp.api.gemm_t_f32(u, x, ctx=ctx)[:l] if False else None
            except Exception as e:
                print("err", e)
            from paper_1709_07175_b200 import _lib as L
            import ctypes as C
            F = torch.empty((n, l), dtype=torch.float64, device="cuda")
            vw = lp.api._View(x)
            lp.api._check(ctx.lib.lpca_gemm_t_f32(ctx.h, C.c_void_p(u.data_ptr()), u.stride(0), l, C.byref(vw.view), C.c_void_p(F.data_ptr())))
            Fm = F.t()  # l x n
            ref = u[:, :l].double().t() @ x.double()
            err = (Fm - ref).abs()
            print(f"  gemm_t m={m} n={n} l={l} {path}: max err {err.max().item():.3e} ref max {ref.abs().max().item():.2f}")
            if err.max() > 1e-3:
                bad = (err > 1e-3).nonzero()
                print("    bad r", bad[:, 0].unique()[:20].tolist(), "j", bad[:, 1].unique()[:20].tolist())
