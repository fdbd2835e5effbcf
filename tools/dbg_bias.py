"""Debug: signed relative bias of the tcgen05 split-TF32 GEMMs vs fp64."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_1709_07175_b200 as lp  # noqa: E402

ctx = lp.Context(0)
torch.manual_seed(0)


def stats(out, ref):
    rel = (out - ref) / ref.abs().clamp_min(1e-30)
    signed = ((out - ref) * ref.sign()).sum() / ref.abs().sum()
    return f"signed bias {signed.item():+.3e}  rms rel {rel.pow(2).mean().sqrt().item():.3e}"


for n in (256, 1024, 4096):
    x = torch.randn(8192, n, device="cuda")
    w = torch.randn(n, 112, device="cuda", dtype=torch.float64)
    ref = x.double() @ w
    for path in ("simt", "tcgen05"):
        ctx.set_gemm_path(path)
        out = lp.sketch_f32(x, w, ctx=ctx).double()
        print(f"sketch K={n} {path}: {stats(out, ref)}")
for m in (1024, 8192, 65536):
    x = torch.randn(m, 1024, device="cuda")
    u = torch.randn(m, 112, device="cuda")
    ref = u.double().t() @ x.double()
    for path in ("simt", "tcgen05"):
        ctx.set_gemm_path(path)
        F = torch.empty((1024, 112), dtype=torch.float64, device="cuda")
        vw = lp.api._View(x)
        lp.api._check(ctx.lib.lpca_gemm_t_f32(ctx.h, C.c_void_p(u.data_ptr()), u.stride(0), 112, C.byref(vw.view),
                                              C.c_void_p(F.data_ptr())))
        print(f"gemm_t K={m} {path}: {stats(F.t(), ref)}")
