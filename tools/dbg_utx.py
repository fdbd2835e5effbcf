"""Debug: tcgen05 U^T X on structured inputs (where do ones land?)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1709_07175_b200 as lp  # noqa: E402

ctx = lp.Context(0)


def run(u, x, l):
    n = x.shape[1]
    F = torch.empty((n, l), dtype=torch.float64, device="cuda")
    vw = lp.api._View(x)
    lp.api._check(ctx.lib.lpca_gemm_t_f32(ctx.h, C.c_void_p(u.data_ptr()), u.stride(0), l, C.byref(vw.view),
                                          C.c_void_p(F.data_ptr())))
    return F.t().cpu().numpy()


m, n, l = 32, 256, 128
u = torch.zeros(m, l, device="cuda")
x = torch.zeros(m, n, device="cuda")
for i in range(m):
    u[i, i] = 1.0
    x[i, i * 2] = 1.0
f = run(u, x, l)
want = (u.double().t() @ x.double()).cpu().numpy()
print("nonzeros got (r, j):", np.argwhere(np.abs(f) > 0.5)[:40].tolist())
print("values", f[np.abs(f) > 0.5][:10])
print("nonzeros want:", np.argwhere(want > 0.5)[:40].tolist())
torch.manual_seed(0)
u = torch.randn(m, l, device="cuda")
x = torch.randn(m, n, device="cuda")
f = run(u, x, l)
want = (u.double().t() @ x.double()).cpu().numpy()
print("rand: max err", np.abs(f - want).max(), "f[0,:4]", f[0, :4], "want", want[0, :4])
