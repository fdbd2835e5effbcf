"""Times the device eigensolver on Gram matrices shaped like the fit's G = F F^T."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1709_07175_b200 as lp  # noqa: E402

os.environ.setdefault("LPCA_VERBOSE", "1")
ctx = lp.Context(0)
rng = np.random.default_rng(0)
for l, n, rho in [(20, 1000, 0.9), (110, 4096, 0.97), (220, 4096, 0.98), (300, 16384, 0.98), (512, 2048, 0.99)]:
    # F = Omega^T X^T X-like: singular values ~ (rho^t)^2 scaled, random bases
    s = (rho ** np.arange(l)) ** 2 * 1e6 + 1e-3
    a, _ = np.linalg.qr(rng.standard_normal((l, l)))
    b, _ = np.linalg.qr(rng.standard_normal((n, l)))
    f = (a * s) @ b.T
    g = f @ f.T
    g = (g + g.T) / 2
    for method in ("tridiag", "jacobi") if l <= 220 else ("tridiag",):
        lp.eigh(g, ctx, method)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e = lp.eigh(g, ctx, method)
        dt = time.perf_counter() - t0
        w = np.linalg.eigvalsh(g)[::-1]
        err = np.max(np.abs(e.eigenvalues - w)) / w[0]
        orth = np.linalg.norm(e.eigenvectors.T @ e.eigenvectors - np.eye(l))
        print(f"l={l} {method}: {dt*1e3:.2f} ms  max|dlam|/lam0 = {err:.2e}  orth {orth:.1e}")
