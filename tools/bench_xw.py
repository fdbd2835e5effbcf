"""Times the fp32 sketch kernel (X W) alone for several W widths, to separate
MMA work (~ npad), W re-reads from L2 (~ npad) and X streaming (constant)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1709_07175_b200 as lp  # noqa: E402

ctx = lp.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
m, n = 1_000_000, 4096
x = torch.randn(m, n, device="cuda")
for w in [int(a) for a in sys.argv[1:]] or [16, 32, 48, 64, 112, 128, 224]:
    W = torch.randn(n, w, device="cuda", dtype=torch.float64)
    out = torch.empty((m, w), device="cuda")
    for _ in range(2):
        lp.sketch_f32(x, W, out, ctx=ctx)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        lp.sketch_f32(x, W, out, ctx=ctx)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    npad = (w + 15) // 16 * 16
    mma_ms = 12 * (128 * npad / 256) * (m / 128) * (n / 32) / 148 / 1.9e6
    print(f"w={w:4d} npad={npad:4d}: {ms:6.2f} ms  X {m*n*4/ms/1e6:6.0f} GB/s  "
          f"W-rereads {(m/128)*2*npad*n*4/ms/1e6:6.0f} GB/s  MMA floor {mma_ms:5.2f} ms")
