"""One rank of the world-size-2 library test (tests/test_gpu_dist.py): runs the
library's own sharded reducers (lpca_fit / lpca_fit_transform / lpca_fit_stream
with world = 2) on cuda:0, with a gloo allreduce behind lpca_ctx_create_hooked
in place of NCCL, and saves every map it produced.
Usage: python tests/helpers/dist_rank.py RANK WORLD PORT OUT_DIR"""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_1709_07175_b200 as lp  # noqa: E402
from cuda.bindings import runtime as cudart  # noqa: E402

sys.path.insert(0, str(ROOT / "tests" / "helpers"))
from dist_cases import CASES, as_input, case_data, projection, shard  # noqa: E402


def main():
    rank, world, port, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), Path(sys.argv[4])
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import datetime
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=120))
    torch.cuda.set_device(0)
    calls = [0]

    def allreduce(ptr, count, stream):
        calls[0] += 1
        if os.environ.get("LPCA_DIST_TRACE"):
            print(f"rank {rank}: allreduce #{calls[0]} count {count}", flush=True)
        torch.cuda.ExternalStream(stream).synchronize()  # the library's (non-blocking) stream
        host = np.empty(count, dtype=np.float64)
        err, = cudart.cudaMemcpy(host.ctypes.data, ptr, 8 * count, cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost)
        assert err == cudart.cudaError_t.cudaSuccess, err
        t = torch.from_numpy(host)
        if os.environ.get("LPCA_DIST_TRACE") and count < 8:
            print(f"rank {rank}: in {host.tolist()}", flush=True)
        dist.all_reduce(t)
        if os.environ.get("LPCA_DIST_TRACE") and count < 8:
            print(f"rank {rank}: out {host.tolist()}", flush=True)
        # the sum goes back on the library's stream (a legacy-stream copy from
        # pageable memory may still be in flight when cudaMemcpy returns)
        err, = cudart.cudaMemcpyAsync(ptr, host.ctypes.data, 8 * count, cudart.cudaMemcpyKind.cudaMemcpyHostToDevice,
                                      stream)
        assert err == cudart.cudaError_t.cudaSuccess, err
        torch.cuda.ExternalStream(stream).synchronize()

    ctx = lp.Context.hooked(0, rank, world, allreduce)
    results = {}
    for name, c in CASES.items():
        x = case_data(name)
        lo, hi = shard(c, x.shape[0], world, rank)
        if c.get("drop_col_on") == rank:
            x = x[:, :-1]
        xs = torch.from_numpy(np.ascontiguousarray(x[lo:hi])).cuda()
        cfg = lp.ReducerConfig(method=c["method"], k=c["k"], l=c["l"], projection=projection(c),
                               power_iters=c.get("q", 0))
        try:
            if c.get("stream"):
                blocks = lp.SliceRowBlockStream(x[lo:hi], c["block_rows"]) if hi > lo else _Empty()
                fn = lp.reduce_spca_streaming if c["method"] == lp.ReducerMethod.spca else lp.reduce_lazy_spca_streaming
                mp = fn(blocks, cfg, ctx=ctx)
                y = None
            elif c.get("sparse"):
                mp, y = lp.fit_transform(as_input(c, np.ascontiguousarray(x[lo:hi])), cfg, ctx=ctx)
            else:
                mp, y = lp.fit_transform(xs, cfg, ctx=ctx)
            results[name + ".v"] = mp.v
            results[name + ".s"] = mp.singular_values
            if y is not None:
                results[name + ".y"] = y
        except lp.Error as e:
            idx = e.index() if hasattr(e, "index") else -1
            results[name + ".err"] = np.array([type(e).__name__, str(e), str(idx)])
            print(f"rank {rank}: {name} raised {type(e).__name__}: {e}", flush=True)
        print(f"rank {rank}: {name} done", flush=True)
    results["calls"] = np.array([calls[0]])
    np.savez(out / f"rank{rank}.npz", **results)
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


class _Empty(lp.RowBlockStream):
    def next(self):
        return None


if __name__ == "__main__":
    main()
