"""CPU, world size 2 (gloo): the row-sharded Lazy SPCA decomposition the
library runs over NCCL — each rank sketches its own rows with the shared Omega,
the n x l partials (Z for power steps, then F) are summed by one allreduce per
exchange, the l x l step is replicated — reproduces the single-process result
(Algorithm 4, proj/core/src/reducer.cpp:300-335, across ranks)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lazypca_oracle as O


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, n, k, l = 1200, 96, 6, 12
    x = O.synth_lowrank(0, m, n, 20, 0.9, 0.01, 7)
    rows = np.array_split(np.arange(m), world)[rank]  # contiguous row shard

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        return t.numpy()

    v, s, u = O.reduce_lazy_spca_sharded(x[rows], k, l, 5, allreduce, power_iters=q)
    y_local = O.apply_map(x[rows], v)  # transform stays local
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), v=v, s=s, y=y_local, rows=rows)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("q", [0, 1])
def test_sharded_fit_matches_single_process(tmp_path, q):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), q, str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    x = O.synth_lowrank(0, 1200, 96, 20, 0.9, 0.01, 7)
    v1, s1, _ = O.reduce_lazy_spca(x, 6, 12, 5, power_iters=q)
    for p in parts:  # every rank holds the identical map
        assert np.max(np.abs(p["s"] - s1) / s1) < 1e-10
        assert O.chordal_distance(p["v"], v1) < 1e-9
    assert np.array_equal(parts[0]["v"], parts[1]["v"])
    y = np.concatenate([p["y"] for p in parts])
    assert np.max(np.abs(y - O.apply_map(x, v1))) < 1e-9 * np.abs(y).max()


def test_bench_rank_env_parsing(monkeypatch):
    import bench
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "4")
    monkeypatch.setenv("LOCAL_RANK", "1")
    assert bench._dist() == (1, 4, 1)
