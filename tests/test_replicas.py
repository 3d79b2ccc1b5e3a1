"""The N > 1 bench path on CPU: world_size-2 gloo processes (no GPU).

DESIGN.md §8(e): the solve does not shard, so N GPUs run N replicas -- independent seeded
right-hand sides, no collective on the data path -- and the job time is the max over ranks.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        cfg = inputs.config(0)
        b = torch.from_numpy(bench.rank_rhs(cfg, rank))
        gathered = [torch.zeros_like(b) for _ in range(world)]
        dist.all_gather(gathered, b)
        t = bench.max_over_ranks(10.0 + rank, dist, "cpu")
        if rank == 0:
            out.put(([g.numpy() for g in gathered], t))
    finally:
        dist.destroy_process_group()


def test_two_replicas_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    vecs, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = inputs.config(0)
    # each rank solves its own seeded system (no data-path collective), identical to a
    # single-process draw with the same seed
    assert not np.array_equal(vecs[0], vecs[1])
    for r in range(2):
        assert np.array_equal(vecs[r], inputs.rhs(cfg, seed=cfg.seed + r))
    assert t == 11.0   # the slowest replica sets the job time
