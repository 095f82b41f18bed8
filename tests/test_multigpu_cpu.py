"""The N>1 host path on CPU (gloo, world_size 2): query sharding covers the batch
exactly once, per-shard results concatenate to the single-process results (the
per-shard engine here is the oracle — the GPU engine is exercised by -m gpu), and
timings reduce by MAX."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2503_21206_b200.dist import shard_bounds


def test_shard_bounds_partition():
    for m in (0, 1, 7, 100, 10_001):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(m, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as orc
    from paper_2503_21206_b200.dist import max_over_ranks
    from tiny import tiny_instance
    inst = tiny_instance(n=300, D=12, dp=6, R=8, m=37, seed=91, member_ratio=0.6)
    lo, hi = shard_bounds(inst["queries"].shape[0], rank, world)
    res = orc.search(inst, queries=inst["queries"][lo:hi], k=5, ef=16, threads=1)
    parts = [None] * world
    dist.all_gather_object(parts, (lo, res["ids"].tolist(), res["d"].tolist()))
    t = max_over_ranks([float(rank + 1), -float(rank)])
    if rank == 0:
        q.put((parts, t))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharded_search_matches_single_process():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import oracle as orc
    from tiny import tiny_instance
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    inst = tiny_instance(n=300, D=12, dp=6, R=8, m=37, seed=91, member_ratio=0.6)
    full = orc.search(inst, k=5, ef=16, threads=1)
    parts.sort(key=lambda x: x[0])
    ids = np.concatenate([np.array(p[1]) for p in parts])
    d = np.concatenate([np.array(p[2]) for p in parts])
    assert np.array_equal(ids, full["ids"]) and np.array_equal(d, full["d"])
    assert t == [2.0, 0.0]
