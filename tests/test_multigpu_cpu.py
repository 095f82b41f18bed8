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


# ------------------------------------------------ bench.py's sharded path -----
class FakeIndex:
    """A CPU stand-in for the C-ABI index in the gloo test: its 'device arrays'
    are uint8 torch tensors (replicated by broadcast exactly like the real
    replica's), and search() runs stage ① of the oracle on the arrays it holds."""
    FIELDS = (("sub_offsets", "int64"), ("sub_neighbors", "int32"), ("reduced", "float32"), ("basis", "float32"),
              ("fes_centroids", "float32"), ("fes_cell_off", "int64"), ("fes_pool_ids", "int32"))

    def __init__(self, bufs, meta):
        self.bufs, self.meta = bufs, meta

    @classmethod
    def build(cls, inst):
        import torch
        arrs = [np.ascontiguousarray(inst[f], dtype=dt) for f, dt in cls.FIELDS]
        meta = [int(inst["N"]), int(inst["D"]), int(inst["dp"]), int(arrs[1].size), int(arrs[4].shape[0]),
                int(arrs[6].size), 1 if inst["metric"] == "ip" else 0]
        return cls([torch.from_numpy(a.view(np.uint8).reshape(-1).copy()) for a in arrs], meta)

    @staticmethod
    def nbytes(meta):
        n, D, dp, nnz, r, pool, _ = meta
        return [(n + 1) * 8, nnz * 4, n * dp * 4, D * D * 4, r * dp * 4, (r + 1) * 8, pool * 4]

    @classmethod
    def empty(cls, meta, device):
        import torch
        return cls([torch.zeros(b, dtype=torch.uint8) for b in cls.nbytes(meta)], list(meta))

    def replica_meta(self):
        class M(list):
            def to_list(self):
                return list(self)
        return M(self.meta)

    def replica_buffers(self):
        return [(i, b.numel()) for i, b in enumerate(self.bufs)]

    def instance(self):
        n, D, dp, nnz, r, pool, metric = self.meta
        shapes = [(n + 1,), (nnz,), (n, dp), (D, D), (r, dp), (r + 1,), (pool,)]
        inst = {f: b.numpy().view(dt).reshape(sh) for (f, dt), b, sh in zip(self.FIELDS, self.bufs, shapes)}
        inst["metric"] = "ip" if metric else "l2"
        return inst

    def search(self, queries, k, ef):
        import oracle as orc
        return orc.search(self.instance(), queries=queries, k=k, ef=ef, stages=1, threads=1)["ids"]


def _bench_worker(rank, world, port, q):
    import sys
    import types
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2503_21206_b200.dist import global_recall, replicate_index
    args = types.SimpleNamespace(config="C0", m=30, cache=None, set=["N=3000"], reduced="fp32")
    built = []

    def build_index(inst):
        built.append(rank)
        return FakeIndex.build(inst)

    ix_holder = [None]

    def replicate_wrapped(ix, rk, dev):
        # the wrap callback must see the (possibly new) replica's buffers
        if ix is not None:
            ix_holder[0] = ix

        def empty(meta, d):
            ix_holder[0] = FakeIndex.empty(meta, d)
            return ix_holder[0]
        return replicate_index(ix, rk, dev, empty_replica=empty, wrap=lambda p, b, d: ix_holder[0].bufs[p])
    cfg, inst, ix, m_total = bench.setup_sharded(args, rank, world, 0, build_index=build_index,
                                                 replicate=replicate_wrapped)
    ids = ix.search(inst["queries"], cfg.k, 32)
    rec = global_recall(ids, inst["gt_sub_ids"], cfg.k, m_total)
    q.put((rank, built, [b.numpy().tobytes() for b in ix.bufs], ids.tolist(), inst["queries"].shape[0], rec,
           m_total))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_bench_sharded_path():
    """bench.setup_sharded at world 2 (gloo): the instance and the index are
    built once (rank 0 only), rank 1 receives a byte-identical replica of every
    index array and its query shard by broadcast; the shards' results equal the
    single-process results, and the all-reduced recall equals the global one."""
    import oracle as orc
    import datagen as dg
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=600) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (r0, built0, bufs0, ids0, m0, rec0, mt), (r1, built1, bufs1, ids1, m1, rec1, _) = out
    assert built0 == [0] and built1 == []                       # built once, on rank 0
    assert bufs0 == bufs1                                       # byte-identical replica
    assert m0 + m1 == mt == 60 and abs(m0 - m1) <= 1
    cfg = dg.get_config("C0", m=60, N=3000)
    inst = dg.build_instance(cfg)
    single = orc.search(inst, k=cfg.k, ef=32, stages=1, threads=1)["ids"]
    assert np.array_equal(np.array(ids0 + ids1), single)
    assert rec0 == rec1
    assert abs(rec0 - orc.recall(single, inst["gt_sub_ids"], cfg.k)) < 1e-12
