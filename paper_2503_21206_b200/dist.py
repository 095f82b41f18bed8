"""Host-side multi-GPU plumbing: one process per GPU, each holding
a full replica of the index and searching a contiguous shard of the query batch.
Queries are independent, so the search path has NO collective: results
are written per shard and only timings (MAX) and recall hit counts (SUM) are
reduced.  The index is built once, on rank 0, and replicated to the other ranks'
GPUs by broadcasting every device array of the C-ABI replica
(pa_replica_meta_of → pa_build_replica → pa_replica_buffers) — over NCCL, i.e.
NVLink/NVSwitch on one B200 box — instead of being regenerated per rank."""
from __future__ import annotations

BCAST_CHUNK = 1 << 30        # bytes per broadcast call (bounds NCCL's per-call buffers)


def shard_bounds(m_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) query range of `rank` (sizes differ by ≤ 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(m_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1 else None


def max_over_ranks(values, device=None):
    """MAX all-reduce of a list of floats (timings); identity when not distributed."""
    import torch
    dist = _dist()
    if dist is None:
        return list(values)
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def sum_over_ranks(values, device=None):
    """SUM all-reduce of a list of integers (e.g. recall hit counts of each shard)."""
    import torch
    dist = _dist()
    if dist is None:
        return [int(v) for v in values]
    t = torch.tensor([int(v) for v in values], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(v) for v in t.tolist()]


def recall_hits(ids, gt, k: int) -> int:
    """|ret_k ∩ gt_k| summed over the rows of one shard."""
    import numpy as np
    ids = np.asarray(ids)[:, :k]
    gt = np.asarray(gt)[:, :k]
    return int(sum(len(set(a.tolist()) & set(b.tolist())) for a, b in zip(ids, gt)))


def global_recall(ids, gt, k: int, m_total: int, device=None) -> float:
    """Recall@k over ALL ranks' shards (each rank passes its own rows)."""
    return sum_over_ranks([recall_hits(ids, gt, k)], device)[0] / float(k * m_total)


def broadcast_object(obj, src: int = 0):
    dist = _dist()
    if dist is None:
        return obj
    box = [obj]
    dist.broadcast_object_list(box, src=src)
    return box[0]


def broadcast_array(arr, src: int, rank: int, device=None):
    """numpy array from `src` to every rank (shape/dtype sent first; the payload
    goes through a `device` tensor — NCCL over NVLink when device is a GPU)."""
    import numpy as np
    import torch
    dist = _dist()
    if dist is None:
        return arr
    meta = broadcast_object((tuple(arr.shape), str(arr.dtype)) if rank == src else None, src)
    shape, dt = meta
    t = torch.from_numpy(np.ascontiguousarray(arr)).to(device) if rank == src else \
        torch.empty(shape, dtype=getattr(torch, np.dtype(dt).name), device=device)
    dist.broadcast(t, src)
    return t.cpu().numpy() if rank != src else arr


def device_bytes(ptr: int, nbytes: int, device: int):
    """A zero-copy torch uint8 CUDA tensor over [ptr, ptr + nbytes) on `device`
    (the __cuda_array_interface__ protocol), so a library-owned device array can
    be handed to torch.distributed."""
    import torch

    class _View:
        __cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                    "version": 3}
    return torch.as_tensor(_View(), device=torch.device("cuda", device))


def broadcast_buffers(tensors, src: int = 0, chunk: int = BCAST_CHUNK):
    """Broadcast each flat uint8 tensor from `src`, in chunks of ≤ `chunk` bytes."""
    dist = _dist()
    if dist is None:
        return
    for t in tensors:
        flat = t.view(-1)
        for s in range(0, flat.numel(), chunk):
            dist.broadcast(flat[s:s + chunk], src)


def replicate_index(ix, rank: int, device: int, src: int = 0, empty_replica=None, wrap=device_bytes):
    """Rank `src` passes its built index; every other rank passes None and gets
    back a replica on `device` whose device arrays are byte copies of the
    source's (meta broadcast, empty replica allocated, buffers broadcast).
    `empty_replica(meta_list, device)` and `wrap(ptr, bytes, device)` default to
    the C-ABI replica and zero-copy CUDA views; tests substitute CPU fakes."""
    if _dist() is None:
        return ix
    if empty_replica is None:
        import paper_2503_21206_b200 as pa

        def empty_replica(vals, dev):
            return pa.Index.empty_replica(pa.ReplicaMeta.from_list(vals), dev)
    meta = broadcast_object(ix.replica_meta().to_list() if rank == src else None, src)
    if rank != src:
        ix = empty_replica(meta, device)
    bufs = ix.replica_buffers()
    sizes = broadcast_object([b for _, b in bufs] if rank == src else None, src)
    if [b for _, b in bufs] != sizes:
        raise RuntimeError(f"replica layout mismatch on rank {rank}: {[b for _, b in bufs]} vs {sizes}")
    broadcast_buffers([wrap(p, b, device) for p, b in bufs], src)
    return ix
