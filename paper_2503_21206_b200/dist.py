"""Host-side multi-GPU plumbing: one process per GPU, each holding
a full replica of the index and searching a contiguous shard of the query batch.
Queries are independent, so the data path has NO collective: results are
written per shard and only timings are reduced (MAX over ranks)."""
from __future__ import annotations


def shard_bounds(m_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) query range of `rank` (sizes differ by ≤ 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(m_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(values, device=None):
    """MAX all-reduce of a list of floats (timings); identity when not distributed."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(values)
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()
