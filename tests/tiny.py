"""Tiny seeded instances for pins and parity (input generation only — no search arithmetic)."""
import numpy as np

import datagen as dg


def orthonormal(D, seed):
    rng = np.random.Generator(np.random.Philox(key=seed))
    A = rng.standard_normal((D, D))
    Q, R = np.linalg.qr(A)
    return Q * np.sign(np.diag(R))[None, :]


def tiny_instance(n=200, D=16, dp=8, R=8, m=16, seed=1, metric="l2", r=4, member_ratio=1.0,
                  ring=True, V=None, pool=None, sub_same_as_full=False):
    """Random instance: X ~ N(0,1), orthonormal V, X̂ = X·V (fp64→fp32), a
    ring-augmented random graph (every node reachable), optional member subset
    whose subgraph is the ring over members, FES cells = contiguous chunks of
    the (ascending) pool with centroid = cell mean."""
    rng = np.random.Generator(np.random.Philox(key=seed + 99))
    X = rng.standard_normal((n, D))
    V = orthonormal(D, seed) if V is None else V
    Xh = (X @ V).astype(np.float32)
    Q = rng.standard_normal((m, D)).astype(np.float32)
    _, full_off, full_nb = dg.ring_graph_fixture(n, R, 1, seed)
    if member_ratio >= 1.0 or sub_same_as_full:
        flags = np.ones(n, np.uint8)
        sub_off, sub_nb = full_off, full_nb
    else:
        mem = np.sort(rng.choice(n, size=max(1, int(member_ratio * n)), replace=False))
        flags = np.zeros(n, np.uint8)
        flags[mem] = 1
        nm = mem.size
        _, o2, nb2 = dg.ring_graph_fixture(nm, R, 1, seed + 5)
        rows = [[int(mem[v]) for v in nb2[o2[i]:o2[i + 1]]] for i in range(nm)]
        adj = [[] for _ in range(n)]
        for i, u in enumerate(mem):
            adj[u] = rows[i]
        sub_off = np.zeros(n + 1, np.int64)
        for u in range(n):
            sub_off[u + 1] = sub_off[u] + len(adj[u])
        sub_nb = np.array([v for row in adj for v in row], np.int32)
    mem = np.flatnonzero(flags)
    pool = mem if pool is None else np.asarray(pool)
    pool = np.sort(pool)
    r = min(r, pool.size)
    cuts = np.linspace(0, pool.size, r + 1).astype(np.int64)
    Xr = Xh[:, :dp]
    cent = np.stack([Xr[pool[cuts[c]:cuts[c + 1]]].astype(np.float64).mean(0) for c in range(r)]).astype(np.float32)
    return dict(metric=metric, N=n, D=D, dp=dp, sub_offsets=sub_off, sub_neighbors=sub_nb.astype(np.int32),
                member_flags=flags, reduced=np.ascontiguousarray(Xr), rotated=Xh,
                basis=V.astype(np.float32), fes_centroids=cent, fes_cell_off=cuts,
                fes_pool_ids=pool.astype(np.int32), full_offsets=full_off,
                full_neighbors=full_nb.astype(np.int32), queries=Q)


def sparse_id_instance(n_total=(1 << 24) + 4096, members=3000, D=16, dp=8, R=16, m=48, seed=11, metric="l2",
                       r=4):
    """Members scattered over a full id space larger than 2^24 (about a third of
    them ≥ 2^24): exercises the wide-id visited hash of the exact kernels.
    Non-member rows are zero; `reduced` is the strided view X̂[:, :d']."""
    rng = np.random.Generator(np.random.Philox(key=seed))
    lo = rng.choice(1 << 24, size=members - members // 3, replace=False)
    hi = (1 << 24) + rng.choice(n_total - (1 << 24), size=members // 3, replace=False)
    mem = np.sort(np.concatenate([lo, hi])).astype(np.int64)
    V = orthonormal(D, seed)
    Xm = rng.standard_normal((mem.size, D))
    Xh = np.zeros((n_total, D), np.float32)
    Xh[mem] = (Xm @ V).astype(np.float32)
    _, o2, nb2 = dg.ring_graph_fixture(mem.size, R, 1, seed + 5)
    deg = np.zeros(n_total, np.int64)
    deg[mem] = np.diff(o2)
    off = np.zeros(n_total + 1, np.int64)
    np.cumsum(deg, out=off[1:])
    nb = mem[nb2].astype(np.int32)                       # rows in ascending member order = ascending id order
    flags = np.zeros(n_total, np.uint8)
    flags[mem] = 1
    cuts = np.linspace(0, mem.size, r + 1).astype(np.int64)
    Xr = Xh[:, :dp]
    cent = np.stack([Xr[mem[cuts[c]:cuts[c + 1]]].astype(np.float64).mean(0) for c in range(r)]).astype(np.float32)
    Q = rng.standard_normal((m, D)).astype(np.float32)
    return dict(metric=metric, N=n_total, D=D, dp=dp, sub_offsets=off, sub_neighbors=nb, member_flags=flags,
                reduced=Xr, rotated=Xh, basis=V.astype(np.float32), fes_centroids=cent, fes_cell_off=cuts,
                fes_pool_ids=mem.astype(np.int32), queries=Q)
