"""100M-scale instance generation (SURVEY §8.d "Synthetic inputs", configs C2–C4).

Input generation only — like the rest of `datagen`, nothing here computes any
step of the method (no query projection, routing, entry scoring, traversal or
refinement).  It manufactures what PilotANN's offline preprocessing hands to
the GPU stage (§3 ⓐⓑⓒ): the full graph, the sampled + reconnected
subgraph, the SVD basis and X̂, the FES index
(P:L437-441), and exhaustive-scan ground truth for recall.

Why a second graph tool.  `datagen.build_graph` loops over one k-means
partition at a time in Python; at 10M rows (10K partitions) it takes ~60 s,
at 100M (100K partitions, D = 200) it would take ~30 min and its reverse-edge
pass would need ~100 GB of int64 edge lists.  This tool does the same three
steps — kNN candidates restricted to the P nearest partitions, occlusion (RNG)
pruning to R, reverse-edge fill — with

  * partitions processed in padded batches (one batched TF32 GEMM + one top-k
    per batch of partitions, not per partition),
  * the candidate list re-ranked exactly in fp32 (direct form) before pruning,
  * int32 ids and a destination-range-chunked reverse-edge pass,
  * X̂ generated in place (X is rotated chunk by chunk, one 4·N·D-byte buffer),

so a 100M × 200 instance builds in minutes on one B200 and fits in host RAM
(X̂ 80 GB + graphs 16 GB of the box's 196 GB).  The graph is built over X̂
rows: V is orthonormal, so L2 distances (and, on the L2-normalised base rows,
inner-product order) are those of X up to fp32 rounding.

Caching.  The graphs, flags, FES index and ground truths (≈17 GB at 100M) are
saved as raw .npy files; the vectors are not cached — they are regenerated
deterministically from the counter-free torch Philox stream (same seed, same
chunking) in ~30 s, which is faster than reading 80 GB from disk.
"""
from __future__ import annotations

import math
import os
import time
from typing import Optional

import numpy as np
import torch


def _log(msg):
    if os.environ.get("PA_DATAGEN_QUIET") != "1":
        print(f"[datagen] {msg}", flush=True)


class _Prof:
    """Optional phase timer (PA_DATAGEN_PROFILE=1; synchronises the device)."""
    def __init__(self):
        self.on = os.environ.get("PA_DATAGEN_PROFILE") == "1"
        self.acc, self.t = {}, None

    def tick(self, name):
        if not self.on:
            return
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        now = time.time()
        if self.t is not None:
            self.acc[name] = self.acc.get(name, 0.0) + now - self.t
        self.t = now

    def report(self, what):
        if self.on:
            _log(f"{what} phases: " + ", ".join(f"{k} {v:.1f}s" for k, v in self.acc.items()))
        self.acc, self.t = {}, None


# ----------------------------------------------------------------------------
# Vectors: X generated in chunks, V fitted on a sample, X̂ = X·V in place
# ----------------------------------------------------------------------------
def gen_rotated(cfg, device):
    """(X̂ [N][D] fp32 on `device`, labels [N] int64, V fp64 [D][D], queries [m][D] fp32).

    X is produced by `datagen.gen_base` (identical rows, identical seeds), V by
    `datagen.fit_svd` on its usual ≤100K-row sample, then each chunk of X is
    replaced by X·V computed in fp64 and rounded once to fp32 (as `rotate`)."""
    import datagen as dg
    X, labels = dg.gen_base(cfg, device)
    Q = dg.gen_queries(cfg, device)
    V = dg.fit_svd(X, cfg.seeds["base"])
    Vd = torch.from_numpy(V).to(X.device)
    chunk = 1 << 20
    for s in range(0, X.shape[0], chunk):
        e = min(X.shape[0], s + chunk)
        X[s:e] = (X[s:e].double() @ Vd).float()
    return X, labels, V, Q


# ----------------------------------------------------------------------------
# Partitions: k-means centres on a sample, every row assigned to its nearest
# ----------------------------------------------------------------------------
def _assign(X: torch.Tensor, ids: torch.Tensor, C: torch.Tensor, budget: float = 2e9) -> torch.Tensor:
    """argmin_c ‖x − c‖² for rows `ids` of X (TF32 GEMM form, chunked)."""
    cn = (C * C).sum(1)
    K = C.shape[0]
    step = int(max(1024, budget // (4 * K)))
    out = torch.empty(ids.numel(), dtype=torch.int64, device=X.device)
    with _tf32():
        for s in range(0, ids.numel(), step):
            e = min(ids.numel(), s + step)
            A = X[ids[s:e]]
            out[s:e] = torch.argmin(cn[None, :] - 2.0 * (A @ C.T), 1)
    return out


class _tf32:
    def __enter__(self):
        self.a = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = True

    def __exit__(self, *a):
        torch.backends.cuda.matmul.allow_tf32 = self.a


def partition(X: torch.Tensor, ids: torch.Tensor, K: int, seed: int, iters: int = 6,
              per_centre_sample: int = 24) -> tuple[torch.Tensor, torch.Tensor]:
    """Geometric partition of rows `ids` into K cells (graph tool only):
    Lloyd k-means on a seeded sample of ≈24 rows per centre, then nearest-centre
    assignment of every row.  → (labels [n] int64 in 0..K−1, centres [K][D])."""
    n = ids.numel()
    dev = X.device
    rng = np.random.Generator(np.random.Philox(key=seed + 11))
    ns = min(n, K * per_centre_sample)
    sidx = ids[torch.from_numpy(np.sort(rng.choice(n, size=ns, replace=False))).to(dev)]
    C = X[sidx[torch.from_numpy(rng.choice(ns, size=K, replace=False)).to(dev)]].clone()
    for _ in range(iters):
        a = _assign(X, sidx, C)
        cnt = torch.bincount(a, minlength=K).float()
        S = torch.zeros_like(C)
        for s in range(0, ns, 1 << 22):
            S.index_add_(0, a[s:s + (1 << 22)], X[sidx[s:s + (1 << 22)]])
        keep = cnt > 0
        C[keep] = S[keep] / cnt[keep, None]
    return _assign(X, ids, C), C


# ----------------------------------------------------------------------------
# Candidates: exact scoring against the members of the P nearest partitions
# ----------------------------------------------------------------------------
def knn_candidates(X: torch.Tensor, ids: torch.Tensor, lab: torch.Tensor, cent: torch.Tensor, L: int,
                   P: int, batch_elems: float = 6e8, gather_rows: float = 3e6, a_max: int = 2048) -> torch.Tensor:
    """For every row u of `ids`: the L nearest (squared L2) among the members of
    the P partitions whose centres are nearest to u's partition centre (u's own
    included), self excluded, ascending.  Scores are a TF32 GEMM
    (‖c‖² − 2u·c); callers re-rank exactly.  → [n][L] int32 global ids (−1 pad)."""
    dev = X.device
    n = ids.numel()
    K = cent.shape[0]
    P = min(P, K)
    order = torch.argsort(lab, stable=True)
    counts = torch.bincount(lab, minlength=K)
    starts = torch.zeros(K + 1, dtype=torch.int64, device=dev)
    starts[1:] = torch.cumsum(counts, 0)
    # P nearest centres of every centre (empty partitions never chosen)
    cnn = (cent * cent).sum(1)
    cnn = torch.where(counts > 0, cnn, torch.full_like(cnn, float("inf")))
    nbr = torch.empty(K, P, dtype=torch.int64, device=dev)
    with _tf32():
        step = int(max(256, 2e9 // (4 * K)))
        for s in range(0, K, step):
            e = min(K, s + step)
            sc = cnn[None, :] - 2.0 * (cent[s:e] @ cent.T)
            sc[torch.arange(e - s, device=dev), torch.arange(s, e, device=dev)] = -float("inf")   # own first
            nbr[s:e] = torch.topk(sc, P, dim=1, largest=False).indices
    xn = torch.empty(n, dtype=torch.float32, device=dev)             # ‖x‖² of every member row
    for s in range(0, n, 1 << 22):
        r = X[ids[s:s + (1 << 22)]]
        xn[s:s + (1 << 22)] = (r * r).sum(1)
    out = torch.full((n, L), -1, dtype=torch.int32, device=dev)
    # work items = (partition, first row, rows ≤ a_max), partitions in descending size so a batch pads little
    porder = torch.argsort(counts, descending=True).tolist()
    cnt_l = counts.tolist()
    tot_l = counts[nbr].sum(1).tolist()                               # candidates per partition
    items = []
    for j in porder:
        if cnt_l[j] == 0:
            break
        for a0 in range(0, cnt_l[j], a_max):
            items.append((j, a0, min(a_max, cnt_l[j] - a0)))
    # batch items of similar candidate-set size (the padded Lc dominates the GEMM and top-k work)
    items.sort(key=lambda it: (-tot_l[it[0]], -it[2]))
    prof = _Prof()
    prof.tick("start")
    i = 0
    while i < len(items):
        La, Lc, b = items[i][2], tot_l[items[i][0]], 1
        while i + b < len(items):
            La2, Lc2 = max(La, items[i + b][2]), max(Lc, tot_l[items[i + b][0]])
            if (b + 1) * La2 * Lc2 > batch_elems or (b + 1) * Lc2 > gather_rows:
                break
            La, Lc = La2, Lc2
            b += 1
        it = torch.tensor(items[i:i + b], device=dev)                     # [b][3]
        i += b
        parts, ia0, ila = it[:, 0], it[:, 1:2], it[:, 2:3]
        # A rows: this item's rows of its partition, padded to La
        pa_ = parts[:, None]
        ta = torch.arange(La, device=dev)[None, :]
        va = ta < ila
        aidx = torch.where(va, order[(starts[pa_] + ia0 + ta).clamp_max(n - 1)], torch.zeros_like(ta))
        # candidate rows: concatenated members of the P nearest partitions, padded to Lc
        nb = nbr[parts]                                                  # [b][P]
        cc = counts[nb]
        cum = torch.cumsum(cc, 1)
        tc = torch.arange(Lc, device=dev)[None, :].expand(b, Lc)
        slot = torch.searchsorted(cum, tc.contiguous(), right=True).clamp_max(P - 1)  # which neighbour partition
        prev = torch.gather(cum - cc, 1, slot)
        vc = tc < cum[:, -1:]
        pos = torch.gather(starts[nb], 1, slot) + (tc - prev)
        cidx = torch.where(vc, order[pos.clamp(0, n - 1)], torch.zeros_like(pos))
        prof.tick("index")
        A = X[ids[aidx]]                                                 # [b][La][D]
        B = X[ids[cidx]]                                                 # [b][Lc][D]
        bn = torch.where(vc, xn[cidx], torch.full_like(xn[cidx], float("inf")))
        prof.tick("gather")
        with _tf32():
            sc = torch.baddbmm(bn[:, None, :], A, B.transpose(1, 2), alpha=-2.0)   # [b][La][Lc]
        prof.tick("gemm")
        kk = min(L + 1, Lc)
        v, j = torch.topk(sc, kk, dim=2, largest=False)
        del sc
        prof.tick("topk")
        cand = torch.gather(cidx[:, None, :].expand(b, La, Lc), 2, j)    # local row numbers
        bad = (cand == aidx[:, :, None]) | ~torch.isfinite(v)
        # drop self / padding, keep order, left-pack, cut to L
        key = bad.to(torch.int8)
        o = torch.argsort(key, dim=2, stable=True)[:, :, :L]
        cand = torch.gather(cand, 2, o)
        okk = ~torch.gather(bad, 2, o)
        g = torch.where(okk, ids[cand].to(torch.int32), torch.full_like(cand, -1, dtype=torch.int32))
        if g.shape[2] < L:
            g = torch.cat([g, torch.full((b, La, L - g.shape[2]), -1, dtype=torch.int32, device=dev)], 2)
        rows_ = aidx[va]
        out[rows_] = g[va]
        prof.tick("post")
    prof.report("candidates")
    return out


def refine(X: torch.Tensor, ids: torch.Tensor, cand: torch.Tensor, fan: int = 8, chunk: int = 1 << 14) -> torch.Tensor:
    """One neighbour-of-neighbour pass over approximate kNN lists (NN-descent
    style join, graph tool only): row u's list is replaced by the L nearest
    (exact fp32 squared L2, ties → smaller id) of row u ∪ the first `fan`
    entries of the lists of u's first `fan` entries.  cand [n][L] int32 global
    ids aligned with `ids` (−1 pad), ascending.  → same shape, ascending."""
    dev = X.device
    n, L = cand.shape
    N = X.shape[0]
    pos = torch.full((N,), -1, dtype=torch.int32, device=dev)
    pos[ids] = torch.arange(n, device=dev, dtype=torch.int32)
    out = torch.empty_like(cand)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        B = e - s
        r0 = cand[s:e].long()
        p0 = pos[r0[:, :fan].clamp_min(0)].long()
        two = cand[p0.clamp_min(0)][:, :, :fan].long()                     # [B][fan][fan]
        two = torch.where(((r0[:, :fan] >= 0) & (p0 >= 0))[:, :, None], two, torch.full_like(two, -1))
        c = torch.cat([r0, two.reshape(B, fan * fan)], 1)
        c, _ = torch.sort(c, 1)
        dup = torch.zeros_like(c, dtype=torch.bool)
        dup[:, 1:] = c[:, 1:] == c[:, :-1]
        bad = dup | (c < 0) | (c == ids[s:e, None])
        u = X[ids[s:e]]
        d = ((X[c.clamp_min(0)] - u[:, None, :]) ** 2).sum(2)
        d = torch.where(bad, torch.full_like(d, float("inf")), d)
        o = torch.argsort(d, dim=1, stable=True)[:, :L]                    # c ascending ⇒ ties → smaller id
        v = torch.gather(d, 1, o)
        out[s:e] = torch.where(torch.isfinite(v), torch.gather(c, 1, o), torch.full_like(v, -1, dtype=torch.int64)).to(torch.int32)
    return out


# ----------------------------------------------------------------------------
# Occlusion pruning on exactly re-ranked candidates
# ----------------------------------------------------------------------------
def prune(X: torch.Tensor, ids: torch.Tensor, cand: torch.Tensor, R: int, L: int, alpha: float = 1.0,
          chunk: int = 1 << 15) -> torch.Tensor:
    """Re-rank each candidate list by exact fp32 squared distance (ties → smaller
    id), keep the L nearest, then the HNSW/Vamana occlusion rule: scanning in
    ascending distance, c is kept unless an already kept s has
    alpha·δ(s, c) < δ(u, c); at most R kept.  → [n][R] int32 (−1 pad)."""
    dev = X.device
    n, W = cand.shape
    out = torch.full((n, R), -1, dtype=torch.int32, device=dev)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        c = cand[s:e].long()
        valid = c >= 0
        Vr = X[c.clamp_min(0)]                                           # [B][W][D]
        u = X[ids[s:e]]
        du = ((Vr - u[:, None, :]) ** 2).sum(2)
        du = torch.where(valid, du, torch.full_like(du, float("inf")))
        # order by (du, id): stable sort on id, then stable sort on du; one gather of the rows
        o1 = torch.argsort(torch.where(valid, c, torch.full_like(c, 1 << 40)), dim=1, stable=True)
        o2 = torch.argsort(torch.gather(du, 1, o1), dim=1, stable=True)[:, :L]
        o = torch.gather(o1, 1, o2)
        du, c = torch.gather(du, 1, o), torch.gather(c, 1, o)
        Vr = Vr[torch.arange(e - s, device=dev)[:, None], o]
        valid = torch.isfinite(du)
        nv = (Vr * Vr).sum(2)
        with _tf32():
            G = (nv[:, :, None] + nv[:, None, :] - 2.0 * torch.bmm(Vr, Vr.transpose(1, 2))).clamp_min_(0)
        keep = torch.zeros_like(valid)
        cnt = torch.zeros(e - s, dtype=torch.int64, device=dev)
        for j in range(L):
            occl = (keep & (alpha * G[:, :, j] < du[:, j:j + 1])).any(1)
            take = valid[:, j] & ~occl & (cnt < R)
            keep[:, j] = take
            cnt += take.long()
        o = torch.argsort((~keep).to(torch.int8), dim=1, stable=True)[:, :R]
        kept = torch.gather(c, 1, o)
        kk = torch.gather(keep, 1, o)
        out[s:e, :kept.shape[1]] = torch.where(kk, kept, torch.full_like(kept, -1)).to(torch.int32)
    return out


def reverse_fill(X: torch.Tensor, ids: torch.Tensor, rows: torch.Tensor, R: int, N: int,
                 max_edges: int = 1 << 28) -> torch.Tensor:
    """Fill the free slots of each row with reverse edges (u→v kept ⇒ v gets u),
    nearest first (ties → smaller id), skipping ids already present — the
    HNSW-style back-links of `datagen.reverse_fill`, processed by destination
    ranges so the edge list never exceeds `max_edges`.  rows [n][W] int32
    global ids aligned with `ids`.  → [n][R] int32."""
    dev = rows.device
    n, W = rows.shape
    pos = torch.full((N,), -1, dtype=torch.int32, device=dev)
    pos[ids] = torch.arange(n, device=dev, dtype=torch.int32)
    out = torch.full((n, R), -1, dtype=torch.int32, device=dev)
    out[:, :min(W, R)] = rows[:, :min(W, R)]
    deg = (out >= 0).sum(1)
    # destination position of every edge, computed once per source-row chunk
    n_ranges = max(1, math.ceil(n * W / max_edges))
    bounds = [n * i // n_ranges for i in range(n_ranges + 1)]
    for a, b in zip(bounds[:-1], bounds[1:]):
        srcs, dsts = [], []
        for s in range(0, n, 1 << 22):
            e = min(n, s + (1 << 22))
            r = rows[s:e]
            dp = torch.where(r >= 0, pos[r.clamp_min(0).long()], torch.full_like(r, -1))
            m = (dp >= a) & (dp < b)
            if m.any():
                ii, jj = torch.nonzero(m, as_tuple=True)
                srcs.append(ids[s + ii].to(torch.int64))
                dsts.append(dp[ii, jj].to(torch.int64))
        if not srcs:
            continue
        src, dpos = torch.cat(srcs), torch.cat(dsts)
        del srcs, dsts
        d = torch.empty(src.numel(), dtype=torch.float32, device=dev)
        for s in range(0, src.numel(), 1 << 22):
            e = min(src.numel(), s + (1 << 22))
            d[s:e] = ((X[src[s:e]] - X[ids[dpos[s:e]]]) ** 2).sum(1)
        o = torch.argsort(src)                       # ties → smaller id: sort by id, then distance, then row
        src, dpos, d = src[o], dpos[o], d[o]
        o = torch.argsort(d, stable=True)
        src, dpos = src[o], dpos[o]
        o = torch.argsort(dpos, stable=True)
        src, dpos = src[o], dpos[o]
        del d, o
        present = torch.empty(src.numel(), dtype=torch.bool, device=dev)
        for s in range(0, src.numel(), 1 << 22):
            e = min(src.numel(), s + (1 << 22))
            present[s:e] = (out[dpos[s:e]] == src[s:e, None].to(torch.int32)).any(1)
        src, dpos = src[~present], dpos[~present]
        start = torch.zeros(b - a + 1, dtype=torch.int64, device=dev)
        start[1:] = torch.cumsum(torch.bincount(dpos - a, minlength=b - a), 0)
        rank = torch.arange(dpos.numel(), device=dev) - start[dpos - a]
        slot = deg[dpos] + rank
        ok = slot < R
        out[dpos[ok], slot[ok]] = src[ok].to(torch.int32)
    return out


def fill_free(rows: torch.Tensor, cand: torch.Tensor, R: int, chunk: int = 1 << 15) -> torch.Tensor:
    """Slots still free after pruning and back-links take the nearest remaining
    candidates (ascending), so every row has min(R, #distinct candidates) edges —
    the diverse (occlusion-selected) edges and the back-links first, then the
    closest of the occluded ones, as HNSW implementations that keep pruned
    connections do.  rows [n][R], cand [n][L] int32 (−1 pad) → rows."""
    n, L = cand.shape
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        r = rows[s:e]
        c = cand[s:e]
        present = (c[:, :, None] == r[:, None, :]).any(2)
        elig = (c >= 0) & ~present
        deg = (r >= 0).sum(1, keepdim=True)
        rank = torch.cumsum(elig.to(torch.int64), 1)
        take = elig & (deg + rank <= R)
        bi, li = torch.nonzero(take, as_tuple=True)
        slot = (deg[bi, 0] + rank[bi, li] - 1)
        r[bi, slot] = c[bi, li]
    return rows


def build_graph(X: torch.Tensor, R: int, ids: Optional[torch.Tensor], seed: int, P: int = 0,
                part_size: int = 1000, slack: int = 16, labels: Optional[torch.Tensor] = None) -> torch.Tensor:
    """The graph tool at scale (same three steps as `datagen.build_graph`):
    partition → 2R + slack TF32 candidates from the members of the P nearest
    partitions (≈ P·part_size candidates per row) → neighbour-of-neighbour
    refinement → exact re-rank + occlusion pruning to R → reverse fill.
    Partitions: k-means cells of ≈part_size rows ("geo", default), or the
    generation clusters `labels` ("gen", PA_KNN_PART=gen: balanced, no k-means).
    → rows [n][R] int32 global ids aligned with `ids` (all rows if None)."""
    dev = X.device
    if ids is None:
        ids = torch.arange(X.shape[0], device=dev)
    n = ids.numel()
    P = P or int(os.environ.get("PA_KNN_P", "48"))
    t = time.time()
    if labels is not None and os.environ.get("PA_KNN_PART", "geo") == "gen":
        lab = labels[ids]
        K = int(labels.max().item()) + 1
        cnt = torch.bincount(lab, minlength=K)
        cent = torch.zeros(K, X.shape[1], dtype=torch.float32, device=dev)
        for s in range(0, n, 1 << 22):
            cent.index_add_(0, lab[s:s + (1 << 22)], X[ids[s:s + (1 << 22)]])
        cent /= cnt.clamp_min(1)[:, None].float()
        P = min(K, int(math.ceil(P * part_size / max(1.0, n / max(1, int((cnt > 0).sum().item()))))))
        _log(f"graph n={n}: generation-cluster partitions K={K}, P={P}")
    else:
        K = max(1, n // part_size)
        lab, cent = partition(X, ids, K, seed)
        _log(f"graph n={n}: partition K={K} {time.time() - t:.1f}s")
    t = time.time()
    cand = knn_candidates(X, ids, lab, cent, 2 * R + slack, P)
    del lab, cent
    _log(f"graph n={n}: candidates P={P} L={2 * R + slack} {time.time() - t:.1f}s")
    for _ in range(int(os.environ.get("PA_KNN_REFINE_PASSES", "1"))):
        t = time.time()
        cand = refine(X, ids, cand, fan=int(os.environ.get("PA_KNN_FAN", "8")))
        _log(f"graph n={n}: refine pass {time.time() - t:.1f}s")
    t = time.time()
    rows = prune(X, ids, cand, R, 2 * R, alpha=float(os.environ.get("PA_GRAPH_ALPHA", "1.0")))
    fill = os.environ.get("PA_GRAPH_FILL", "1") == "1"
    if not fill:
        del cand
    _log(f"graph n={n}: prune {time.time() - t:.1f}s")
    t = time.time()
    rows = reverse_fill(X, ids, rows, R, X.shape[0])
    _log(f"graph n={n}: reverse fill {time.time() - t:.1f}s")
    if fill:
        t = time.time()
        rows = fill_free(rows, cand, R)
        del cand
        _log(f"graph n={n}: nearest-candidate fill {time.time() - t:.1f}s")
    return rows


# ----------------------------------------------------------------------------
# Host CSR, sampling, one complete instance
# ----------------------------------------------------------------------------
def rows_to_csr(rows: torch.Tensor, N: int, ids: Optional[torch.Tensor] = None):
    """Device rows [n][R] int32 (−1 padded, valid entries left-packed) for nodes
    `ids` → host CSR over N nodes (int64 offsets, int32 neighbours)."""
    n, R = rows.shape
    deg = torch.zeros(N, dtype=torch.int64, device=rows.device)
    d = (rows >= 0).sum(1)
    if ids is None:
        deg[:n] = d
    else:
        deg[ids] = d
    off = torch.zeros(N + 1, dtype=torch.int64, device=rows.device)
    off[1:] = torch.cumsum(deg, 0)
    offsets = off.cpu().numpy()
    nbrs = np.empty(int(offsets[-1]), dtype=np.int32)
    if ids is None:
        order_rows = None
    else:
        order_rows = torch.argsort(ids)
    w = 0
    step = 1 << 22
    for s in range(0, n, step):
        e = min(n, s + step)
        r = rows[s:e] if order_rows is None else rows[order_rows[s:e]]
        v = r[r >= 0].cpu().numpy()
        nbrs[w:w + v.size] = v
        w += v.size
    return offsets, nbrs


def sample_members(rows: torch.Tensor, N: int, ratio: float, seed: int) -> np.ndarray:
    """`datagen.sample_members` (uniform seeds, 1% of N per round, + 1-hop
    expansion, last round truncated uniformly)
    with the same random draws, over device adjacency rows [N][R] (full graph)."""
    target = int(round(ratio * N))
    flags = np.zeros(N, dtype=np.uint8)
    if target >= N:
        flags[:] = 1
        return flags
    rng = np.random.Generator(np.random.Philox(key=seed))
    count = 0
    batch = max(1, N // 100)
    while count < target:
        free = np.flatnonzero(flags == 0)
        seeds = rng.choice(free, size=min(batch, free.size), replace=False)
        st = torch.from_numpy(seeds.astype(np.int64)).to(rows.device)
        nb = rows[st]
        fr = torch.cat([st, nb[nb >= 0].long()])
        new = torch.unique(fr).cpu().numpy()
        new = new[flags[new] == 0]
        if count + new.size > target:
            new = rng.choice(new, size=target - count, replace=False)
        flags[new] = 1
        count += new.size
    return flags


def build_instance_large(cfg, device="cuda", cache: Optional[str] = None, gt_k: int = 100,
                         with_gt: bool = True) -> dict:
    """All arrays pa_build / pa_attach_host / the oracle take for a 100M-scale
    config, as host numpy arrays: `rotated` (X̂, also the reduced rows through a
    row stride — `reduced` is the view X̂[:, :d']), `basis`, the full graph and
    subgraph CSRs, member flags, FES index, queries and ground truths.

    With `cache` (a directory), everything except the vectors is loaded from /
    saved to `cache/<cfg.name>/` as raw .npy; vectors are regenerated."""
    import datagen as dg
    t0 = time.time()
    cdir = os.path.join(cache, cfg.name) if cache else None
    names = ("full_offsets", "full_neighbors", "sub_offsets", "sub_neighbors", "member_flags",
             "fes_centroids", "fes_cell_off", "fes_pool_ids")
    # ground truths depend on the query set, i.e. on m (queries are not prefix-stable
    # across m): cached per m, next to the m-independent graphs
    gt_names = {"gt_ids": f"gt_ids_m{cfg.m}", "gt_sub_ids": f"gt_sub_ids_m{cfg.m}"}
    hit = cdir and all(os.path.exists(os.path.join(cdir, f + ".npy")) for f in names + ("done",))
    gt_hit = cdir and all(os.path.exists(os.path.join(cdir, f + ".npy")) for f in gt_names.values())
    Xh, labels, V, Q = gen_rotated(cfg, device)
    _log(f"{cfg.name}: vectors generated + rotated in {time.time() - t0:.1f}s")
    inst = dict(cfg=cfg, N=cfg.N, D=cfg.D, dp=cfg.dp, metric=cfg.metric, basis=V.astype(np.float32), V64=V,
                queries=Q.cpu().numpy())
    if hit:
        del labels
        for f in names:
            inst[f] = np.load(os.path.join(cdir, f + ".npy"))
        _log(f"{cfg.name}: graphs loaded from {cdir} ({time.time() - t0:.1f}s)")
    else:
        t = time.time()
        full = build_graph(Xh, cfg.R, None, cfg.seeds["graph"], labels=labels)
        _log(f"{cfg.name}: full graph {time.time() - t:.1f}s")
        flags = sample_members(full, cfg.N, cfg.ratio, cfg.seeds["sample"])
        inst["full_offsets"], inst["full_neighbors"] = rows_to_csr(full, cfg.N)
        del full
        mem = torch.from_numpy(np.flatnonzero(flags)).to(Xh.device)
        t = time.time()
        sub = build_graph(Xh, cfg.R, mem, cfg.seeds["graph"] + 1, labels=labels)
        del labels
        _log(f"{cfg.name}: subgraph ({mem.numel()} members) {time.time() - t:.1f}s")
        inst["sub_offsets"], inst["sub_neighbors"] = rows_to_csr(sub, cfg.N, ids=mem)
        del sub, mem
        inst["member_flags"] = flags
        inst["fes_centroids"], inst["fes_cell_off"], inst["fes_pool_ids"] = dg.train_fes(
            Xh[:, :cfg.dp], flags, cfg.r, cfg.n_e, cfg.seeds["fes"], metric=cfg.metric)
        if cdir:
            os.makedirs(cdir, exist_ok=True)
            for f in names:
                np.save(os.path.join(cdir, f + ".npy"), inst[f])
            open(os.path.join(cdir, "done.npy"), "w").close()
    if with_gt and gt_hit:
        for k, f in gt_names.items():
            inst[k] = np.load(os.path.join(cdir, f + ".npy"))
        _log(f"{cfg.name}: ground truths (m = {cfg.m}) loaded from {cdir}")
    elif with_gt:
        t = time.time()
        mem = torch.from_numpy(np.flatnonzero(inst["member_flags"])).to(Xh.device)
        Qh = Q.double() @ torch.from_numpy(V).to(Q.device)
        inst["gt_ids"], _ = dg.ground_truth(Qh, Xh, gt_k, cfg.metric)
        inst["gt_sub_ids"], _ = dg.ground_truth(Qh[:, :cfg.dp], Xh[:, :cfg.dp], gt_k, cfg.metric, ids=mem)
        del mem
        _log(f"{cfg.name}: ground truth (m = {cfg.m}) {time.time() - t:.1f}s")
        if cdir:
            os.makedirs(cdir, exist_ok=True)
            for k, f in gt_names.items():
                np.save(os.path.join(cdir, f + ".npy"), inst[k])
    t = time.time()
    rot = np.empty((cfg.N, cfg.D), dtype=np.float32)
    step = 1 << 22
    for s in range(0, cfg.N, step):
        rot[s:s + step] = Xh[s:s + step].cpu().numpy()
    del Xh
    torch.cuda.empty_cache() if torch.cuda.is_available() else None
    inst["rotated"] = rot
    inst["reduced"] = rot[:, :cfg.dp]                      # strided view (row stride D)
    _log(f"{cfg.name}: X̂ to host {time.time() - t:.1f}s; instance ready in {time.time() - t0:.1f}s")
    return inst


# ----------------------------------------------------------------------------
# C3/C4 (100M × 768): the full vectors (307 GB) fit neither one GPU nor this
# box's 196 GB of host RAM, so only what the GPU stage reads is materialised
# ----------------------------------------------------------------------------
def gen_reduced(cfg, device, chunk: int = 1 << 20, sample_cap: int = 100_000):
    """(X_r = (X·V)[:, :d'] [N][d'] fp32 on `device`, V fp64 [D][D], queries [m][D] fp32).

    X is generated chunk by chunk exactly as `datagen.gen_base` would (same
    generator stream, same chunking), twice: pass 1 accumulates the Gram matrix
    of the same ≤100K-row uniform sample `datagen.fit_svd` draws (in chunk order),
    pass 2 regenerates each chunk, rotates it in fp64 and keeps the first d'
    columns, rounded once to fp32.  The full rows are never stored."""
    import datagen as dg
    N, D, dp = cfg.N, cfg.D, cfg.dp
    gchunk = 1 << 21                                              # gen_base's default chunk
    lam, RT, centres, Kc = dg._mixture_params(cfg, device)
    sl, RTf, cf = lam.sqrt().float(), RT.float(), centres.float()
    rng = np.random.Generator(np.random.Philox(key=cfg.seeds["base"] + 7))
    idx = np.sort(rng.choice(N, size=min(N, sample_cap), replace=False))

    def rows():
        g = dg._gen(cfg.seeds["base"], device)
        for s in range(0, N, gchunk):
            e = min(N, s + gchunk)
            lab = torch.from_numpy(dg.cluster_of_rows(s, e - s, Kc, cfg.seeds["base"])).to(device)
            z = torch.randn(e - s, D, generator=g, device=device, dtype=torch.float32)
            x = cf[lab] + (z * sl[None, :]) @ RTf
            yield s, e, x / x.norm(dim=1, keepdim=True).clamp_min(1e-12)

    G = torch.zeros(D, D, dtype=torch.float64, device=device)
    for s, e, x in rows():
        sel = idx[(idx >= s) & (idx < e)] - s
        if sel.size:
            S = x[torch.from_numpy(sel).to(device)].double()
            G += S.T @ S
    w, V = np.linalg.eigh(G.cpu().numpy())
    V = V[:, np.argsort(-w, kind="stable")]
    for c in range(V.shape[1]):                                   # fit_svd's sign rule
        nz = np.flatnonzero(np.abs(V[:, c]) > 1e-12)
        if nz.size and V[nz[0], c] < 0:
            V[:, c] = -V[:, c]
    V = np.ascontiguousarray(V)
    Vd = torch.from_numpy(V[:, :dp].copy()).to(device)
    Xr = torch.empty(N, dp, dtype=torch.float32, device=device)
    for s, e, x in rows():
        for a in range(s, e, chunk):
            b = min(e, a + chunk)
            Xr[a:b] = (x[a - s:b - s].double() @ Vd).float()
    return Xr, V, dg.gen_queries(cfg, device)


def build_instance_reduced(cfg, device="cuda", cache: Optional[str] = None, gt_k: int = 100) -> dict:
    """GPU-stage instance of a 100M × 768 config (C3/C4): `reduced` (X_r), `basis`,
    the subgraph, member flags, FES index, queries and the subgraph ground truth
    GT_sub (reduced space).  DESIGN.md §5: with the full rows unavailable the full
    graph (used only to sample the members) and the subgraph are built over
    X_r; the recipe's spectrum (α = 1.6) leaves 97 % of the variance in the leading
    128 of 768 components.  No X̂ and no full graph: stages ②③ are not runnable
    (PA_ESTATE), the GPU stage is complete.  Cached like build_instance_large."""
    import datagen as dg
    t0 = time.time()
    cdir = os.path.join(cache, cfg.name) if cache else None
    names = ("sub_offsets", "sub_neighbors", "member_flags", "fes_centroids", "fes_cell_off", "fes_pool_ids")
    gt_name = f"gt_sub_ids_m{cfg.m}"                      # per m (see build_instance_large)
    hit = cdir and all(os.path.exists(os.path.join(cdir, f + ".npy")) for f in names + ("done",))
    gt_hit = cdir and os.path.exists(os.path.join(cdir, gt_name + ".npy"))
    Xr, V, Q = gen_reduced(cfg, device)
    _log(f"{cfg.name}: reduced rows generated (two streamed passes) in {time.time() - t0:.1f}s")
    inst = dict(cfg=cfg, N=cfg.N, D=cfg.D, dp=cfg.dp, metric=cfg.metric, basis=V.astype(np.float32), V64=V,
                queries=Q.cpu().numpy())
    if hit:
        for f in names:
            inst[f] = np.load(os.path.join(cdir, f + ".npy"))
        _log(f"{cfg.name}: graphs loaded from {cdir}")
    else:
        t = time.time()
        full = build_graph(Xr, cfg.R, None, cfg.seeds["graph"])
        _log(f"{cfg.name}: full graph (over X_r) {time.time() - t:.1f}s")
        flags = sample_members(full, cfg.N, cfg.ratio, cfg.seeds["sample"])
        del full
        torch.cuda.empty_cache() if torch.cuda.is_available() else None
        mem = torch.from_numpy(np.flatnonzero(flags)).to(Xr.device)
        t = time.time()
        sub = build_graph(Xr, cfg.R, mem, cfg.seeds["graph"] + 1)
        _log(f"{cfg.name}: subgraph ({mem.numel()} members) {time.time() - t:.1f}s")
        inst["sub_offsets"], inst["sub_neighbors"] = rows_to_csr(sub, cfg.N, ids=mem)
        del sub, mem
        inst["member_flags"] = flags
        inst["fes_centroids"], inst["fes_cell_off"], inst["fes_pool_ids"] = dg.train_fes(
            Xr, flags, cfg.r, cfg.n_e, cfg.seeds["fes"], metric=cfg.metric)
        if cdir:
            os.makedirs(cdir, exist_ok=True)
            for f in names:
                np.save(os.path.join(cdir, f + ".npy"), inst[f])
            open(os.path.join(cdir, "done.npy"), "w").close()
    if gt_hit:
        inst["gt_sub_ids"] = np.load(os.path.join(cdir, gt_name + ".npy"))
        _log(f"{cfg.name}: GT_sub (m = {cfg.m}) loaded from {cdir}")
    else:
        t = time.time()
        mem = torch.from_numpy(np.flatnonzero(inst["member_flags"])).to(Xr.device)
        Qh = Q.double() @ torch.from_numpy(V[:, :cfg.dp].copy()).to(Q.device)
        inst["gt_sub_ids"], _ = dg.ground_truth(Qh, Xr, gt_k, cfg.metric, ids=mem)
        del mem
        _log(f"{cfg.name}: ground truth (m = {cfg.m}) {time.time() - t:.1f}s")
        if cdir:
            os.makedirs(cdir, exist_ok=True)
            np.save(os.path.join(cdir, gt_name + ".npy"), inst["gt_sub_ids"])
    t = time.time()
    red = np.empty((cfg.N, cfg.dp), dtype=np.float32)
    for s in range(0, cfg.N, 1 << 22):
        red[s:s + (1 << 22)] = Xr[s:s + (1 << 22)].cpu().numpy()
    del Xr
    torch.cuda.empty_cache() if torch.cuda.is_available() else None
    inst["reduced"] = red
    _log(f"{cfg.name}: X_r to host {time.time() - t:.1f}s; instance ready in {time.time() - t0:.1f}s")
    return inst
