"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This module holds NONE of the method's search arithmetic (no projection of
queries, no routing, no entry scoring, no traversal, no refinement): it only
manufactures the *inputs* that PilotANN's `build()` and `search()` take
(SURVEY.md §8.d "Synthetic inputs"), plus ground truth by exhaustive scan for
recall measurement.  Both `oracle/` and the product receive the arrays this
module returns; neither imports the other.

Offline preprocessing that the paper performs before search and hands to the
GPU stage as inputs is generated here (§3 ⓐⓑⓒ):
  * the full graph index                (kNN graph, SURVEY §8.d "Graphs")
  * the sampled + reconnected subgraph
  * the SVD basis V and rotated base vectors X̂ = X·V
  * the FES entry index (k-means into r coarse cells)

Recipes (DESIGN.md §"Input recipe"):
  * "iid"     : C0 — i.i.d. N(0,1) rows (BASELINE.json configs[0]).
  * "mixture" : DEEP/T2I/WIKI/LAION-shaped — Gaussian mixture with decaying
                spectrum λ_i=(i+1)^-α under a fixed random rotation, K_c=N/1000
                centres, cluster of row r = splitmix64(r) mod K_c (ids carry no
                locality), rows L2-normalised; IP ("t2i") queries are shifted
                out-of-distribution and not normalised.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np
import torch

__all__ = [
    "Config", "CONFIGS", "get_config", "splitmix64",
    "gen_base", "gen_queries", "knn_graph", "sample_members", "reconnect",
    "fit_svd", "rotate", "train_fes", "ground_truth", "build_instance",
    "csr_from_rows", "ring_graph_fixture",
]


# ----------------------------------------------------------------------------
# Configurations (BASELINE.json "configs")
# ----------------------------------------------------------------------------
@dataclasses.dataclass
class Config:
    name: str
    N: int
    D: int
    dp: int                 # d' (reduced dimension)
    metric: str             # "l2" | "ip"
    ratio: float            # sampling ratio s
    m: int                  # queries
    k: int = 10
    ef: int = 64
    R: int = 32             # subgraph / full graph degree
    r: int = 32             # FES cells
    n_e: int = 65536        # FES pool cap (SURVEY §8.0 †)
    shape: str = "iid"      # "iid" | "mixture"
    alpha: float = 1.6      # spectrum decay (tuned, DESIGN.md §Input recipe)
    sc: float = 1.0         # centre scale (tuned: clusters overlap → navigable kNN graph)
    ood_shift: float = 0.0  # IP query shift (T2I-shaped)
    seed: int = 2503
    gt_k: int = 100

    @property
    def seeds(self):
        b = self.seed
        return dict(base=b, query=b + 1000, graph=b + 2000, sample=b + 3000, fes=b + 4000)


CONFIGS = {
    # configs[0]: 10K random fp32 d=96, degree-32 kNN, 50% subgraph, d'=32, 100 q, k=10, ef=64
    "C0": Config("C0-random-10K", N=10_000, D=96, dp=32, metric="l2", ratio=0.5, m=100,
                 k=10, ef=64, shape="iid", seed=2503),
    # configs[1]: DEEP-shaped 10M x 96 L2, d'=48, 10K queries, 1 B200 (s=0.33 from Table 4 DEEP)
    "C1": Config("C1-DEEP-10M", N=10_000_000, D=96, dp=48, metric="l2", ratio=0.33, m=10_000,
                 k=10, ef=64, shape="mixture", seed=2504),
    # configs[2]: T2I-shaped 100M x 200 IP, d'=64 (s=0.25)
    "C2": Config("C2-T2I-100M", N=100_000_000, D=200, dp=64, metric="ip", ratio=0.25, m=10_000,
                 k=10, ef=64, shape="mixture", ood_shift=0.5, seed=2505),
    # configs[3]: LAION-shaped 100M x 768, d'=128 (s=0.25)
    "C3": Config("C3-LAION-100M", N=100_000_000, D=768, dp=128, metric="l2", ratio=0.25, m=10_000,
                 k=10, ef=64, shape="mixture", seed=2506),
    # configs[4]: WIKI-shaped 100M x 768 sweep
    "C4": Config("C4-WIKI-100M", N=100_000_000, D=768, dp=128, metric="l2", ratio=0.25, m=65_536,
                 k=10, ef=64, shape="mixture", seed=2507),
    # scaled-size measurement configs of the 100M rows (same recipe; the 100M graph tool is round 2)
    "C2S": Config("C2S-T2I-shaped-10M", N=10_000_000, D=200, dp=64, metric="ip", ratio=0.25, m=10_000,
                  k=10, ef=64, shape="mixture", ood_shift=0.5, seed=2515),
    "C3S": Config("C3S-LAION-shaped-2M", N=2_000_000, D=768, dp=128, metric="l2", ratio=0.25, m=10_000,
                  k=10, ef=64, shape="mixture", seed=2516),
    # scaled-down shaped configs used by parity tests (same recipe, oracle-sized)
    "S1": Config("S1-DEEP-shaped-20K", N=20_000, D=96, dp=48, metric="l2", ratio=0.33, m=256,
                 k=10, ef=64, shape="mixture", seed=2604),
    "S2": Config("S2-T2I-shaped-20K", N=20_000, D=200, dp=64, metric="ip", ratio=0.25, m=256,
                 k=10, ef=64, shape="mixture", ood_shift=0.5, seed=2605),
}


def get_config(name: str, **overrides) -> Config:
    cfg = dataclasses.replace(CONFIGS[name])
    for k, v in overrides.items():
        setattr(cfg, k, v)
    return cfg


# ----------------------------------------------------------------------------
# Counter-based hash (used only to scatter rows over clusters)
# ----------------------------------------------------------------------------
def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser over uint64 counters (vectorised, wraps mod 2^64)."""
    z = (np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15))
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def _mixture_params(cfg: Config, device):
    """Spectrum, rotation and cluster centres of the shaped recipe."""
    D = cfg.D
    g = _gen(cfg.seeds["base"] + 17, "cpu")
    lam = torch.tensor([(i + 1.0) ** (-cfg.alpha) for i in range(D)], dtype=torch.float64)
    A = torch.randn(D, D, generator=g, dtype=torch.float64)
    Qr, Rr = torch.linalg.qr(A)
    Qr = Qr * torch.sign(torch.diagonal(Rr))[None, :]          # sign fix -> unique rotation
    Kc = max(1, cfg.N // 1000)
    G = torch.randn(Kc, D, generator=g, dtype=torch.float64)
    centres = cfg.sc * (G * lam.sqrt()[None, :]) @ Qr.T          # μ_j = s_c (g_j ⊙ √λ) R_D
    return lam.to(device), Qr.T.contiguous().to(device), centres.to(device), Kc


def cluster_of_rows(start: int, count: int, Kc: int, salt: int) -> np.ndarray:
    r = np.arange(start, start + count, dtype=np.uint64) ^ np.uint64(salt)
    return (splitmix64(r) % np.uint64(Kc)).astype(np.int64)


def gen_base(cfg: Config, device="cpu", chunk: int = 1 << 21):
    """Base vectors X [N][D] fp32 (torch, on `device`) and cluster labels (or None)."""
    N, D = cfg.N, cfg.D
    g = _gen(cfg.seeds["base"], device)
    X = torch.empty(N, D, dtype=torch.float32, device=device)
    if cfg.shape == "iid":
        for s in range(0, N, chunk):
            e = min(N, s + chunk)
            X[s:e] = torch.randn(e - s, D, generator=g, device=device, dtype=torch.float32)
        return X, None
    lam, RT, centres, Kc = _mixture_params(cfg, device)
    labels = torch.empty(N, dtype=torch.int64, device=device)
    sl = lam.sqrt().float()
    RTf, cf = RT.float(), centres.float()
    for s in range(0, N, chunk):
        e = min(N, s + chunk)
        lab = torch.from_numpy(cluster_of_rows(s, e - s, Kc, cfg.seeds["base"])).to(device)
        z = torch.randn(e - s, D, generator=g, device=device, dtype=torch.float32)
        x = cf[lab] + (z * sl[None, :]) @ RTf
        x = x / x.norm(dim=1, keepdim=True).clamp_min(1e-12)
        X[s:e] = x
        labels[s:e] = lab
    return X, labels


def gen_queries(cfg: Config, device="cpu"):
    """Queries Q [m][D] fp32.  Shaped: same mixture (in-distribution) for L2;
    IP (T2I-shaped) queries get a fixed shift Δ and are not normalised."""
    m, D = cfg.m, cfg.D
    g = _gen(cfg.seeds["query"], device)
    if cfg.shape == "iid":
        return torch.randn(m, D, generator=g, device=device, dtype=torch.float32)
    lam, RT, centres, Kc = _mixture_params(cfg, device)
    lab = torch.from_numpy(cluster_of_rows(0, m, Kc, cfg.seeds["query"])).to(device)
    z = torch.randn(m, D, generator=g, device=device, dtype=torch.float32)
    x = centres.float()[lab] + (z * lam.sqrt().float()[None, :]) @ RT.float()
    if cfg.metric == "ip" and cfg.ood_shift > 0:
        gs = _gen(cfg.seeds["query"] + 1, "cpu")
        delta = torch.randn(D, generator=gs, dtype=torch.float64)
        spread = centres.std(dim=0).norm().item()
        delta = (delta / delta.norm() * cfg.ood_shift * spread).float().to(device)
        return (x + delta[None, :]).contiguous()
    return (x / x.norm(dim=1, keepdim=True).clamp_min(1e-12)).contiguous()


# ----------------------------------------------------------------------------
# Graph construction tools (offline; "same trained graph index" stand-in)
# ----------------------------------------------------------------------------
def _sqdist(A: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
    an = (A * A).sum(1, keepdim=True)
    bn = (B * B).sum(1)[None, :]
    return (an + bn - 2.0 * (A @ B.T)).clamp_min_(0)


def _score(A, B, metric):
    return _sqdist(A, B) if metric == "l2" else -(A @ B.T)


def csr_from_rows(rows: np.ndarray, N: int, ids: Optional[np.ndarray] = None):
    """rows [n][R] int (−1 padded) for nodes `ids` (default 0..n−1) → CSR over N nodes."""
    rows = np.asarray(rows)
    if ids is None:
        ids = np.arange(rows.shape[0])
    deg = np.zeros(N, dtype=np.int64)
    valid = rows >= 0
    deg[ids] = valid.sum(1)
    offsets = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(deg, out=offsets[1:])
    nbrs = np.empty(offsets[-1], dtype=np.int32)
    order = np.argsort(ids, kind="stable")
    r = rows[order]
    nbrs[:] = r[r >= 0]                    # row-major boolean indexing keeps row order
    return offsets, nbrs


def knn_graph(X: torch.Tensor, R: int, ids: Optional[torch.Tensor] = None, labels=None,
              metric: str = "l2", P: int = 0, chunk: int = 4096, refine: int = -1):
    """Degree-R kNN graph over the rows `ids` of X (all rows if None), neighbour
    lists in ascending-distance order, self excluded.  Exact brute force when
    `labels` is None; otherwise candidates are restricted to the P nearest
    generation clusters (cluster-local exact kNN, SURVEY §8.d "Graphs").
    Returns rows [n][R] int64 of global ids (−1 padded) aligned with `ids`."""
    dev = X.device
    if ids is None:
        ids = torch.arange(X.shape[0], device=dev)
    n = ids.numel()
    Xs = X[ids]
    out = torch.full((n, R), -1, dtype=torch.int64, device=dev)
    if labels is None:
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            d = _sqdist(Xs[s:e], Xs) if metric == "l2" else _sqdist(Xs[s:e], Xs)
            d[torch.arange(e - s, device=dev), torch.arange(s, e, device=dev)] = float("inf")
            kk = min(R, n - 1)
            if kk <= 0:
                continue
            v, j = torch.topk(d, kk, dim=1, largest=False)
            j = torch.where(torch.isfinite(v), ids[j], torch.full_like(j, -1))
            out[s:e, :kk] = j
        return out
    lab = labels[ids]
    Kc = int(labels.max().item()) + 1
    P = P or int(__import__("os").environ.get("PA_KNN_P", "64"))
    order = torch.argsort(lab, stable=True)
    counts = torch.bincount(lab, minlength=Kc)
    starts = torch.zeros(Kc + 1, dtype=torch.int64, device=dev)
    starts[1:] = torch.cumsum(counts, 0)
    cent = torch.zeros(Kc, X.shape[1], dtype=torch.float32, device=dev)
    cent.index_add_(0, lab, Xs)
    cent = cent / counts.clamp_min(1)[:, None].float()
    nc = torch.empty(Kc, min(P, Kc), dtype=torch.int64, device=dev)
    for s in range(0, Kc, chunk):
        e = min(Kc, s + chunk)
        d = _sqdist(cent[s:e], cent)
        d[:, counts == 0] = float("inf")
        nc[s:e] = torch.topk(d, min(P, Kc), dim=1, largest=False).indices
    st, ct = starts.tolist(), counts.tolist()
    ncl = nc.tolist()
    for j in range(Kc):
        if ct[j] == 0:
            continue
        a = order[st[j]:st[j] + ct[j]]
        cand = torch.cat([order[st[c]:st[c] + ct[c]] for c in ncl[j] if ct[c] > 0])
        d = _sqdist(Xs[a], Xs[cand])
        d[a[:, None] == cand[None, :]] = float("inf")
        kk = min(R, cand.numel() - 1)
        if kk <= 0:
            continue
        v, jj = torch.topk(d, kk, dim=1, largest=False)
        g = torch.where(torch.isfinite(v), ids[cand[jj]], torch.full_like(jj, -1))
        out[a, :kk] = g
    if refine < 0:          # default: one neighbour-of-neighbour pass above 200K rows (graph_quality.py:
        big = n > 200_000 and X.shape[1] <= 256             # (too many gathers at D = 768)
        refine = int(__import__("os").environ.get("PA_KNN_REFINE", "1" if big else "0"))
    if refine:              # 10M, P=64: 10-NN accuracy 0.745 → 0.894)
        out = refine_knn(X, out, ids, iters=refine)
    return out


def build_graph(X: torch.Tensor, R: int, ids: Optional[torch.Tensor] = None, labels=None):
    """The graph tool used for both the full graph and the subgraph reconnect
    ("same graph construction algorithm"): kNN candidates (L = 2R) →
    occlusion pruning to R → reverse-edge fill.  PA_GRAPH=knn gives plain kNN."""
    import os
    if ids is None:
        ids = torch.arange(X.shape[0], device=X.device)
    if os.environ.get("PA_GRAPH", "rng") == "knn":
        return knn_graph(X, R, ids=ids, labels=labels)
    cand = knn_graph(X, 2 * R, ids=ids, labels=labels)
    rows = prune_rng(X, ids, cand, R, alpha=float(os.environ.get("PA_GRAPH_ALPHA", "1.0")))
    return reverse_fill(rows, ids, X, R)


def partition_labels(X: torch.Tensor, K: int, seed: int, iters: int = 8, sample: int = 1 << 20,
                     chunk: int = 1 << 18) -> torch.Tensor:
    """Geometric partition for kNN candidate generation (graph tool only):
    k-means (random init, `iters` Lloyd steps on a ≤`sample`-row sample), then
    every row is assigned to its nearest centre.  → int64 labels [N]."""
    N = X.shape[0]
    dev = X.device
    rng = np.random.Generator(np.random.Philox(key=seed + 11))
    sidx = torch.from_numpy(np.sort(rng.choice(N, size=min(N, sample), replace=False))).to(dev)
    S = X[sidx]
    C = S[torch.from_numpy(rng.choice(S.shape[0], size=K, replace=False)).to(dev)].clone()
    for _ in range(iters):
        a = torch.cat([torch.argmin(_sqdist(S[s:s + chunk], C), 1) for s in range(0, S.shape[0], chunk)])
        cnt = torch.bincount(a, minlength=K).float()
        newC = torch.zeros_like(C).index_add_(0, a, S)
        keep = cnt > 0
        C[keep] = newC[keep] / cnt[keep, None]
    return torch.cat([torch.argmin(_sqdist(X[s:s + chunk], C), 1) for s in range(0, N, chunk)])


def refine_knn(X: torch.Tensor, rows: torch.Tensor, ids: torch.Tensor, iters: int = 2, chunk: int = 2048):
    """Neighbour-of-neighbour refinement of an approximate kNN graph (NN-descent
    style join; graph tool only).  rows [n][R] global ids (−1 padded) aligned with
    `ids`; each pass replaces a row by the R nearest of (row ∪ rows of its row)."""
    dev = X.device
    n, R = rows.shape
    N = X.shape[0]
    pos = torch.full((N,), -1, dtype=torch.int64, device=dev)
    pos[ids] = torch.arange(n, device=dev)
    for _ in range(iters):
        new = torch.empty_like(rows)
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            r0 = rows[s:e]                                           # [B][R]
            p0 = pos[r0.clamp_min(0)]
            two = rows[p0.clamp_min(0)]                              # [B][R][R]
            two = torch.where((r0 >= 0)[:, :, None] & (p0 >= 0)[:, :, None], two, torch.full_like(two, -1))
            cand = torch.cat([r0, two.reshape(e - s, R * R)], 1)
            cand, _ = torch.sort(cand, 1)
            dup = torch.zeros_like(cand, dtype=torch.bool)
            dup[:, 1:] = cand[:, 1:] == cand[:, :-1]
            me = ids[s:e][:, None]
            bad = dup | (cand < 0) | (cand == me)
            x = X[cand.clamp_min(0)]                                 # [B][C][D]
            d = ((x - X[ids[s:e]][:, None, :]) ** 2).sum(2)
            d = torch.where(bad, torch.full_like(d, float("inf")), d)
            v, j = torch.topk(d, R, dim=1, largest=False)
            new[s:e] = torch.where(torch.isfinite(v), torch.gather(cand, 1, j), torch.full_like(j, -1))
        rows = new
    return rows


def prune_rng(X: torch.Tensor, ids: torch.Tensor, cand: torch.Tensor, R: int, alpha: float = 1.0,
              chunk: int = 8192) -> torch.Tensor:
    """Occlusion (RNG) pruning of distance-sorted candidate lists, the HNSW/Vamana
    neighbour-selection heuristic ("occlusion rule"): candidate c is dropped
    if an already kept s has alpha·δ(s, c) < δ(u, c).  → rows [n][R] (−1 padded)."""
    dev = X.device
    n, L = cand.shape
    out = torch.full((n, R), -1, dtype=torch.int64, device=dev)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        c = cand[s:e]
        valid = c >= 0
        V = X[c.clamp_min(0)]                                    # [B][L][D]
        u = X[ids[s:e]]
        du = ((V - u[:, None, :]) ** 2).sum(2)                   # [B][L]
        nv = (V * V).sum(2)
        G = (nv[:, :, None] + nv[:, None, :] - 2.0 * torch.bmm(V, V.transpose(1, 2))).clamp_min_(0)
        keep = torch.zeros_like(valid)
        cnt = torch.zeros(e - s, dtype=torch.int64, device=dev)
        for j in range(L):
            occl = (keep & (alpha * G[:, :, j] < du[:, j:j + 1])).any(1)
            take = valid[:, j] & ~occl & (cnt < R)
            keep[:, j] = take
            cnt += take.long()
        # kept ids in candidate order, left-packed
        order = torch.argsort((~keep).to(torch.int8), dim=1, stable=True)[:, :R]
        kept = torch.gather(c, 1, order)
        kk = torch.gather(keep, 1, order)
        out[s:e, :kept.shape[1]] = torch.where(kk, kept, torch.full_like(kept, -1))
    return out


def reverse_fill(rows: torch.Tensor, ids: torch.Tensor, X: torch.Tensor, R: int) -> torch.Tensor:
    """Fill the free slots of each row with reverse edges (u→v kept ⇒ v gets u),
    nearest first, skipping ids already present (HNSW-style back-links)."""
    dev = rows.device
    n, W = rows.shape
    N = X.shape[0]
    pos = torch.full((N,), -1, dtype=torch.int64, device=dev)
    pos[ids] = torch.arange(n, device=dev)
    src = ids[:, None].expand(n, W).reshape(-1)
    dst = rows.reshape(-1)
    ok = dst >= 0
    src, dst = src[ok], dst[ok]
    dpos = pos[dst]
    ok = dpos >= 0
    src, dpos = src[ok], dpos[ok]
    d = torch.empty(src.numel(), dtype=torch.float32, device=dev)
    step = 1 << 22
    for a0 in range(0, src.numel(), step):
        a1 = min(src.numel(), a0 + step)
        d[a0:a1] = ((X[src[a0:a1]] - X[ids[dpos[a0:a1]]]) ** 2).sum(1)
    # sort by (target row, distance)
    o = torch.argsort(d)
    src, dpos, d = src[o], dpos[o], d[o]
    o = torch.argsort(dpos, stable=True)
    src, dpos = src[o], dpos[o]
    out = torch.full((n, R), -1, dtype=torch.int64, device=dev)
    out[:, :min(W, R)] = rows[:, :min(W, R)]
    deg = (out >= 0).sum(1)
    present = torch.empty(src.numel(), dtype=torch.bool, device=dev)
    for a0 in range(0, src.numel(), step):
        a1 = min(src.numel(), a0 + step)
        present[a0:a1] = (out[dpos[a0:a1]] == src[a0:a1, None]).any(1)
    src, dpos = src[~present], dpos[~present]
    start = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    start[1:] = torch.cumsum(torch.bincount(dpos, minlength=n), 0)
    rank = torch.arange(dpos.numel(), device=dev) - start[dpos]
    slot = deg[dpos] + rank
    ok = slot < R
    out[dpos[ok], slot[ok]] = src[ok]
    return out


def sample_members(offsets: np.ndarray, nbrs: np.ndarray, ratio: float, seed: int) -> np.ndarray:
    """Uniform node-wise seed sampling + 1-hop expansion until the target ratio
    (seed batch = 1% of N per round); the last
    round's additions are truncated uniformly to hit the target.  → uint8 flags."""
    N = offsets.shape[0] - 1
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
        frontier = [seeds]
        for s in seeds:
            frontier.append(nbrs[offsets[s]:offsets[s + 1]])
        new = np.unique(np.concatenate(frontier).astype(np.int64))
        new = new[flags[new] == 0]
        if count + new.size > target:
            new = rng.choice(new, size=target - count, replace=False)
        flags[new] = 1
        count += new.size
    return flags


def reconnect(X: torch.Tensor, flags: np.ndarray, R: int, labels=None, metric="l2", plain_knn: bool = False):
    """Rebuild edges among members with the same construction.
    Returns the subgraph CSR over the full id space (non-members: empty rows)."""
    N = X.shape[0]
    mem = np.flatnonzero(flags)
    ids = torch.from_numpy(mem).to(X.device)
    rows = (knn_graph(X, R, ids=ids, labels=labels) if plain_knn else build_graph(X, R, ids=ids, labels=labels)).cpu().numpy()
    return csr_from_rows(rows, N, ids=mem)


# ----------------------------------------------------------------------------
# SVD basis
# ----------------------------------------------------------------------------
def fit_svd(X: torch.Tensor, seed: int, sample_cap: int = 100_000) -> np.ndarray:
    """V [D][D] fp64, columns = right singular vectors of a ≤sample_cap uniform
    row sample, by descending singular value; no centering; sign
    rule: first nonzero component of each column ≥ 0."""
    N = X.shape[0]
    rng = np.random.Generator(np.random.Philox(key=seed + 7))
    idx = np.sort(rng.choice(N, size=min(N, sample_cap), replace=False))
    S = X[torch.from_numpy(idx).to(X.device)].double()
    G = (S.T @ S).cpu().numpy()
    w, V = np.linalg.eigh(G)
    order = np.argsort(-w, kind="stable")
    V = V[:, order]
    for c in range(V.shape[1]):
        nz = np.flatnonzero(np.abs(V[:, c]) > 1e-12)
        if nz.size and V[nz[0], c] < 0:
            V[:, c] = -V[:, c]
    return np.ascontiguousarray(V)


def rotate(X: torch.Tensor, V: np.ndarray, chunk: int = 1 << 20) -> torch.Tensor:
    """X̂ = X·V computed in fp64 and rounded once to fp32 (offline preprocessing)."""
    Vd = torch.from_numpy(V).to(X.device)
    out = torch.empty_like(X)
    for s in range(0, X.shape[0], chunk):
        e = min(X.shape[0], s + chunk)
        out[s:e] = (X[s:e].double() @ Vd).float()
    return out


# ----------------------------------------------------------------------------
# FES entry index training
# ----------------------------------------------------------------------------
def train_fes(Xr: torch.Tensor, flags: np.ndarray, r: int, n_e: int, seed: int,
              iters: int = 25, metric: str = "l2"):
    """k-means (k-means++ init, `iters` Lloyd steps, empty cells reseeded from the
    largest cell's farthest point) over a seeded uniform sample of n_e members.
    Returns centroids [r][d'] fp32, cell_off [r+1] int64, pool_ids int32 grouped
    by cell (ascending id within a cell)."""
    rng = np.random.Generator(np.random.Philox(key=seed))
    mem = np.flatnonzero(flags)
    if mem.size < r:
        raise ValueError("fewer members than FES cells")
    pool = np.sort(rng.choice(mem, size=min(n_e, mem.size), replace=False))
    P = Xr[torch.from_numpy(pool).to(Xr.device)].double()
    n = P.shape[0]
    # k-means++
    first = int(rng.integers(n))
    C = [P[first]]
    d2 = ((P - C[0]) ** 2).sum(1)
    for _ in range(1, r):
        p = (d2 / d2.sum()).cpu().numpy()
        p = p / p.sum()
        nxt = int(rng.choice(n, p=p))
        C.append(P[nxt])
        d2 = torch.minimum(d2, ((P - P[nxt]) ** 2).sum(1))
    C = torch.stack(C)
    for _ in range(iters):
        d = ((P[:, None, :] - C[None, :, :]) ** 2).sum(2) if n * r * P.shape[1] < 5e7 else _sqdist(P, C)
        a = torch.argmin(d, dim=1)
        cnt = torch.bincount(a, minlength=r)
        newC = torch.zeros_like(C)
        newC.index_add_(0, a, P)
        for c in range(r):
            if cnt[c] == 0:
                big = int(torch.argmax(cnt).item())
                mem_big = torch.nonzero(a == big).flatten()
                far = mem_big[torch.argmax(d[mem_big, big])]
                a[far] = c
                cnt = torch.bincount(a, minlength=r)
                newC = torch.zeros_like(C)
                newC.index_add_(0, a, P)
        C = newC / cnt.clamp_min(1)[:, None].double()
    d = _sqdist(P, C)
    a = torch.argmin(d, dim=1).cpu().numpy()
    cnt = np.bincount(a, minlength=r)
    for c in range(r):                       # guarantee non-empty cells
        if cnt[c] == 0:
            big = int(np.argmax(cnt))
            j = np.flatnonzero(a == big)[0]
            a[j] = c
            cnt = np.bincount(a, minlength=r)
    order = np.lexsort((pool, a))
    pool_ids = pool[order].astype(np.int32)
    cell_off = np.zeros(r + 1, dtype=np.int64)
    np.cumsum(cnt, out=cell_off[1:])
    return C.float().cpu().numpy(), cell_off, pool_ids


# ----------------------------------------------------------------------------
# Ground truth by exhaustive scan (recall measurement; pinned to the oracle's
# brute force in tests/test_datagen.py)
# ----------------------------------------------------------------------------
def ground_truth(Qh: torch.Tensor, Xh: torch.Tensor, k: int, metric: str = "l2",
                 ids: Optional[torch.Tensor] = None, slack: int = 32, chunk: Optional[int] = None):
    """Exact top-k by (δ, id) of each query row of Qh (fp64) over rows `ids` of
    Xh (fp32): fp32 scan keeps k+slack candidates, then an fp64 direct-form
    re-rank with ties to the smaller id.  → (ids int64 [m][k], δ fp64 [m][k])."""
    dev = Xh.device
    m = Qh.shape[0]
    if ids is None:
        ids = torch.arange(Xh.shape[0], device=dev)
    kk = min(k + slack, ids.numel())
    if chunk is None:                       # keep the m × chunk score block ≲ 1.5 GB
        chunk = int(min(1 << 20, max(4096, 1.5e9 // (4 * max(1, m)))))
    best_v = torch.full((m, kk), float("inf"), device=dev)
    best_i = torch.full((m, kk), -1, dtype=torch.int64, device=dev)
    Qf = Qh.float().to(dev)
    for s in range(0, ids.numel(), chunk):
        e = min(ids.numel(), s + chunk)
        blk = ids[s:e]
        sc = _score(Qf, Xh[blk], metric)
        v, j = torch.topk(sc, min(kk, e - s), dim=1, largest=False)
        allv = torch.cat([best_v, v], 1)
        alli = torch.cat([best_i, blk[j]], 1)
        bv, bj = torch.topk(allv, kk, dim=1, largest=False)
        best_v, best_i = bv, torch.gather(alli, 1, bj)
    # fp64 re-rank (direct form)
    cand = best_i.clamp_min(0)
    Xc = Xh[cand].double()                       # [m][kk][D]
    Qd = Qh.double().to(dev)[:, None, :]
    if metric == "l2":
        dd = ((Xc - Qd) ** 2).sum(2)
    else:
        dd = -(Xc * Qd).sum(2)
    dd = torch.where(best_i >= 0, dd, torch.full_like(dd, float("inf")))
    dd_np, id_np = dd.cpu().numpy(), best_i.cpu().numpy()
    out_i = np.empty((m, k), dtype=np.int64)
    out_d = np.empty((m, k), dtype=np.float64)
    for q in range(m):
        o = np.lexsort((id_np[q], dd_np[q]))[:k]
        out_i[q], out_d[q] = id_np[q][o], dd_np[q][o]
    return out_i, out_d


# ----------------------------------------------------------------------------
# One complete instance
# ----------------------------------------------------------------------------
def build_instance(cfg: Config, device="cpu", with_full_graph: bool = True, gt: bool = True,
                   gt_k: Optional[int] = None) -> dict:
    """All arrays `pa_build` / `pa_attach_host` / `pa_search` / the oracle take,
    as host numpy arrays, plus ground truths for recall.  Deterministic per cfg."""
    X, labels = gen_base(cfg, device)
    Q = gen_queries(cfg, device)
    lab = None                       # ≤ 50K rows: exact brute-force kNN
    if cfg.N > 50_000:               # larger: cluster-local kNN + neighbour-of-neighbour refinement
        use_gen = __import__("os").environ.get("PA_KNN_LABELS", "geo") == "gen" and labels is not None
        lab = labels if use_gen else partition_labels(X, max(1, cfg.N // 1000), cfg.seeds["graph"])
    full_rows = build_graph(X, cfg.R, labels=lab) if cfg.shape == "mixture" else knn_graph(X, cfg.R, labels=lab)
    full_off, full_nbrs = csr_from_rows(full_rows.cpu().numpy(), cfg.N)
    del full_rows
    if cfg.ratio >= 1.0:             # every node sampled: reconnecting with the same construction IS the full graph
        flags = np.ones(cfg.N, np.uint8)
        sub_off, sub_nbrs = full_off, full_nbrs
    else:
        flags = sample_members(full_off, full_nbrs, cfg.ratio, cfg.seeds["sample"])
        sub_off, sub_nbrs = reconnect(X, flags, cfg.R, labels=lab, plain_knn=cfg.shape != "mixture")
    V = fit_svd(X, cfg.seeds["base"])
    Xh = rotate(X, V)
    del X
    Xr = Xh[:, :cfg.dp].contiguous()
    cent, cell_off, pool_ids = train_fes(Xr, flags, cfg.r, cfg.n_e, cfg.seeds["fes"], metric=cfg.metric)
    inst = dict(cfg=cfg, N=cfg.N, D=cfg.D, dp=cfg.dp, metric=cfg.metric,
                sub_offsets=sub_off, sub_neighbors=sub_nbrs, member_flags=flags,
                basis=V.astype(np.float32), V64=V, fes_centroids=cent, fes_cell_off=cell_off,
                fes_pool_ids=pool_ids, queries=Q.cpu().numpy(), labels=None if labels is None else labels.cpu().numpy())
    if with_full_graph:
        inst["full_offsets"], inst["full_neighbors"] = full_off, full_nbrs
    inst["rotated"] = Xh.cpu().numpy()
    inst["reduced"] = np.ascontiguousarray(inst["rotated"][:, :cfg.dp])
    if gt:
        gk = gt_k or cfg.gt_k
        Qh = Q.double() @ torch.from_numpy(V).to(Q.device)       # fp64 rotated queries (GT only)
        inst["gt_ids"], inst["gt_d"] = ground_truth(Qh, Xh, min(gk, cfg.N), cfg.metric)
        mem_t = torch.from_numpy(np.flatnonzero(flags)).to(Xh.device)
        inst["gt_sub_ids"], inst["gt_sub_d"] = ground_truth(Qh[:, :cfg.dp], Xr, min(gk, int(flags.sum())),
                                                            cfg.metric, ids=mem_t)
    return inst


# ----------------------------------------------------------------------------
# Tiny hand fixtures
# ----------------------------------------------------------------------------
def ring_graph_fixture(n: int, R: int, D: int, seed: int, dp: Optional[int] = None, metric="l2"):
    """A tiny random instance whose graph contains a Hamiltonian ring, so every
    node is reachable from any entry (for brute-force pins)."""
    rng = np.random.Generator(np.random.Philox(key=seed))
    X = rng.standard_normal((n, D)).astype(np.float32)
    rows = np.full((n, R), -1, dtype=np.int64)
    for u in range(n):
        nb = [(u + 1) % n] if n > 1 else []
        others = rng.permutation(n)
        for v in others:
            if len(nb) >= R:
                break
            if v != u and v not in nb:
                nb.append(int(v))
        k = rng.integers(1, R + 1) if n > 1 else 0
        nb = nb[:max(1, k)] if n > 1 else []
        rows[u, :len(nb)] = nb
    off, nbrs = csr_from_rows(rows, n)
    return X, off, nbrs
