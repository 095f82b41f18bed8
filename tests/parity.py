"""Tie-aware parity protocol: GPU stage-① traces vs the oracle's (SURVEY §8.c
"Parity protocol").

Per query:
  1. routing: same cell, or both cells' fp64 δ within tol (near-tie);
  2. entries: same set, or every differing entry within tol of the oracle's E-th key;
  3. lockstep: visits (entries as a set, then in order) and expansions in order.
     At the first differing expansion the common prefix fixes Vis, and by I7 C is
     top-ef(Vis) in each arithmetic; the divergence must be a decision-point
     near-tie: |δ(u_gpu) − δ(u_orc)| ≤ tol (selection) or u_orc / u_gpu within
     tol of the ef boundary of the fp64 order (eviction);
  4. distances of every returned id within tol of the oracle's fp64 δ;
  5. |recall@k(GPU) − recall@k(oracle)| ≤ 0.002 against the same ground truth.
tol(δ) = 1e-5·|δ| + 1e-6·sqrt(|δ|·‖q'‖²)  (L2; the second term bounds the
fp32 projection error near δ → 0) and 1e-5·(Σ|q'_i x_i| + |δ|) for IP.
"""
from __future__ import annotations

import numpy as np

import oracle as orc

REL = 1e-5


class ParityReport:
    def __init__(self):
        self.exact = 0
        self.tie = 0
        self.fail = []
        self.div_steps = []

    def __repr__(self):
        return f"ParityReport(exact={self.exact}, tie_diverged={self.tie}, fail={len(self.fail)})"


def _tol(d, qn2, ipscale=None):
    d = np.abs(d)
    if ipscale is None:
        return REL * d + 1e-6 * np.sqrt(d * qn2) + 1e-30
    return REL * (ipscale + d) + 1e-30


def compare(inst, gpu: dict, ref: dict, k: int, ef: int, gt_ids=None, check_traces=True, width: int = 1) -> ParityReport:
    """width w > 1: an iteration expands the w best unchecked keys, so a first
    differing expansion is explained by a near-tie with any of them."""
    metric = inst.get("metric", "l2")
    Qh = orc.project(inst["queries"], inst["basis"])
    dp = inst["reduced"].shape[1]
    Qp = Qh[:, :dp]
    Xr = inst["reduced"]                   # may be a strided view (X̂[:, :d'] at 100M): rows gathered on demand
    m = Qp.shape[0]
    rep = ParityReport()

    def delta(q, ids):
        ids = np.asarray(ids, dtype=np.int64)
        x = Xr[ids].astype(np.float64)
        return ((x - Qp[q]) ** 2).sum(1) if metric == "l2" else -(x @ Qp[q])

    def tol(q, ids, d):
        qn2 = float((Qp[q] ** 2).sum())
        if metric == "l2":
            return _tol(d, qn2)
        sc = np.abs(Xr[np.asarray(ids, np.int64)].astype(np.float64) * Qp[q]).sum(1)
        return _tol(d, qn2, sc)

    def near(q, a, b):
        da, db = delta(q, [a, b])
        t = max(tol(q, [a], np.array([da]))[0], tol(q, [b], np.array([db]))[0])
        return abs(da - db) <= t

    C = inst["fes_centroids"].astype(np.float64)
    for q in range(m):
        why = None
        # ---- 4. distances of returned ids
        gi, gd = gpu["ids"][q], gpu["d"][q].astype(np.float64)
        ok = gi >= 0
        if ok.any():
            want = delta(q, gi[ok])
            if np.any(np.abs(gd[ok] - want) > tol(q, gi[ok], want)):
                bad = np.argmax(np.abs(gd[ok] - want) - tol(q, gi[ok], want))
                rep.fail.append((q, f"distance id {gi[ok][bad]} gpu {gd[ok][bad]!r} oracle {want[bad]!r}"))
                continue
        if not np.array_equal(np.sort(gi[ok]), np.unique(gi[ok])):
            rep.fail.append((q, "duplicate ids in result"))
            continue
        # ---- 1. routing
        cg, co = int(gpu["cell"][q]), int(ref["cell"][q])
        if cg != co:
            dc = ((C[[cg, co]] - Qp[q]) ** 2).sum(1) if metric == "l2" else -(C[[cg, co]] @ Qp[q])
            scale = None if metric == "l2" else float(np.abs(C[[cg, co]] * Qp[q]).sum(1).max())
            t = _tol(max(abs(dc[0]), abs(dc[1])), float((Qp[q] ** 2).sum()), scale)
            if abs(dc[0] - dc[1]) > t:
                rep.fail.append((q, f"routing {cg} vs {co} (δ {dc})"))
                continue
            rep.tie += 1
            rep.div_steps.append(-2)
            continue
        # ---- 2. entries
        eg = gpu["entries"][q]
        eo = ref["entries"][q]
        sg, so = set(eg[eg >= 0].tolist()), set(eo[eo >= 0].tolist())
        if sg != so:
            diff = list(sg ^ so)
            bnd = ref["entries_d"][q][eo >= 0].max()
            dd = delta(q, diff)
            if np.all(np.abs(dd - bnd) <= tol(q, diff, np.maximum(np.abs(dd), abs(bnd)))):
                rep.tie += 1
                rep.div_steps.append(-1)
                continue
            rep.fail.append((q, f"entries differ beyond near-ties: {sorted(diff)[:6]}"))
            continue
        if not check_traces:
            rep.exact += 1
            continue
        # ---- 3. lockstep traces
        ne_g, nv_g = int(gpu["trace_nexp"][q]), int(gpu["trace_nvis"][q])
        ne_o, nv_o = int(ref["trace_nexp"][q]), int(ref["trace_nvis"][q])
        cap = gpu["trace_expand"].shape[1]
        if max(ne_g, nv_g, ne_o, nv_o) > cap:
            rep.fail.append((q, f"trace capacity {cap} too small"))
            continue
        xg, xo = gpu["trace_expand"][q][:ne_g], ref["trace_expand"][q][:ne_o]
        vg, vo = gpu["trace_visit"][q][:nv_g], ref["trace_visit"][q][:nv_o]
        nE = len(so)
        if set(vg[:nE].tolist()) != set(vo[:nE].tolist()):
            rep.fail.append((q, "entry visits differ"))
            continue
        t = 0
        while t < min(ne_g, ne_o) and xg[t] == xo[t]:
            t += 1
        if t == ne_g == ne_o:
            if np.array_equal(vg[nE:], vo[nE:]):
                rep.exact += 1
                continue
            rep.fail.append((q, "identical expansions but different visits"))
            continue
        # common prefix of t expansions: are the visits so far identical?  The
        # oracle's visit trace fixes which neighbours of the common expansions
        # were new (rows hold distinct ids and a visited — or bloom-positive —
        # id never becomes new again), so the prefix is found by matching each
        # row, in stored order, against the trace; this holds for the exact
        # visited set and for the bloom filter (O13) alike.
        off, nb = inst["sub_offsets"], inst["sub_neighbors"]
        vis_set = set(vo[:nE].tolist())
        nvis_prefix = nE
        for u in xo[:t]:
            for v in nb[off[u]:off[u + 1]]:
                if nvis_prefix < nv_o and vo[nvis_prefix] == v:
                    vis_set.add(int(v))
                    nvis_prefix += 1
        if not np.array_equal(vg[nE:nvis_prefix], vo[nE:nvis_prefix]):
            rep.fail.append((q, f"visit prefix differs before expansion step {t}"))
            continue
        vis = np.array(sorted(vis_set), np.int64)
        dv = delta(q, vis)
        order = np.lexsort((vis, dv))
        K = vis[order]
        Kd = dv[order]
        expanded = set(xo[:t].tolist())
        topk = K[:ef]
        un = [u for u in topk if u not in expanded]
        u_orc = un[0] if un else None
        u_gpu = int(xg[t]) if t < ne_g else None
        bidx = min(ef, len(K) - 1)
        bnd = Kd[bidx] if len(K) > ef else None

        def at_boundary(u):
            if u is None or bnd is None:
                return False
            du = delta(q, [u])[0]
            return abs(du - bnd) <= tol(q, [u], np.array([max(abs(du), abs(bnd))]))[0] or \
                abs(du - Kd[ef - 1]) <= tol(q, [u], np.array([max(abs(du), abs(Kd[ef - 1]))]))[0]

        explained = False
        if u_gpu is not None and any(near(q, u_gpu, x) for x in un[:width]):
            explained = True
        elif at_boundary(u_orc) or at_boundary(u_gpu):
            explained = True
        if explained:
            rep.tie += 1
            rep.div_steps.append(t)
        else:
            rep.fail.append((q, f"trajectory diverged at expansion {t}: gpu {u_gpu} oracle {u_orc}"))
    # ---- 5. recall
    if gt_ids is not None:
        rg = orc.recall(gpu["ids"], gt_ids, k)
        ro = orc.recall(ref["ids"], gt_ids, k)
        rep.recall_gpu, rep.recall_orc = rg, ro
        if abs(rg - ro) > 0.002:
            rep.fail.append((-1, f"recall gpu {rg:.4f} vs oracle {ro:.4f}"))
    return rep
