"""Pins of oracle O14 (two-hop entry selection, the FES baseline of P:L986-989;
DESIGN.md reading Q30) against things other than itself:

  * a hand-derived golden on a 7-node graph (1-D points, identity basis), where
    the hop-1 set, the beam choice and the hop-2 set are worked out by hand —
    fails if hop 2 expands the wrong hop-1 nodes, skips e0, or revisits;
  * beam = R on a random graph: the entries are exactly the E smallest keys of the
    whole 2-hop neighbourhood, computed with plain Python sets and numpy distances;
  * beam = 0: the entries are {e0} ∪ N(e0) sorted (numpy lexsort);
  * prefix property: entries for E are the first E of entries for E' > E;
  * n_dist = |{e0} ∪ hop-1 ∪ hop-2| (Python set count).
"""
import numpy as np
import pytest

import oracle as orc
from tiny import tiny_instance


def _csr(adj, n):
    off = np.zeros(n + 1, np.int64)
    for u in range(n):
        off[u + 1] = off[u] + len(adj.get(u, []))
    nb = np.array([v for u in range(n) for v in adj.get(u, [])], np.int32)
    return off, nb


def _inst_1d(points, adj, queries, metric="l2"):
    n = len(points)
    X = np.zeros((n, 2), np.float32)
    X[:, 0] = points
    off, nb = _csr(adj, n)
    Q = np.zeros((len(queries), 2), np.float32)
    Q[:, 0] = queries
    return dict(metric=metric, sub_offsets=off, sub_neighbors=nb, reduced=X, basis=np.eye(2, dtype=np.float32),
                fes_centroids=X[:1].copy(), fes_cell_off=np.array([0, 1], np.int64),
                fes_pool_ids=np.array([0], np.int32), queries=Q)


def test_two_hop_hand_golden():
    # points on a line; e0 = 0 at x = 0; query at x = 10
    #   N(0) = [1, 2, 3] at x = 4, 9, -5  → hop-1 keys: 2 (δ=1), 1 (δ=36), 3 (δ=225)
    #   beam 1 expands node 2 only: N(2) = [4, 0, 5] → 4 (x=11, δ=1), 5 (x=30, δ=400); 0 already visited
    #   N(1) = [6] (x = 10, δ=0) is NOT reached with beam 1, but is with beam 2
    points = [0.0, 4.0, 9.0, -5.0, 11.0, 30.0, 10.0]
    adj = {0: [1, 2, 3], 1: [6, 0], 2: [4, 0, 5], 3: [0], 4: [2], 5: [2], 6: [1]}
    inst = _inst_1d(points, adj, [10.0])
    r = orc.two_hop(inst, e0=0, beam=1, E=4)
    # visited: 0 (100), 1 (36), 2 (1), 3 (225), 4 (1), 5 (400) → keys by (δ, id): 2, 4, 1, 0
    assert list(r["ids"][0]) == [2, 4, 1, 0]
    assert list(r["d"][0]) == [1.0, 1.0, 36.0, 100.0]
    assert r["n_dist"][0] == 6
    r = orc.two_hop(inst, e0=0, beam=2, E=3)                 # node 1 expanded too → 6 (δ = 0) first
    assert list(r["ids"][0]) == [6, 2, 4] and r["d"][0][0] == 0.0
    assert r["n_dist"][0] == 7
    r = orc.two_hop(inst, e0=0, beam=0, E=8)                 # hop 1 only, padded
    assert list(r["ids"][0]) == [2, 1, 0, 3, -1, -1, -1, -1]
    assert np.isinf(r["d"][0][4:]).all()


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_two_hop_full_beam_is_brute_force_over_neighbourhood(metric):
    inst = tiny_instance(n=400, D=12, dp=6, R=8, m=12, seed=31, metric=metric, member_ratio=0.6)
    off, nb = inst["sub_offsets"], inst["sub_neighbors"]
    mem = np.flatnonzero(inst["member_flags"])
    e0 = int(mem[len(mem) // 2])
    Qh = inst["queries"].astype(np.float64) @ inst["basis"].astype(np.float64)
    X = inst["reduced"].astype(np.float64)
    hop1 = [int(v) for v in nb[off[e0]:off[e0 + 1]]]
    H = {e0} | set(hop1)
    for u in hop1:
        H |= set(int(v) for v in nb[off[u]:off[u + 1]])
    H = np.array(sorted(H))
    E = len(H) + 3
    r = orc.two_hop(inst, e0=e0, beam=64, E=E)
    for q in range(inst["queries"].shape[0]):
        if metric == "l2":
            d = ((X[H] - Qh[q, :6]) ** 2).sum(1)
        else:
            d = -(X[H] @ Qh[q, :6])
        o = np.lexsort((H, d))
        assert list(r["ids"][q][:len(H)]) == list(H[o])
        np.testing.assert_allclose(r["d"][q][:len(H)], d[o], rtol=1e-12, atol=1e-12)
        assert list(r["ids"][q][len(H):]) == [-1] * 3
        assert r["n_dist"][q] == len(H)


def test_two_hop_beam0_and_prefix():
    inst = tiny_instance(n=300, D=10, dp=5, R=8, m=8, seed=32)
    off, nb = inst["sub_offsets"], inst["sub_neighbors"]
    e0 = 17
    Hs = np.array(sorted({e0} | set(int(v) for v in nb[off[e0]:off[e0 + 1]])))
    Qh = inst["queries"].astype(np.float64) @ inst["basis"].astype(np.float64)
    X = inst["reduced"].astype(np.float64)
    r0 = orc.two_hop(inst, e0=e0, beam=0, E=len(Hs))
    for q in range(8):
        d = ((X[Hs] - Qh[q, :5]) ** 2).sum(1)
        assert list(r0["ids"][q]) == list(Hs[np.lexsort((Hs, d))])
    big = orc.two_hop(inst, e0=e0, beam=3, E=40)
    small = orc.two_hop(inst, e0=e0, beam=3, E=11)
    assert np.array_equal(big["ids"][:, :11], small["ids"])
    assert np.array_equal(big["d"][:, :11], small["d"])
