"""Pins of the ORACLE (oracle/oracle.cpp) against things other than itself.

Each O-step of the oracle is pinned here (SURVEY §8.c table "P"):
  O1 projection   — orthonormal V preserves norms; signed-permutation V gives an
                    exact permutation; equals a numpy fp64 matmul (library routine).
  O2 distance     — SPEC worked examples ([0,0] vs [3,4] → 25); golden fixtures.
  O3 routing      — r = 1 → cell 0; q' = centroid j → j; = numpy argmin.
  O4 FES          — r = 1 → entries = brute-force top-E over the whole pool (numpy);
                    work = Σ_c m_c·n_c and the Table 3 closed form.
  O5–O7 stage ①   — golden fixtures F1–F4 (hand-derived traces, tests/golden/);
                    ef ≥ reachable n ⇒ brute force (recall 1.0); single node ⇒ 1 calc;
                    query = member ⇒ rank 1, δ = 0; invariants I1–I9 on traces.
  O8–O9 stages ②③ — all toggles off ⇒ plain Alg 1 ⇒ with ef ≥ N on a connected graph
                    equals exhaustive brute force; d' = D ⇒ identity re-rank;
                    refine_iters = 0 ⇒ no stage-② expansions.
  O11 brute force — SPEC examples; equals numpy lexsort of numpy distances.
  O12 recall      — SPEC examples.
"""
import numpy as np
import pytest

import oracle as orc
from conftest import golden_names, instance_from_golden, load_golden
from tiny import orthonormal, tiny_instance


# ------------------------------------------------------------------ goldens --
@pytest.mark.parametrize("name", golden_names())
def test_golden_traces(name):
    g = load_golden(name)
    inst = instance_from_golden(g)
    res = orc.search(inst, k=g["k"], ef=g["ef"], stages=1, trace_cap=64, entries=g["entries"])
    ne, nv = int(res["trace_nexp"][0]), int(res["trace_nvis"][0])
    assert list(res["trace_expand"][0][:ne]) == g["expand"]
    assert list(res["trace_visit"][0][:nv]) == g["visit"]
    assert list(res["ids"][0]) == g["result_ids"]
    assert np.array_equal(res["d"][0], np.array(g["result_d"]))
    assert res["n_dist1"][0] == len(g["visit"])          # I9
    assert res["n_exp1"][0] == len(g["expand"])


# ---------------------------------------------------------- O11 / O12 -------
def test_brute_force_spec_examples():
    X = np.array([[0, 0], [3, 4]], np.float32)
    ids, d = orc.brute_force(np.array([[0.0, 0.0]]), X, 2)
    assert list(ids[0]) == [0, 1] and list(d[0]) == [0.0, 25.0]
    ids, d = orc.brute_force(np.array([[3.0, 4.0]]), X, 1)
    assert ids[0, 0] == 1 and d[0, 0] == 0.0
    ids, d = orc.brute_force(np.array([[0.0, 0.0]]), X, 3)
    assert ids[0, 2] == -1 and np.isinf(d[0, 2])                        # Q26 padding


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_brute_force_equals_numpy(metric):
    rng = np.random.default_rng(3)
    X = rng.standard_normal((500, 12)).astype(np.float32)
    X[7] = X[3]                                                           # exact tie → id order
    Qh = rng.standard_normal((20, 12))
    Qh[0] = X[3]
    ids, d = orc.brute_force(Qh, X, 10, metric=metric)
    Xd = X.astype(np.float64)
    for q in range(20):
        if metric == "l2":
            dd = ((Xd - Qh[q]) ** 2).sum(1)
        else:
            dd = -(Xd @ Qh[q])
        o = np.lexsort((np.arange(500), dd))[:10]
        assert list(ids[q]) == list(o)
        np.testing.assert_allclose(d[q], dd[o], rtol=1e-13, atol=1e-13)
    if metric == "l2":
        assert list(ids[0][:2]) == [3, 7] and d[0][0] == 0.0


def test_brute_force_subset_and_prefix_dims():
    rng = np.random.default_rng(4)
    X = rng.standard_normal((100, 8)).astype(np.float32)
    Qh = rng.standard_normal((5, 8))
    sub = np.arange(0, 100, 3, dtype=np.int32)
    ids, d = orc.brute_force(Qh, X, 4, ids=sub, dim=5)
    for q in range(5):
        dd = ((X[sub, :5].astype(np.float64) - Qh[q, :5]) ** 2).sum(1)
        o = np.lexsort((sub, dd))[:4]
        assert list(ids[q]) == list(sub[o])


def test_recall_spec_examples():
    gt = np.array([[1, 2, 3, 4]])
    assert orc.recall(np.array([[1, 2, 9, 8]]), gt, 4) == 0.5
    assert orc.recall(gt, gt, 4) == 1.0
    assert orc.recall(np.array([[5, 6, 7, 8]]), gt, 4) == 0.0
    assert orc.recall(np.array([[4, 3, 2, 1]]), gt, 4) == 1.0            # permutation invariance
    # tie-aware (Q25): id 9 at the same distance as gt's last counts
    r = orc.recall(np.array([[1, 2, 3, 9]]), gt, 4, ret_d=np.array([[0.0, 1.0, 2.0, 3.0]]),
                   gt_d=np.array([[0.0, 1.0, 2.0, 3.0]]))
    assert r == 1.0


# ------------------------------------------------------------------ O1 -------
def test_projection_signed_permutation_is_exact():
    D = 10
    perm = np.random.default_rng(5).permutation(D)
    sign = np.where(np.arange(D) % 3 == 0, -1.0, 1.0)
    V = np.zeros((D, D), np.float32)
    V[perm, np.arange(D)] = sign
    Q = np.random.default_rng(6).standard_normal((7, D)).astype(np.float32)
    Qh = orc.project(Q, V)
    assert np.array_equal(Qh, Q[:, perm].astype(np.float64) * sign[None, :])


def test_projection_orthonormal_norms_and_numpy():
    D = 32
    V = orthonormal(D, 9)
    Q = np.random.default_rng(7).standard_normal((11, D)).astype(np.float32)
    Qh = orc.project(Q, V.astype(np.float32))
    np.testing.assert_allclose(Qh, Q.astype(np.float64) @ V.astype(np.float32).astype(np.float64), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose((Qh ** 2).sum(1), (Q.astype(np.float64) ** 2).sum(1), rtol=1e-6)


# ------------------------------------------------------------------ O3 / O4 --
def test_routing_r1_and_centroid_queries():
    inst = tiny_instance(n=120, D=8, dp=8, r=1, m=6, seed=11, V=np.eye(8))
    res = orc.search(inst, k=5, ef=16)
    assert np.all(res["cell"] == 0)
    inst = tiny_instance(n=120, D=8, dp=8, r=6, m=6, seed=12, V=np.eye(8))
    inst["queries"] = inst["fes_centroids"][[3, 0, 5, 1, 2, 4]].copy()   # D = d', V = I
    res = orc.search(inst, k=5, ef=16)
    assert list(res["cell"]) == [3, 0, 5, 1, 2, 4]


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_routing_equals_numpy_argmin(metric):
    inst = tiny_instance(n=300, D=12, dp=6, r=8, m=40, seed=13, metric=metric)
    res = orc.search(inst, k=5, ef=16)
    Qh = inst["queries"].astype(np.float64) @ inst["basis"].astype(np.float64)
    C = inst["fes_centroids"].astype(np.float64)
    if metric == "l2":
        d = ((Qh[:, None, :6] - C[None]) ** 2).sum(2)
    else:
        d = -(Qh[:, :6] @ C.T)
    assert list(res["cell"]) == list(np.argmin(d, 1))


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_fes_r1_is_brute_force_over_pool(metric):
    inst = tiny_instance(n=300, D=12, dp=6, r=1, m=20, seed=14, metric=metric)
    E = 17
    res = orc.search(inst, k=5, ef=32, entries=E)
    Qh = orc.project(inst["queries"], inst["basis"])
    pool = inst["fes_pool_ids"]
    bi, bd = orc.brute_force(Qh, inst["reduced"], E, metric=metric, ids=pool)
    assert np.array_equal(res["entries"], bi)
    np.testing.assert_array_equal(res["entries_d"], bd)
    # independent numpy check of the same set
    for q in range(3):
        X = inst["reduced"][pool].astype(np.float64)
        dd = ((X - Qh[q, :6]) ** 2).sum(1) if metric == "l2" else -(X @ Qh[q, :6])
        o = np.lexsort((pool, dd))[:E]
        assert list(res["entries"][q]) == list(pool[o])


def test_fes_work_matches_table3():
    # Table 3: FES (general) = m·n·d / r for balanced cells; count_fes_work(4,8,2,2)=32
    m, n, d, r = 4, 8, 2, 2
    X = np.array([[0, 0], [0, 1], [1, 0], [1, 1], [10, 10], [10, 11], [11, 10], [11, 11]], np.float32)
    inst = dict(metric="l2", sub_offsets=np.zeros(9, np.int64), sub_neighbors=np.zeros(0, np.int32),
                reduced=X, rotated=X, basis=np.eye(2, dtype=np.float32),
                fes_centroids=np.array([[0.5, 0.5], [10.5, 10.5]], np.float32),
                fes_cell_off=np.array([0, 4, 8]), fes_pool_ids=np.arange(8, dtype=np.int32),
                queries=np.array([[0, 0], [1, 1], [10, 10], [12, 12]], np.float32))
    res = orc.search(inst, k=2, ef=4)
    assert list(res["cell"]) == [0, 0, 1, 1]
    assert int(res["fes_work"].sum()) * d == m * n * d // r == 32
    res1 = orc.search(dict(inst, queries=inst["queries"][:1]), k=2, ef=4)
    assert int(res1["fes_work"][0]) == n // r                            # FES (1 query): n/r


def test_no_fes_uses_pool_order():
    inst = tiny_instance(n=100, D=8, dp=4, r=4, m=3, seed=15)
    res = orc.search(inst, k=3, ef=8, entries=5, flags=orc.NO_FES)
    pool = inst["fes_pool_ids"][:5]
    for q in range(3):
        assert set(res["entries"][q]) == set(pool)


# ------------------------------------------------------------------ O5–O7 ----
def test_single_node_graph_one_distance():
    X = np.array([[1.0, 2.0]], np.float32)
    inst = dict(metric="l2", sub_offsets=np.zeros(2, np.int64), sub_neighbors=np.zeros(0, np.int32),
                reduced=X, rotated=X, basis=np.eye(2, dtype=np.float32),
                fes_centroids=X.copy(), fes_cell_off=np.array([0, 1]), fes_pool_ids=np.array([0], np.int32),
                queries=np.array([[0.0, 0.0]], np.float32))
    res = orc.search(inst, k=3, ef=4)
    assert list(res["ids"][0]) == [0, -1, -1] and res["d"][0][0] == 5.0
    assert res["n_dist1"][0] == 1 and res["n_exp1"][0] == 1


@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("seed", [21, 22, 23])
def test_stage1_ef_ge_n_equals_brute_force(metric, seed):
    """BASELINE north_star: recall must be 1.0 when ef ≥ n (all members reachable)."""
    inst = tiny_instance(n=150, D=10, dp=5, R=6, m=12, seed=seed, metric=metric, member_ratio=0.6)
    nm = int(inst["member_flags"].sum())
    res = orc.search(inst, k=10, ef=nm, entries=4)
    Qh = orc.project(inst["queries"], inst["basis"])
    bi, bd = orc.brute_force(Qh, inst["reduced"], 10, metric=metric, ids=np.flatnonzero(inst["member_flags"]))
    assert np.array_equal(res["ids"], bi)
    np.testing.assert_array_equal(res["d"], bd)
    assert orc.recall(res["ids"], bi, 10) == 1.0
    assert np.all(inst["member_flags"][res["cand1_ids"][res["cand1_ids"] >= 0]] == 1)   # I8


def test_query_equal_member_is_rank1():
    inst = tiny_instance(n=200, D=8, dp=8, R=8, m=4, seed=31, V=np.eye(8))
    inst["queries"] = inst["reduced"][[5, 17, 101, 150]].copy()        # V = I, d' = D
    res = orc.search(inst, k=5, ef=32)
    assert list(res["ids"][:, 0]) == [5, 17, 101, 150]
    assert np.all(res["d"][:, 0] == 0.0)


@pytest.mark.parametrize("ef,w", [(8, 1), (24, 1), (16, 2), (12, 3)])
def test_stage1_invariants_on_traces(ef, w):
    """I1, I2, I4, I5, I6, I7, I8, I9 (SURVEY §8.c "I")."""
    inst = tiny_instance(n=400, D=12, dp=6, R=10, m=20, seed=40 + ef, member_ratio=0.7)
    res = orc.search(inst, k=5, ef=ef, trace_cap=4096, width=w, entries=min(ef, 6))
    Qh = orc.project(inst["queries"], inst["basis"])
    off, nb = inst["sub_offsets"], inst["sub_neighbors"]
    for q in range(20):
        exp = res["trace_expand"][q][:res["trace_nexp"][q]]
        vis = res["trace_visit"][q][:res["trace_nvis"][q]]
        assert len(set(vis)) == len(vis)                                   # I4 no revisits
        assert res["n_dist1"][q] == len(vis)                               # I9
        assert res["n_exp1"][q] == len(exp)
        assert len(set(exp)) == len(exp)                                   # I5 expanded once
        pos = {v: i for i, v in enumerate(vis)}
        assert all(u in pos for u in exp)                                  # I5 expanded ⊂ visited
        visset = set(vis)
        for u in exp:                                                      # I6
            assert set(nb[off[u]:off[u + 1]]) <= visset
        c = res["cand1_ids"][q]
        c = c[c >= 0]
        assert len(c) <= ef and len(set(c)) == len(c)                      # I1, I2
        dd = ((inst["reduced"][vis].astype(np.float64) - Qh[q, :6]) ** 2).sum(1)
        o = np.lexsort((vis, dd))[:ef]                                     # I7 bounded best-first
        assert list(c) == list(np.asarray(vis)[o])
        assert np.all(inst["member_flags"][c] == 1)                        # I8
        # I6: every entry of C is checked (expanded) at termination
        assert set(c) <= set(exp)


# ------------------------------------------------------------------ O8–O9 ----
@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_all_toggles_off_full_ef_is_brute_force(metric):
    inst = tiny_instance(n=120, D=10, dp=4, R=5, m=10, seed=51, metric=metric, member_ratio=0.5)
    res = orc.search(inst, k=10, ef=120, stages=3, flags=orc.NO_FES | orc.NO_STAGE1 | orc.NO_STAGE2,
                     entries=1, ef2=120)
    Qh = orc.project(inst["queries"], inst["basis"])
    bi, bd = orc.brute_force(Qh, inst["rotated"], 10, metric=metric)
    assert np.array_equal(res["ids"], bi)
    np.testing.assert_array_equal(res["d"], bd)


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_full_pipeline_large_ef3_is_brute_force(metric):
    inst = tiny_instance(n=150, D=12, dp=4, R=6, m=10, seed=52, metric=metric, member_ratio=0.4)
    # ef2 ≥ N too: ids evicted from C2 stay visited and never re-enter stage ③ (Q14, Q23)
    res = orc.search(inst, k=10, ef=16, stages=3, ef3=150, ef2=150)
    Qh = orc.project(inst["queries"], inst["basis"])
    bi, _ = orc.brute_force(Qh, inst["rotated"], 10, metric=metric)
    assert orc.recall(res["ids"], bi, 10) == 1.0


def test_stage2_identity_rerank_when_dprime_is_D():
    inst = tiny_instance(n=200, D=8, dp=8, R=6, m=10, seed=53, member_ratio=0.5)
    ef = 20
    r1 = orc.search(inst, k=10, ef=ef, stages=1)
    r3 = orc.search(inst, k=10, ef=ef, stages=3, refine_iters=0, ef2=ef, flags=0)
    # d' = D: full δ == primary δ, so the re-rank keeps the stage-① order
    assert r3["n_exp2"].sum() == 0 and np.all(r3["n_dist2"] == (r1["cand1_ids"] >= 0).sum(1))
    np.testing.assert_allclose(r1["cand1_d"][:, :10], r1["d"], rtol=0)


def test_primary_plus_residual_is_full_distance():
    """δ_full = δ' + δ_res for orthonormal V."""
    inst = tiny_instance(n=100, D=16, dp=5, m=6, seed=54)
    Qh = orc.project(inst["queries"], inst["basis"])
    _, dfull = orc.brute_force(Qh, inst["rotated"], 100)
    _, dprim = orc.brute_force(Qh, inst["rotated"], 100, dim=5)
    ids_f, _ = orc.brute_force(Qh, inst["rotated"], 100)
    X = inst["rotated"].astype(np.float64)
    for q in range(6):
        full = ((X - Qh[q]) ** 2).sum(1)
        prim = ((X[:, :5] - Qh[q, :5]) ** 2).sum(1)
        res = ((X[:, 5:] - Qh[q, 5:]) ** 2).sum(1)
        np.testing.assert_allclose(full, prim + res, rtol=1e-12)
        np.testing.assert_allclose(dfull[q], full[ids_f[q]], rtol=1e-13)


def test_carry_with_true_topk_gives_recall_one():
    inst = tiny_instance(n=200, D=10, dp=10, R=6, m=8, seed=55, V=np.eye(10))
    Qh = orc.project(inst["queries"], inst["basis"])
    bi, _ = orc.brute_force(Qh, inst["rotated"], 10)
    # entries = true top-10 (FES off, pool = those ids is per query; use one query at a time)
    for q in range(8):
        one = dict(inst, queries=inst["queries"][q:q + 1], fes_pool_ids=np.sort(bi[q]).astype(np.int32),
                   fes_cell_off=np.array([0, 10]), fes_centroids=inst["fes_centroids"][:1])
        res = orc.search(one, k=10, ef=10, stages=3, flags=orc.NO_FES | orc.NO_STAGE1, entries=10, ef2=10)
        assert orc.recall(res["ids"], bi[q:q + 1], 10) == 1.0


def test_multithread_equals_single_thread(s1):
    a = orc.search(s1, k=10, ef=32, stages=1, threads=1)
    b = orc.search(s1, k=10, ef=32, stages=1, threads=8)
    for key in ("ids", "d", "cand1_ids", "counters", "entries"):
        assert np.array_equal(a[key], b[key])


# ------------------------------------------------------------ O13 bloom -----
# The stage-① visited set as the paper's bloom filter,
# partitioned into 3 segments of 2^s bits (reading Q17b).
def _bloom_inst(seed=70):
    return tiny_instance(n=600, D=12, dp=6, R=10, m=16, seed=seed, member_ratio=0.8)


def test_bloom_huge_filter_equals_exact_visited():
    """With 3 × 2^20 bits and ≤ 600 inserts a false positive has probability
    < 1e-9 per test, so the bloom search must reproduce the exact-set search
    (itself pinned by the goldens / brute force above) trace for trace."""
    inst = _bloom_inst()
    a = orc.search(inst, k=10, ef=24, trace_cap=4096, entries=6)
    b = orc.search(inst, k=10, ef=24, trace_cap=4096, entries=6, bloom_log2=20)
    for key in ("cand1_ids", "cand1_d", "trace_expand", "trace_visit", "trace_nexp", "trace_nvis", "n_dist1"):
        np.testing.assert_array_equal(a[key], b[key])


def test_bloom_all_positive_filter_keeps_only_entries():
    """a filter that answers 'visited' for everything (s = 0: one bit per
    segment, set by the first entry) leaves C = the entries — the same list as
    the no-stage-① toggle (pinned above)."""
    inst = _bloom_inst(71)
    b = orc.search(inst, k=5, ef=16, entries=8, trace_cap=256, bloom_log2=0)
    t = orc.search(inst, k=5, ef=16, entries=8, flags=orc.NO_STAGE1)
    np.testing.assert_array_equal(b["cand1_ids"], t["cand1_ids"])
    assert np.all(b["n_dist1"] == 8) and np.all(b["trace_nvis"] == 8)


def test_bloom_no_false_negatives_and_fp_rate():
    """No false negatives: no id is ever visited twice.  False-positive
    rate: replaying each trace against the true visited set, a fresh neighbour
    tested after n inserts is skipped with probability (1 − (1 − 2^−s)^n)^3 for
    three independent uniform segment hashes; the observed skip count must match
    the sum of these probabilities within 5σ (a test that required any ONE bit,
    or a single shared segment, would be off by many σ)."""
    inst = _bloom_inst(72)
    s = 7
    res = orc.search(inst, k=10, ef=32, trace_cap=8192, entries=6, bloom_log2=s)
    off, nb = inst["sub_offsets"], inst["sub_neighbors"]
    exp_fp, var, obs, tests = 0.0, 0.0, 0, 0
    for q in range(inst["queries"].shape[0]):
        vis = list(res["trace_visit"][q][:res["trace_nvis"][q]])
        assert len(set(vis)) == len(vis)                                   # no revisits
        E = 6
        T = set(vis[:E])
        nxt = E
        for u in res["trace_expand"][q][:res["trace_nexp"][q]]:
            for v in nb[off[u]:off[u + 1]]:
                if v in T:
                    continue
                p = (1.0 - (1.0 - 2.0 ** -s) ** len(T)) ** 3
                tests += 1
                exp_fp += p
                var += p * (1 - p)
                if nxt < len(vis) and vis[nxt] == v:
                    T.add(v)
                    nxt += 1
                else:
                    obs += 1                                               # skipped: false positive
        assert nxt == len(vis)
    assert tests > 2000 and exp_fp > 20
    assert abs(obs - exp_fp) <= 5 * np.sqrt(var), (obs, exp_fp, var)


def test_bloom_stage1_invariants():
    """I1, I2, I7 (C = the ef best of what was visited), I8, I9 hold under FPs."""
    inst = _bloom_inst(73)
    ef = 16
    res = orc.search(inst, k=5, ef=ef, trace_cap=4096, entries=5, bloom_log2=7)
    Qh = orc.project(inst["queries"], inst["basis"])
    for q in range(inst["queries"].shape[0]):
        vis = res["trace_visit"][q][:res["trace_nvis"][q]]
        assert res["n_dist1"][q] == len(vis)
        c = res["cand1_ids"][q]
        c = c[c >= 0]
        dd = ((inst["reduced"][vis].astype(np.float64) - Qh[q, :6]) ** 2).sum(1)
        assert list(c) == list(np.asarray(vis)[np.lexsort((vis, dd))[:ef]])
        assert np.all(inst["member_flags"][c] == 1)


# ------------------------------------------------ O8–O9 hand-derived golden --
@pytest.mark.parametrize("name", __import__("conftest").golden23_names())
def test_stage23_golden(name):
    """O8 pinned (VERDICT r1 'What's weak' #1): a hand-derived stages-②③ trace on
    a fixture whose subgraph differs from the full graph and whose d' < D — the
    final top-k and all six stage counters (tests/golden23/, derivation inside)."""
    from conftest import instance_from_golden23, load_golden23
    g = load_golden23(name)
    inst = instance_from_golden23(g)
    r = orc.search(inst, k=g["k"], ef=g["ef1"], stages=3, entries=g["entries"], ef1=g["ef1"], ef2=g["ef2"],
                   ef3=g["ef3"], refine_iters=g["refine_iters"])
    assert list(r["ids"][0]) == g["result_ids"]
    assert list(r["d"][0]) == g["result_d"]
    for key, v in g["counters"].items():
        assert int(r[key][0]) == v, key
