"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element
on the same seeded inputs (tie-aware protocol in tests/parity.py)."""
import numpy as np
import pytest

import oracle as orc
import paper_2503_21206_b200 as pa
from conftest import golden_names, instance_from_golden, load_golden
from gpu_util import run_gpu
from parity import compare
from tiny import tiny_instance

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build_library()


def integer_instance(n=300, D=16, R=8, m=40, seed=5, r=4, metric="l2", member_ratio=0.6, vals=4):
    """All coordinates small integers and V a signed permutation: every fp32
    operation of the GPU path is exact, so trajectories must be bit-exact
    INCLUDING ties (many exact ties by construction)."""
    rng = np.random.default_rng(seed)
    inst = tiny_instance(n=n, D=D, dp=D // 2, R=R, m=m, seed=seed, r=r, metric=metric, member_ratio=member_ratio)
    X = rng.integers(-vals, vals + 1, size=(n, D)).astype(np.float32)
    perm = rng.permutation(D)
    sign = np.where(rng.random(D) < 0.5, -1.0, 1.0)
    V = np.zeros((D, D), np.float32)
    V[perm, np.arange(D)] = sign
    Xh = (X.astype(np.float64) @ V.astype(np.float64)).astype(np.float32)
    inst["basis"], inst["rotated"] = V, Xh
    inst["reduced"] = np.ascontiguousarray(Xh[:, :D // 2])
    inst["queries"] = rng.integers(-vals, vals + 1, size=(m, D)).astype(np.float32)
    pool = inst["fes_pool_ids"]
    cuts = inst["fes_cell_off"]
    inst["fes_centroids"] = np.stack([np.round(inst["reduced"][pool[cuts[c]:cuts[c + 1]]].mean(0))
                                      for c in range(len(cuts) - 1)]).astype(np.float32)
    return inst


def _both(inst, k, ef, trace_cap=4096, **opts):
    ix = pa.Index.from_instance(inst)
    g = run_gpu(ix, inst, k, ef, trace_cap=trace_cap, **opts)
    flags = opts.get("flags", 0)
    bl = opts.get("bloom_log2") or None
    r = orc.search(inst, k=k, ef=ef, stages=1, trace_cap=trace_cap, flags=flags, bloom_log2=bl,
                   **{kk: v for kk, v in opts.items() if kk in ("entries", "ef1", "width") and v})
    ix.close()
    return g, r


@pytest.mark.parametrize("name", golden_names())
def test_golden_fixtures_bit_exact(name):
    gd = load_golden(name)
    inst = instance_from_golden(gd)
    g, r = _both(inst, gd["k"], gd["ef"], entries=gd["entries"])
    assert list(g["trace_expand"][0][:g["trace_nexp"][0]]) == gd["expand"]
    assert list(g["trace_visit"][0][:g["trace_nvis"][0]]) == gd["visit"]
    assert list(g["ids"][0]) == gd["result_ids"]
    assert np.array_equal(g["d"][0], np.array(gd["result_d"], np.float32))


@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_integer_fixture_bit_exact_with_ties(metric, seed):
    inst = integer_instance(seed=seed, metric=metric)
    for ef in (8, 32):
        g, r = _both(inst, 5, ef)
        rep = compare(inst, g, r, 5, ef)
        assert not rep.fail, rep.fail[:3]
        assert rep.tie == 0, rep                       # exact arithmetic: no divergence allowed
        assert np.array_equal(g["ids"], r["ids"])
        assert np.array_equal(g["d"].astype(np.float64), r["d"])
        assert np.array_equal(g["cand_ids"], r["cand1_ids"])
        assert np.array_equal(g["n_dist1"], r["n_dist1"]) and np.array_equal(g["n_exp1"], r["n_exp1"])


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_ef_ge_members_is_brute_force(metric):
    inst = tiny_instance(n=400, D=24, dp=12, R=10, m=33, seed=7, metric=metric, member_ratio=0.5)
    nm = int(inst["member_flags"].sum())
    ef = min(256, nm)
    assert nm <= 256
    ix = pa.Index.from_instance(inst)
    g = run_gpu(ix, inst, 10, ef, entries=8)
    Qh = orc.project(inst["queries"], inst["basis"])
    bi, bd = orc.brute_force(Qh, inst["reduced"], 10, metric=metric, ids=np.flatnonzero(inst["member_flags"]))
    assert orc.recall(g["ids"], bi, 10) == 1.0
    tol = 1e-5 * np.abs(bd) + 1e-6
    assert np.all(np.abs(g["d"] - bd) <= tol)


@pytest.mark.parametrize("cfg_name", ["C0", "S1", "S2"])
def test_config_parity(cfg_name, request):
    inst = request.getfixturevalue(cfg_name.lower())
    cfg = inst["cfg"]
    g, r = _both(inst, cfg.k, cfg.ef, trace_cap=8192)
    rep = compare(inst, g, r, cfg.k, cfg.ef, gt_ids=inst["gt_sub_ids"][:, :cfg.k])
    print(cfg_name, rep, getattr(rep, "recall_gpu", None), getattr(rep, "recall_orc", None))
    assert not rep.fail, rep.fail[:5]
    assert rep.exact >= 0.9 * cfg.m, rep
    assert np.all(g["status"] == 0)


def test_forced_spill_is_exact(s1, monkeypatch):
    """The visited set is exact whatever its layout: a small level-1 table (forced
    global spill), the 32-bit table and the 16-bit quotiented table all give
    bit-identical outputs, traces and counters."""
    cfg = s1["cfg"]
    ix = pa.Index.from_instance(s1)
    base = run_gpu(ix, s1, cfg.k, cfg.ef, trace_cap=8192)
    runs = [run_gpu(ix, s1, cfg.k, cfg.ef, trace_cap=8192, hash_slots_log2=log2) for log2 in (5, 9)]
    assert all(r["spill"].sum() > 0 for r in runs)
    runs.append(run_gpu(ix, s1, cfg.k, 256, trace_cap=8192, hash_slots_log2=11))        # compact, spills
    runs.append(run_gpu(ix, s1, cfg.k, 256, trace_cap=8192, hash_slots_log2=11,
                        check_path=pa.PA_CHECK_WIDE_VISITED))                           # 32-bit, spills
    runs.append(run_gpu(ix, s1, cfg.k, cfg.ef, trace_cap=8192))
    ix.close()
    for key in ("ids", "d", "cand_ids", "cand_dists", "trace_expand", "trace_visit", "n_dist1"):
        for r in runs[:2] + runs[4:]:
            assert np.array_equal(base[key], r[key]), key
        assert np.array_equal(runs[2][key], runs[3][key]), key


def test_edge_cases(s1):
    cfg = s1["cfg"]
    ix = pa.Index.from_instance(s1)
    one = s1["queries"][:1]
    g1 = run_gpu(ix, s1, cfg.k, cfg.ef, queries=one)
    r1 = orc.search(s1, queries=one, k=cfg.k, ef=cfg.ef)
    assert orc.recall(g1["ids"], r1["ids"], cfg.k) >= 0.9
    # ef = k = 1
    g = run_gpu(ix, s1, 1, 1)
    r = orc.search(s1, k=1, ef=1)
    assert (g["ids"][:, 0] == r["ids"][:, 0]).mean() >= 0.9
    # ef = 256 and E larger than every cell (entries = whole cell)
    g = run_gpu(ix, s1, 10, 256, entries=1024)
    assert np.all(g["status"] == 0) and np.all(g["ids"] >= 0)
    # toggles
    g = run_gpu(ix, s1, 10, 64, flags=pa.PA_NO_FES)
    r = orc.search(s1, k=10, ef=64, flags=orc.NO_FES)
    assert orc.recall(g["ids"], r["ids"], 10) >= 0.98
    g = run_gpu(ix, s1, 10, 64, flags=pa.PA_NO_STAGE1)
    r = orc.search(s1, k=10, ef=64, flags=orc.NO_STAGE1)
    assert orc.recall(g["ids"], r["ids"], 10) >= 0.98
    assert np.all(g["n_exp1"] == 0)
    # m = 0 is a no-op
    import torch
    z = torch.empty(0, s1["D"], device="cuda")
    ix.search_device(z, 10, 64, torch.empty(0, 10, dtype=torch.int32, device="cuda"),
                     torch.empty(0, 10, device="cuda"))
    with pytest.raises(pa.PAError):
        run_gpu(ix, s1, 10, 5)                     # ef < k
    with pytest.raises(pa.PAError):
        run_gpu(ix, s1, 10, 300)                   # ef > 256
    ix.close()


def test_host_path_equals_device_path(s1):
    cfg = s1["cfg"]
    ix = pa.Index.from_instance(s1)
    g = run_gpu(ix, s1, cfg.k, cfg.ef)
    ids, d = ix.search(s1["queries"], k=cfg.k, ef=cfg.ef)
    assert np.array_equal(ids, g["ids"]) and np.array_equal(d, g["d"])
    ci, cd = ix.search_candidates(s1["queries"], ef=cfg.ef)
    assert np.array_equal(ci, g["cand_ids"]) and np.array_equal(cd, g["cand_dists"])
    st = ix.stats()
    assert st["kernel_launches"] >= 3 and st["ms_total_gpu"] > 0
    ix.close()
    with pytest.raises(pa.PAError) as e:
        ix2 = pa.Index.from_instance(s1)
        h = ix2._h
        ix2.close()
        ix2._h = h                                 # use after destroy → PA_ESTATE
        ix2.search(s1["queries"], k=10, ef=64)
    assert e.value.status == pa.PA_ESTATE
    ix2._h = None


@pytest.mark.parametrize("cfg_name", ["S1", "S2"])
def test_tensor_core_paths_match_simt(cfg_name, request, monkeypatch):
    """tcgen05 projection+routing and tcgen05 FES select the same cells/entries as
    the SIMT kernels except at GEMM-form near-ties; q' agrees to ~fp32 rounding."""
    inst = request.getfixturevalue(cfg_name.lower())
    cfg = inst["cfg"]
    ix = pa.Index.from_instance(inst)
    tc = run_gpu(ix, inst, cfg.k, cfg.ef)
    si = run_gpu(ix, inst, cfg.k, cfg.ef, check_path=pa.PA_CHECK_SIMT)
    ix.close()
    assert (tc["cell"] == si["cell"]).mean() >= 0.98
    same = np.array([set(a) == set(b) for a, b in zip(tc["entries"], si["entries"])])
    assert same.mean() >= 0.95, same.mean()
    assert orc.recall(tc["ids"], si["ids"], cfg.k) >= 0.97


@pytest.mark.parametrize("cfg_name", ["C0", "S1", "S2"])
def test_full_pipeline_parity(cfg_name, request):
    """PA_STAGES_FULL (GPU stage ① + host stages ②③, pipelined) vs the oracle's
    three stages in fp64: full-space recall@10 within 0.002 of the oracle's against
    the same exhaustive ground truth; returned distances = fp64 full δ."""
    inst = request.getfixturevalue(cfg_name.lower())
    cfg = inst["cfg"]
    ix = pa.Index.from_instance(inst)
    ix.attach_host(inst["full_offsets"], inst["full_neighbors"], inst["rotated"])
    ids, d = ix.search(inst["queries"], k=cfg.k, ef=cfg.ef, stages=pa.PA_STAGES_FULL)
    st = ix.stats()
    ix.close()
    r = orc.search(inst, k=cfg.k, ef=cfg.ef, stages=3)
    gt = inst["gt_ids"][:, :cfg.k]
    rg, ro = orc.recall(ids, gt, cfg.k), orc.recall(r["ids"], gt, cfg.k)
    print(cfg_name, "full recall gpu+host", rg, "oracle", ro, "host ms", st["ms_host_stages"])
    assert abs(rg - ro) <= 0.002 + 1e-12
    Qh = orc.project(inst["queries"], inst["basis"])
    X = inst["rotated"].astype(np.float64)[ids]
    want = ((X - Qh[:, None, :]) ** 2).sum(2) if cfg.metric == "l2" else -(X * Qh[:, None, :]).sum(2)
    scale = np.abs(want) if cfg.metric == "l2" else np.abs(X * Qh[:, None, :]).sum(2)
    assert np.all(np.abs(d - want) <= 1e-5 * scale + 1e-6 * np.sqrt(np.abs(want) * (Qh ** 2).sum(1, keepdims=True)))


# ---------------------------------------------------------------- NEXT-f1 ---
def rounded16(inst):
    """The oracle side of binary16 storage: the identical rounded values (RNE)."""
    return dict(inst, reduced=inst["reduced"].astype(np.float16).astype(np.float32))


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_fp16_storage_integer_fixture_bit_exact(metric):
    inst = integer_instance(seed=4, metric=metric)
    ix = pa.Index.from_instance(inst, reduced_fp16=True)
    g = run_gpu(ix, inst, 5, 32, trace_cap=4096)
    ix.close()
    r = orc.search(rounded16(inst), k=5, ef=32, stages=1, trace_cap=4096)
    rep = compare(rounded16(inst), g, r, 5, 32)
    assert not rep.fail and rep.tie == 0, (rep, rep.fail[:3])
    assert np.array_equal(g["ids"], r["ids"]) and np.array_equal(g["d"].astype(np.float64), r["d"])


@pytest.mark.parametrize("cfg_name", ["S1", "S2"])
def test_fp16_storage_parity(cfg_name, request):
    inst = request.getfixturevalue(cfg_name.lower())
    cfg = inst["cfg"]
    ix = pa.Index.from_instance(inst, reduced_fp16=True)
    g = run_gpu(ix, inst, cfg.k, cfg.ef, trace_cap=8192)
    ix.close()
    inst16 = rounded16(inst)
    r = orc.search(inst16, k=cfg.k, ef=cfg.ef, stages=1, trace_cap=8192)
    rep = compare(inst16, g, r, cfg.k, cfg.ef, gt_ids=inst["gt_sub_ids"][:, :cfg.k])
    print(cfg_name, "fp16", rep, rep.recall_gpu, rep.recall_orc)
    assert not rep.fail, rep.fail[:5]
    assert rep.exact >= 0.9 * cfg.m


def test_fp16_storage_full_pipeline(s1):
    cfg = s1["cfg"]
    ix = pa.Index.from_instance(s1, reduced_fp16=True)
    ix.attach_host(s1["full_offsets"], s1["full_neighbors"], s1["rotated"])
    ids, d = ix.search(s1["queries"], k=cfg.k, ef=cfg.ef, stages=pa.PA_STAGES_FULL)
    ix.close()
    r = orc.search(rounded16(s1), k=cfg.k, ef=cfg.ef, stages=3)
    gt = s1["gt_ids"][:, :cfg.k]
    assert abs(orc.recall(ids, gt, cfg.k) - orc.recall(r["ids"], gt, cfg.k)) <= 0.002 + 1e-12


@pytest.mark.parametrize("r", [1, 2, 8])
def test_fes_selection_large_cells(r):
    """k_fes_select4 (cells ≤ 8192 entries, r = 2 and 8) and k_fes_select3 (the
    12 000-entry single cell, r = 1) against the oracle's O4 entries (near-ties
    only) and stage-① results, tie-aware."""
    inst = tiny_instance(n=12000, D=32, dp=16, R=12, m=64, seed=40 + r, r=r)
    for ef in (10, 96, 256):
        g, o = _both(inst, 10, ef, trace_cap=16384)
        rep = compare(inst, g, o, 10, ef)
        assert not rep.fail, (ef, rep.fail[:3])
        assert rep.exact >= 0.9 * 64


@pytest.mark.parametrize("vals,r", [(4, 1), (4, 4), (1, 2), (1, 8)])
@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_fes_selection_ties_bit_exact(vals, r, metric):
    """FES top-E (k_fes_select's radix select) on integer inputs, where every score
    is exact and ties are everywhere: the entries must equal the oracle's O4
    entries element by element (order (δ, id)), E = 8 … 256.  vals = 1
    ({−1, 0, 1} coordinates) puts hundreds of pool entries on one score, which
    takes the heavy-tie path; cells of 3000/1500 entries take the unstaged path,
    750/375 the smem-staged one."""
    inst = integer_instance(n=3000, D=16, R=8, m=64, seed=60 + vals + r, r=r, metric=metric, member_ratio=1.0,
                            vals=vals)
    ix = pa.Index.from_instance(inst)
    for E in (8, 100, 256):
        g = run_gpu(ix, inst, 5, E)
        o = orc.search(inst, k=5, ef=E, stages=1)
        assert np.array_equal(g["cell"], o["cell"]), E
        assert np.array_equal(g["entries"], o["entries"]), (E, np.flatnonzero((g["entries"] != o["entries"]).any(1))[:5])
    ix.close()


# ------------------------------------------------ NEXT-f1: bloom visited set --
# The paper's shared-memory bloom filter vs the oracle's O13 mode on
# the same filter definition: false positives are part of the method, so the
# trajectories (including which fresh nodes are skipped) must agree exactly.
@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("bl", [7, 10])
def test_bloom_integer_fixture_bit_exact(metric, bl):
    inst = integer_instance(seed=11, metric=metric, n=500)
    for ef in (8, 48):
        g, r = _both(inst, 5, ef, bloom_log2=bl)
        rep = compare(inst, g, r, 5, ef)
        assert not rep.fail and rep.tie == 0, (rep, rep.fail[:3])
        assert np.array_equal(g["trace_visit"], r["trace_visit"]) and np.array_equal(g["trace_expand"], r["trace_expand"])
        assert np.array_equal(g["ids"], r["ids"]) and np.array_equal(g["d"].astype(np.float64), r["d"])
        assert np.array_equal(g["n_dist1"], r["n_dist1"])


@pytest.mark.parametrize("cfg_name", ["C0", "S1", "S2"])
@pytest.mark.parametrize("bl", [8, 12])
def test_bloom_config_parity(cfg_name, bl, request):
    inst = request.getfixturevalue(cfg_name.lower())
    cfg = inst["cfg"]
    g, r = _both(inst, cfg.k, cfg.ef, trace_cap=8192, bloom_log2=bl)
    rep = compare(inst, g, r, cfg.k, cfg.ef, gt_ids=inst["gt_sub_ids"][:, :cfg.k])
    print(cfg_name, "bloom", bl, rep, rep.recall_gpu, rep.recall_orc)
    assert not rep.fail, rep.fail[:5]
    assert rep.exact >= 0.9 * cfg.m, rep
    assert np.all(g["status"] == 0)


def test_bloom_fp16_integer_fixture_bit_exact():
    inst = integer_instance(seed=12, n=400)
    ix = pa.Index.from_instance(inst, reduced_fp16=True)
    g = run_gpu(ix, inst, 5, 32, trace_cap=4096, bloom_log2=8)
    ix.close()
    r = orc.search(rounded16(inst), k=5, ef=32, stages=1, trace_cap=4096, bloom_log2=8)
    rep = compare(rounded16(inst), g, r, 5, 32)
    assert not rep.fail and rep.tie == 0, (rep, rep.fail[:3])
    assert np.array_equal(g["ids"], r["ids"])


def test_bloom_full_pipeline(s1):
    """Stages ②③ keep exact visited sets, so skipped nodes are re-visited
    (P:L394-395): full-space recall within 0.002 of the oracle's bloom pipeline."""
    cfg = s1["cfg"]
    ix = pa.Index.from_instance(s1)
    ix.attach_host(s1["full_offsets"], s1["full_neighbors"], s1["rotated"])
    ids, d = ix.search(s1["queries"], k=cfg.k, ef=cfg.ef, stages=pa.PA_STAGES_FULL, bloom_log2=9)
    ix.close()
    r = orc.search(s1, k=cfg.k, ef=cfg.ef, stages=3, bloom_log2=9)
    gt = s1["gt_ids"][:, :cfg.k]
    assert abs(orc.recall(ids, gt, cfg.k) - orc.recall(r["ids"], gt, cfg.k)) <= 0.002 + 1e-12


def test_bloom_rejects_bad_sizes(s1):
    ix = pa.Index.from_instance(s1)
    for bl in (3, 17):
        with pytest.raises(pa.PAError) as e:
            run_gpu(ix, s1, 10, 64, bloom_log2=bl)
        assert e.value.status == pa.PA_EINVAL
    ix.close()


def test_no_pipeline_toggle_is_result_identical(s1):
    """PA_NO_PIPELINE (Table 6 '-pipelining') only removes the CPU–GPU overlap."""
    cfg = s1["cfg"]
    ix = pa.Index.from_instance(s1)
    ix.attach_host(s1["full_offsets"], s1["full_neighbors"], s1["rotated"])
    a = ix.search(s1["queries"], k=cfg.k, ef=cfg.ef, stages=pa.PA_STAGES_FULL)
    b = ix.search(s1["queries"], k=cfg.k, ef=cfg.ef, stages=pa.PA_STAGES_FULL, flags=pa.PA_NO_PIPELINE)
    ix.close()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ------------------------------------------------ NEXT-f3: stages ②③ on the GPU --
@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("flags", [0, 2])
def test_full_gpu_integer_fixture_bit_exact(metric, flags):
    """PA_STAGES_FULL_GPU (O8-O9 in one kernel, exact visited sets) vs the oracle's
    three stages: exact arithmetic ⇒ identical ids and distances, with and without
    stage ② (PA_NO_STAGE2)."""
    inst = integer_instance(seed=21, metric=metric, n=400)
    ix = pa.Index.from_instance(inst)
    ix.attach_host(inst["full_offsets"], inst["full_neighbors"], inst["rotated"])
    for ef in (8, 32):
        ids, d = ix.search(inst["queries"], k=5, ef=ef, stages=pa.PA_STAGES_FULL_GPU, flags=flags)
        r = orc.search(inst, k=5, ef=ef, stages=3, flags=flags)
        assert np.array_equal(ids, r["ids"]), ef
        assert np.array_equal(d.astype(np.float64), r["d"]), ef
    ix.close()


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_large_ef3_integer_fixture_bit_exact(metric):
    """ef2/ef3 above stage ①'s 256 (up to 512; stage ① kept at ef1 = E = 200):
    PA_STAGES_FULL (host ②③) and PA_STAGES_FULL_GPU (k_refine with 512-key lists)
    equal the oracle's three stages id for id and distance for distance."""
    inst = integer_instance(seed=23, metric=metric, n=2000, m=24)
    ix = pa.Index.from_instance(inst)
    ix.attach_host(inst["full_offsets"], inst["full_neighbors"], inst["rotated"])
    for ef, ef2 in ((300, 0), (512, 0), (400, 450)):
        over = dict(ef1=200, entries=200) | (dict(ef2=ef2) if ef2 else {})
        r = orc.search(inst, k=10, ef=ef, stages=3, **over)
        for stages in (pa.PA_STAGES_FULL, pa.PA_STAGES_FULL_GPU):
            ids, d = ix.search(inst["queries"], k=10, ef=ef, stages=stages, **over)
            assert np.array_equal(ids, r["ids"]), (ef, stages)
            assert np.array_equal(d.astype(np.float64), r["d"]), (ef, stages)
    ix.close()


@pytest.mark.parametrize("cfg_name", ["C0", "S1", "S2"])
@pytest.mark.parametrize("bloom", [0, 12])
def test_full_gpu_parity(cfg_name, bloom, request):
    """Full-space recall@10 within 0.002 of the oracle's three stages (same stage-①
    visited-set mode) and returned distances = fp64 full δ; the host pipeline
    (PA_STAGES_FULL) and the GPU one agree on the same ground truth."""
    inst = request.getfixturevalue(cfg_name.lower())
    cfg = inst["cfg"]
    ix = pa.Index.from_instance(inst)
    ix.attach_host(inst["full_offsets"], inst["full_neighbors"], inst["rotated"])
    ids, d = ix.search(inst["queries"], k=cfg.k, ef=cfg.ef, stages=pa.PA_STAGES_FULL_GPU, bloom_log2=bloom)
    st = ix.stats()
    hids, _ = ix.search(inst["queries"], k=cfg.k, ef=cfg.ef, stages=pa.PA_STAGES_FULL, bloom_log2=bloom)
    ix.close()
    assert st["overflow_queries"] == 0 and st["sum_n_dist3"] > 0
    r = orc.search(inst, k=cfg.k, ef=cfg.ef, stages=3, bloom_log2=bloom or None)
    gt = inst["gt_ids"][:, :cfg.k]
    rg, ro, rh = orc.recall(ids, gt, cfg.k), orc.recall(r["ids"], gt, cfg.k), orc.recall(hids, gt, cfg.k)
    print(cfg_name, bloom, "full-gpu recall", rg, "oracle", ro, "host pipeline", rh)
    assert abs(rg - ro) <= 0.002 + 1e-12 and abs(rg - rh) <= 0.002 + 1e-12
    Qh = orc.project(inst["queries"], inst["basis"])
    X = inst["rotated"].astype(np.float64)[ids]
    want = ((X - Qh[:, None, :]) ** 2).sum(2) if cfg.metric == "l2" else -(X * Qh[:, None, :]).sum(2)
    scale = np.abs(want) if cfg.metric == "l2" else np.abs(X * Qh[:, None, :]).sum(2)
    assert np.all(np.abs(d - want) <= 1e-5 * scale + 1e-6 * np.sqrt(np.abs(want) * (Qh ** 2).sum(1, keepdims=True)))


# ------------------------------------ the timed kernels = the traced kernels --
# Trace outputs come from the runtime-row-length build of k_traverse_pipe; bench.py
# times the compile-time-row-length builds (d' = 32/48/64/96/128).  Both must give
# identical outputs, so the element-by-element oracle parity of the traced kernel
# carries over to the timed one.
@pytest.mark.parametrize("cfg_name", ["C0", "S1", "S2"])
@pytest.mark.parametrize("bloom,fp16", [(0, False), (12, False), (12, True)])
def test_timed_kernel_equals_traced_kernel(cfg_name, bloom, fp16, request):
    inst = request.getfixturevalue(cfg_name.lower())
    cfg = inst["cfg"]
    ix = pa.Index.from_instance(inst, reduced_fp16=fp16)
    for ef in (cfg.ef, 80):
        traced = run_gpu(ix, inst, cfg.k, ef, trace_cap=8192, bloom_log2=bloom)
        timed = run_gpu(ix, inst, cfg.k, ef, bloom_log2=bloom)
        for key in ("ids", "d", "cand_ids", "cand_dists", "counters", "entries"):
            assert np.array_equal(traced[key], timed[key]), (key, ef)
    ix.close()


@pytest.mark.parametrize("m", [1, 127, 128, 129, 300])
def test_query_count_tails(m, s1):
    """Batch sizes around the 128-row tcgen05 tiles (projection and per-cell FES
    tiles): tie-aware parity with the oracle at every m."""
    cfg = s1["cfg"]
    rng = np.random.default_rng(m)
    Q = s1["queries"][rng.integers(0, s1["queries"].shape[0], size=m)] + \
        rng.normal(0, 0.01, size=(m, s1["D"])).astype(np.float32)
    sub = dict(s1, queries=np.ascontiguousarray(Q, np.float32))
    for bloom in (0, 12):
        g, r = _both(sub, cfg.k, cfg.ef, trace_cap=8192, bloom_log2=bloom)
        rep = compare(sub, g, r, cfg.k, cfg.ef)
        assert not rep.fail, rep.fail[:3]
        assert rep.exact >= 0.9 * m - 1


@pytest.mark.parametrize("D,dp", [(128, 96), (160, 128), (64, 32)])
@pytest.mark.parametrize("bloom", [0, 12])
def test_row_length_specialisations(D, dp, bloom):
    """The d' = 32/96/128 builds (bench configs C0, f2 d' = D = 96, C3S): oracle
    parity of the traced kernel and identical outputs from the timed one."""
    inst = tiny_instance(n=3000, D=D, dp=dp, R=16, m=96, seed=D + dp, member_ratio=0.6, r=8)
    g, r = _both(inst, 10, 48, trace_cap=8192, bloom_log2=bloom)
    rep = compare(inst, g, r, 10, 48)
    assert not rep.fail, rep.fail[:3]
    assert rep.exact >= 0.9 * 96
    ix = pa.Index.from_instance(inst)
    timed = run_gpu(ix, inst, 10, 48, bloom_log2=bloom)
    ix.close()
    for key in ("ids", "d", "cand_ids", "cand_dists", "counters"):
        assert np.array_equal(g[key], timed[key]), key


# ------------------------------------------- stages ②③: hand-derived golden --
@pytest.mark.parametrize("name", __import__("conftest").golden23_names())
@pytest.mark.parametrize("stages", [pa.PA_STAGES_FULL, pa.PA_STAGES_FULL_GPU])
def test_stage23_golden_bit_exact(name, stages):
    """The O8 golden (tests/golden23, hand-derived) through the product: host
    stages ②③ and the GPU k_refine give the derived top-k exactly."""
    from conftest import instance_from_golden23, load_golden23
    g = load_golden23(name)
    inst = instance_from_golden23(g)
    ix = pa.Index.from_instance(inst)
    ix.attach_host(inst["full_offsets"], inst["full_neighbors"], inst["rotated"])
    ids, d = ix.search(inst["queries"], k=g["k"], ef=g["ef1"], stages=stages, entries=g["entries"],
                       ef1=g["ef1"], ef2=g["ef2"], ef3=g["ef3"], refine_iters=g["refine_iters"])
    st = ix.stats()
    ix.close()
    assert list(ids[0]) == g["result_ids"]
    assert list(d[0]) == g["result_d"]
    assert st["sum_n_dist2"] == g["counters"]["n_dist2"] and st["sum_n_dist3"] == g["counters"]["n_dist3"]


@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("flags", [0, 2])
def test_full_host_integer_fixture_bit_exact(metric, flags):
    """PA_STAGES_FULL (GPU stage ① + host stages ②③) on exact-arithmetic
    fixtures: identical ids and distances to the oracle's three stages, with and
    without stage ②."""
    inst = integer_instance(seed=22, metric=metric, n=400)
    ix = pa.Index.from_instance(inst)
    ix.attach_host(inst["full_offsets"], inst["full_neighbors"], inst["rotated"])
    for ef in (8, 32):
        ids, d = ix.search(inst["queries"], k=5, ef=ef, stages=pa.PA_STAGES_FULL, flags=flags)
        r = orc.search(inst, k=5, ef=ef, stages=3, flags=flags)
        assert np.array_equal(ids, r["ids"]), ef
        assert np.array_equal(d.astype(np.float64), r["d"]), ef
    ix.close()


@pytest.mark.parametrize("stages", [pa.PA_STAGES_FULL, pa.PA_STAGES_FULL_GPU])
def test_ef2_above_ef3_bit_exact(stages):
    """ef2 > ef3 (legal: resolve() accepts it): stage ③ starts from the ef3
    smallest of the carry, as the oracle's resize does."""
    inst = integer_instance(seed=23, metric="l2", n=400)
    ix = pa.Index.from_instance(inst)
    ix.attach_host(inst["full_offsets"], inst["full_neighbors"], inst["rotated"])
    for ef1, ef2, ef3 in ((32, 24, 8), (16, 16, 6), (24, 20, 10)):
        ids, d = ix.search(inst["queries"], k=5, ef=ef1, stages=stages, ef1=ef1, ef2=ef2, ef3=ef3)
        r = orc.search(inst, k=5, ef=ef1, stages=3, ef1=ef1, ef2=ef2, ef3=ef3)
        assert np.array_equal(ids, r["ids"]), (ef1, ef2, ef3)
        assert np.array_equal(d.astype(np.float64), r["d"]), (ef1, ef2, ef3)
    ix.close()


def test_candidates_rejects_full_stages(s1):
    """pa_search_candidates returns stage-① lists only; asking it for stages ②③
    is PA_EINVAL (it used to launch k_refine without the device full graph)."""
    ix = pa.Index.from_instance(s1)
    ix.attach_host(s1["full_offsets"], s1["full_neighbors"], s1["rotated"])
    for st in (pa.PA_STAGES_FULL, pa.PA_STAGES_FULL_GPU):
        with pytest.raises(pa.PAError) as e:
            ix.search_candidates(s1["queries"][:4], ef=32, stages=st)
        assert e.value.status == pa.PA_EINVAL
    ids, _ = ix.search_candidates(s1["queries"][:4], ef=32)          # the index is still usable
    assert ids.shape == (4, 32) and (ids[:, 0] >= 0).all()
    ix.close()


def test_searches_on_two_streams_serialise(s1):
    """Two pa_search_device calls enqueued back to back on different streams
    share the index workspace: the second waits for the first on the device, so
    both results equal the one-stream results."""
    import torch
    cfg = s1["cfg"]
    ix = pa.Index.from_instance(s1)
    q = torch.from_numpy(s1["queries"]).cuda()
    m = q.shape[0]
    ref = []
    for ef in (32, 96):
        oi = torch.empty(m, cfg.k, dtype=torch.int32, device="cuda")
        od = torch.empty(m, cfg.k, dtype=torch.float32, device="cuda")
        ix.search_device(q, cfg.k, ef, oi, od)
        torch.cuda.synchronize()
        ref.append((oi.cpu(), od.cpu()))
    s_a, s_b = torch.cuda.Stream(), torch.cuda.Stream()
    outs = [(torch.empty(m, cfg.k, dtype=torch.int32, device="cuda"),
             torch.empty(m, cfg.k, dtype=torch.float32, device="cuda")) for _ in range(2)]
    for _ in range(3):
        ix.search_device(q, cfg.k, 32, *outs[0], stream=s_a.cuda_stream)
        ix.search_device(q, cfg.k, 96, *outs[1], stream=s_b.cuda_stream)
        torch.cuda.synchronize()
        for (oi, od), (ri, rd) in zip(outs, ref):
            assert torch.equal(oi.cpu(), ri) and torch.equal(od.cpu(), rd)
    ix.close()


# ------------------------------------------------- configurations untested in r1 --
def _full_checks(inst, ids, d, k, r_ids):
    Qh = orc.project(inst["queries"], inst["basis"])
    gt, _ = orc.brute_force(Qh, inst["rotated"], k, metric=inst["metric"])
    rg, ro = orc.recall(ids, gt, k), orc.recall(r_ids, gt, k)
    assert abs(rg - ro) <= 0.002 + 1e-12, (rg, ro)
    X = inst["rotated"].astype(np.float64)[ids]
    want = ((X - Qh[:, None, :]) ** 2).sum(2) if inst["metric"] == "l2" else -(X * Qh[:, None, :]).sum(2)
    scale = np.abs(want) if inst["metric"] == "l2" else np.abs(X * Qh[:, None, :]).sum(2)
    assert np.all(np.abs(d - want) <= 1e-5 * scale + 1e-6 * np.sqrt(np.abs(want) * (Qh ** 2).sum(1, keepdims=True)))
    return rg, ro


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_d768_parity(metric):
    """LAION/WIKI shape D = 768, d' = 128 (C3/C4): the tcgen05 projection with
    q_res (r + D = 800 columns, four column tiles) and tcgen05 FES, stage ① tie-aware
    against the oracle, stages ②③ (host and GPU) by recall and fp64 distances."""
    inst = tiny_instance(n=2500, D=768, dp=128, R=16, m=130, seed=768, member_ratio=0.5, r=8, metric=metric)
    for bloom in (0, 12):
        g, r = _both(inst, 10, 48, trace_cap=8192, bloom_log2=bloom)
        rep = compare(inst, g, r, 10, 48)
        assert not rep.fail, rep.fail[:3]
        assert rep.exact >= 0.9 * 130
    ix = pa.Index.from_instance(inst)
    ix.attach_host(inst["full_offsets"], inst["full_neighbors"], inst["rotated"])
    r3 = orc.search(inst, k=10, ef=48, stages=3)
    for stages in (pa.PA_STAGES_FULL, pa.PA_STAGES_FULL_GPU):
        ids, d = ix.search(inst["queries"], k=10, ef=48, stages=stages)
        print(metric, stages, _full_checks(inst, ids, d, 10, r3["ids"]))
    ix.close()


@pytest.mark.parametrize("bloom", [0, 12])
def test_ids_above_2pow24(bloom):
    """Member ids ≥ 2^24 (100M-scale id space): the exact kernels switch to the
    wide (32-bit) visited hash; parity with the oracle, tie-aware, plus stage ②③
    on the GPU."""
    from tiny import sparse_id_instance
    inst = sparse_id_instance()
    assert inst["fes_pool_ids"].max() >= (1 << 24)
    g, r = _both(inst, 10, 64, trace_cap=8192, bloom_log2=bloom)
    rep = compare(inst, g, r, 10, 64)
    assert not rep.fail, rep.fail[:3]
    assert rep.exact >= 0.9 * inst["queries"].shape[0]
    assert (g["ids"] >= (1 << 24)).any()


def test_degree_64_parity():
    """Subgraph degrees up to 64 (ELL width 64, the ABI's max_degree bound): exact
    visited set, tie-aware parity; the bloom filter rejects width 64 (PA_ENOTSUP)."""
    inst = tiny_instance(n=3000, D=32, dp=16, R=64, m=96, seed=64, member_ratio=0.6, r=8)
    assert np.diff(inst["sub_offsets"]).max() > 32
    g, r = _both(inst, 10, 64, trace_cap=16384)
    rep = compare(inst, g, r, 10, 64)
    assert not rep.fail, rep.fail[:3]
    assert rep.exact >= 0.9 * 96
    ix = pa.Index.from_instance(inst)
    with pytest.raises(pa.PAError) as e:
        run_gpu(ix, inst, 10, 64, bloom_log2=12)
    assert e.value.status == pa.PA_ENOTSUP
    ix.attach_host(inst["full_offsets"], inst["full_neighbors"], inst["rotated"])
    ids, d = ix.search(inst["queries"], k=10, ef=64, stages=pa.PA_STAGES_FULL_GPU)
    r3 = orc.search(inst, k=10, ef=64, stages=3)
    _full_checks(inst, ids, d, 10, r3["ids"])
    ix.close()


# ---------------------------------------------------- NEXT-f3: search width w > 1 --
@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("w", [2, 4])
def test_width_integer_fixture_bit_exact(metric, w):
    """Search width w (oracle O6 generalisation: the w best unchecked expanded per
    iteration, rows in key order) on exact-arithmetic fixtures: stage ① traces,
    lists and counters identical to the oracle's; stages ②③ (host and GPU) give
    identical ids and distances."""
    inst = integer_instance(seed=30 + w, metric=metric, n=400)
    for ef in (8, 32):
        g, r = _both(inst, 5, ef, width=w)
        ro = orc.search(inst, k=5, ef=ef, stages=1, trace_cap=4096, width=w)
        assert np.array_equal(g["ids"], ro["ids"]) and np.array_equal(g["d"].astype(np.float64), ro["d"])
        assert np.array_equal(g["cand_ids"], ro["cand1_ids"])
        for q in range(inst["queries"].shape[0]):
            ne = int(ro["trace_nexp"][q])
            assert list(g["trace_expand"][q][:ne]) == list(ro["trace_expand"][q][:ne]) and g["trace_nexp"][q] == ne
        assert np.array_equal(g["n_dist1"], ro["n_dist1"])
    ix = pa.Index.from_instance(inst)
    ix.attach_host(inst["full_offsets"], inst["full_neighbors"], inst["rotated"])
    for stages in (pa.PA_STAGES_FULL, pa.PA_STAGES_FULL_GPU):
        for ef in (8, 32):
            ids, d = ix.search(inst["queries"], k=5, ef=ef, stages=stages, width=w)
            r = orc.search(inst, k=5, ef=ef, stages=3, width=w)
            assert np.array_equal(ids, r["ids"]), (stages, ef)
            assert np.array_equal(d.astype(np.float64), r["d"]), (stages, ef)
    with pytest.raises(pa.PAError) as e:
        ix.search(inst["queries"], k=5, ef=32, width=w, bloom_log2=12)
    assert e.value.status == pa.PA_ENOTSUP
    ix.close()


@pytest.mark.parametrize("w", [2, 3])
def test_width_config_parity(w, s1):
    """w > 1 on float data: tie-aware stage-① parity with the oracle's width-w search."""
    cfg = s1["cfg"]
    ix = pa.Index.from_instance(s1)
    g = run_gpu(ix, s1, cfg.k, cfg.ef, trace_cap=8192, width=w)
    ix.close()
    r = orc.search(s1, k=cfg.k, ef=cfg.ef, stages=1, trace_cap=8192, width=w)
    rep = compare(s1, g, r, cfg.k, cfg.ef, width=w)
    assert not rep.fail, rep.fail[:3]
    assert rep.exact >= 0.9 * s1["queries"].shape[0]
