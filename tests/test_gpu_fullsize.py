"""Parity at BASELINE.json's full size (configs[1], C1: 10M × 96, d' = 48, 10K
queries) in the launch configuration bench.py times (one pa_search_device call
over the whole 10K batch): every output of a sample of queries is checked one by
one against the oracle with the tie-aware protocol, and properties that hold at
any size are checked on all 10K (ids are members, rows sorted, no duplicates,
distances = fp64 δ' of the returned ids)."""
import numpy as np
import pytest

import oracle as orc
import paper_2503_21206_b200 as pa
from gpu_util import run_gpu
from parity import compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build_library()
    import datagen as dg
    cfg = dg.get_config("C1")
    return dg.build_instance(cfg, device="cuda", gt=False)


@pytest.mark.parametrize("ef,bloom", [(32, 0), (128, 0), (80, 12)])
def test_c1_full_size_sampled_parity(c1, ef, bloom):
    """(80, 12) is bench.py's headline launch: ef 80 with the paper's bloom
    visited set of 3 × 2^12 bits, checked against the oracle's O13 mode; the
    timed (compile-time row length) kernel must reproduce the traced one."""
    cfg = c1["cfg"]
    ix = pa.Index.from_instance(c1)
    g = run_gpu(ix, c1, cfg.k, ef, trace_cap=6144, bloom_log2=bloom)
    timed = run_gpu(ix, c1, cfg.k, ef, bloom_log2=bloom)
    ix.close()
    for key in ("ids", "d", "cand_ids", "cand_dists", "counters"):
        assert np.array_equal(g[key], timed[key]), key
    m = c1["queries"].shape[0]
    assert m == 10_000 and np.all(g["status"] == 0)
    # properties on all queries
    ids, d = g["ids"], g["d"]
    assert np.all(ids >= 0)
    assert np.all(c1["member_flags"][ids] == 1)
    assert np.all(np.diff(d, axis=1) >= 0)
    assert all(len(set(r)) == len(r) for r in ids)
    # sampled queries: oracle one by one (tie-aware lockstep protocol)
    sample = np.arange(0, m, 50)
    sub = dict(c1, queries=c1["queries"][sample])
    gs = {k: v[sample] for k, v in g.items()}
    r = orc.search(sub, k=cfg.k, ef=ef, stages=1, trace_cap=6144, bloom_log2=bloom or None)
    rep = compare(sub, gs, r, cfg.k, ef)
    print(f"C1 ef={ef} bloom={bloom}", rep)
    assert not rep.fail, rep.fail[:5]
    assert rep.exact >= 0.8 * sample.size
    # distances of every returned id on all queries vs fp64 (vectorised property check)
    Qh = orc.project(c1["queries"], c1["basis"])[:, :cfg.dp]
    X = c1["reduced"][ids].astype(np.float64)
    want = ((X - Qh[:, None, :]) ** 2).sum(2)
    tol = 1e-5 * want + 1e-6 * np.sqrt(want * (Qh ** 2).sum(1, keepdims=True))
    assert np.all(np.abs(d - want) <= tol)


@pytest.fixture(scope="module")
def ip1m():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build_library()
    import datagen as dg
    from datagen import large as lg
    cfg = dg.get_config("C2S", N=1_000_000, m=1000)
    return lg.build_instance_large(cfg, device="cuda", gt_k=10)


@pytest.mark.parametrize("bloom", [0, 12])
def test_ip_1m_sampled_parity(ip1m, bloom):
    """Inner product (T2I shape, OOD queries) at 1M rows through the 100M-scale
    instance path (strided X̂ rows): sampled tie-aware parity with the oracle and
    Recall@10 (GT_sub) within 0.002 of the oracle's on the sample."""
    inst = ip1m
    cfg = inst["cfg"]
    ix = pa.Index.from_instance(inst)
    g = run_gpu(ix, inst, cfg.k, 64, trace_cap=8192, bloom_log2=bloom)
    ix.close()
    sample = np.arange(0, inst["queries"].shape[0], 5)
    sub = dict(inst, queries=inst["queries"][sample])
    gs = {k: v[sample] for k, v in g.items()}
    r = orc.search(sub, k=cfg.k, ef=64, stages=1, trace_cap=8192, bloom_log2=bloom or None)
    rep = compare(sub, gs, r, cfg.k, 64, gt_ids=inst["gt_sub_ids"][sample, :cfg.k])
    print("IP 1M", bloom, rep, rep.recall_gpu, rep.recall_orc)
    assert not rep.fail, rep.fail[:5]
    assert rep.exact >= 0.8 * sample.size
