"""The 100M-scale instance path (datagen/large.py: X̂-strided reduced rows,
batched graph tool) through the product, against the oracle."""
import numpy as np
import pytest

import oracle as orc
import paper_2503_21206_b200 as pa
from gpu_util import run_gpu
from parity import compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def small_large():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build_library()
    import datagen as dg
    from datagen import large as lg
    cfg = dg.get_config("S2", N=60_000, m=200)
    return lg.build_instance_large(cfg, device="cuda")


@pytest.mark.parametrize("strided", [True, False])
@pytest.mark.parametrize("bloom", [0, 12])
def test_strided_reduced_parity(small_large, strided, bloom):
    """reduced = X̂[:, :d'] passed with row stride D (no host copy) gives the same
    results as a contiguous copy, and both match the oracle (tie-aware)."""
    inst = small_large if strided else dict(small_large, reduced=np.ascontiguousarray(small_large["reduced"]))
    assert (inst["reduced"].strides[0] == 4 * inst["D"]) == strided
    cfg = inst["cfg"]
    ix = pa.Index.from_instance(inst)
    g = run_gpu(ix, inst, cfg.k, 64, trace_cap=8192, bloom_log2=bloom)
    ix.close()
    r = orc.search(inst, k=cfg.k, ef=64, stages=1, trace_cap=8192, bloom_log2=bloom or None)
    rep = compare(inst, g, r, cfg.k, 64, gt_ids=inst["gt_sub_ids"][:, :cfg.k])
    print(strided, bloom, rep, rep.recall_gpu, rep.recall_orc)
    assert not rep.fail, rep.fail[:3]
    assert rep.exact >= 0.9 * inst["queries"].shape[0]
