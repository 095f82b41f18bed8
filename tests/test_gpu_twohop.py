"""GPU parity of NEXT-f4's entry selection (pa_entries_device) against the oracle:
the two-hop baseline vs O14 and the FES entries vs O4, through the C ABI.

Integer instances (every fp32 operation exact) must match bit for bit including
ties; random instances match as sets up to near-ties (tests/parity.py tolerance)
at the E boundary or at the hop-1 beam boundary."""
import numpy as np
import pytest

import oracle as orc
import paper_2503_21206_b200 as pa
from parity import _tol
from test_gpu_parity import integer_instance
from tiny import tiny_instance

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build_library()


def _gpu_two_hop(inst, e0, beam, E):
    import torch
    ix = pa.Index.from_instance(inst)
    q = torch.from_numpy(inst["queries"]).cuda()
    m = q.shape[0]
    d = torch.empty(m, E, dtype=torch.float32, device="cuda")
    nd = torch.empty(m, dtype=torch.int32, device="cuda")
    ids = ix.entries_device(q, E, method=pa.PA_ENTRIES_TWO_HOP, e0=e0, beam=beam, out_d=d, n_dist=nd)
    torch.cuda.synchronize()
    out = ids.cpu().numpy(), d.cpu().numpy(), nd.cpu().numpy()
    ix.close()
    return out


def _members(inst):
    return np.flatnonzero(inst["member_flags"]) if "member_flags" in inst else np.arange(inst["sub_offsets"].size - 1)


@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("beam", [0, 1, 5, 32])
def test_two_hop_integer_bit_exact(metric, beam):
    inst = integer_instance(n=400, D=16, R=8, m=48, seed=41, metric=metric)
    e0 = int(_members(inst)[7])
    E = 40
    gi, gd, gn = _gpu_two_hop(inst, e0, beam, E)
    r = orc.two_hop(inst, e0=e0, beam=beam, E=E)
    assert np.array_equal(gi, r["ids"])
    ok = r["ids"] >= 0
    assert np.array_equal(gd[ok].astype(np.float64), r["d"][ok])
    assert np.all(np.isinf(gd[~ok]))
    assert np.array_equal(gn, r["n_dist"])


@pytest.mark.parametrize("metric", ["l2", "ip"])
@pytest.mark.parametrize("E,beam", [(16, 4), (64, 32), (200, 32), (256, 12)])
def test_two_hop_random_parity(metric, E, beam):
    inst = tiny_instance(n=3000, D=24, dp=12, R=32, m=64, seed=43, metric=metric, member_ratio=0.5)
    e0 = int(_members(inst)[11])
    gi, gd, gn = _gpu_two_hop(inst, e0, beam, E)
    r = orc.two_hop(inst, e0=e0, beam=beam, E=E)
    Qh = orc.project(inst["queries"], inst["basis"])[:, :12]
    X = inst["reduced"].astype(np.float64)

    def delta(q, ids):
        x = X[np.asarray(ids, np.int64)]
        return ((x - Qh[q]) ** 2).sum(1) if metric == "l2" else -(x @ Qh[q])

    def tol(q, ids, d):
        sc = None if metric == "l2" else np.abs(X[np.asarray(ids, np.int64)] * Qh[q]).sum(1)
        return _tol(d, float((Qh[q] ** 2).sum()), sc)

    exact = 0
    for q in range(inst["queries"].shape[0]):
        ok = gi[q] >= 0
        want = delta(q, gi[q][ok])
        assert np.all(np.abs(gd[q][ok] - want) <= tol(q, gi[q][ok], want)), q
        sg, so = set(gi[q][ok].tolist()), set(r["ids"][q][r["ids"][q] >= 0].tolist())
        if sg == so:
            exact += 1
            continue
        # a near-tie at the E boundary, or at the beam boundary among hop-1 keys
        diff = sorted(sg ^ so)
        bnd = r["d"][q][(r["ids"][q] >= 0)].max()
        dd = delta(q, diff)
        at_e = np.all(np.abs(dd - bnd) <= tol(q, diff, np.maximum(np.abs(dd), abs(bnd))))
        off, nb = inst["sub_offsets"], inst["sub_neighbors"]
        h1 = np.unique(nb[off[e0]:off[e0 + 1]])
        h1 = h1[h1 != e0]
        k1 = delta(q, h1)
        o = np.lexsort((h1, k1))
        at_beam = 0 < beam < len(h1) and abs(k1[o[beam - 1]] - k1[o[beam]]) <= tol(q, [h1[o[beam]]], np.array([abs(k1[o[beam]])]))[0]
        assert at_e or at_beam, (q, diff[:6])
    assert exact >= 0.9 * inst["queries"].shape[0]


def test_fes_entries_match_search_entries():
    """PA_ENTRIES_FES returns exactly the entries stage ① is seeded with (pa_search_device's debug output)."""
    import torch
    inst = tiny_instance(n=3000, D=24, dp=12, R=16, m=80, seed=44, member_ratio=0.5, r=8)
    ix = pa.Index.from_instance(inst)
    q = torch.from_numpy(inst["queries"]).cuda()
    m, E = q.shape[0], 48
    got = ix.entries_device(q, E, method=pa.PA_ENTRIES_FES)
    ent = torch.empty(m, E, dtype=torch.int32, device="cuda")
    dbg = pa.Debug(entries=ent.data_ptr())
    oi = torch.empty(m, 10, dtype=torch.int32, device="cuda")
    od = torch.empty(m, 10, dtype=torch.float32, device="cuda")
    ix.search_device(q, 10, E, oi, od, debug=dbg, entries=E)
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy(), ent.cpu().numpy())
    r = orc.search(inst, k=10, ef=E, stages=1, entries=E)
    same = np.mean([set(a[a >= 0]) == set(b[b >= 0]) for a, b in zip(got.cpu().numpy(), r["entries"])])
    assert same >= 0.95
    ix.close()


def test_entries_rejects_bad_arguments():
    import torch
    inst = tiny_instance(n=300, D=16, dp=8, R=8, m=4, seed=45)
    ix = pa.Index.from_instance(inst)
    q = torch.from_numpy(inst["queries"]).cuda()
    for kw, code in ((dict(E=0), pa.PA_EINVAL), (dict(E=257), pa.PA_EINVAL),
                     (dict(E=8, method=pa.PA_ENTRIES_TWO_HOP, e0=-1), pa.PA_EINVAL),
                     (dict(E=8, method=pa.PA_ENTRIES_TWO_HOP, e0=300), pa.PA_EINVAL),
                     (dict(E=8, method=pa.PA_ENTRIES_TWO_HOP, beam=-1), pa.PA_EINVAL),
                     (dict(E=8, method=7), pa.PA_EINVAL)):
        E = kw.pop("E")
        with pytest.raises(pa.PAError) as ei:
            ix.entries_device(q, E, out=torch.empty(4, E, dtype=torch.int32, device="cuda"), **kw)
        assert ei.value.status == code
    ix.close()
