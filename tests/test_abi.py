"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/pilotann.h declares, and pa_build rejects invalid inputs with
the specific error codes of SURVEY §8.b before touching any device."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2503_21206_b200 as pa
from tiny import tiny_instance

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "pilotann.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pa_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    import __graft_entry__ as g
    g.build_library()
    return pa.lib()


def test_exports_every_header_symbol(L):
    syms = header_symbols()
    assert set(syms) == set(pa.EXPORTS)
    for s in syms:
        assert hasattr(L, s), s


def test_version_and_null_safety(L):
    assert "sm_100a" in pa.version()
    L.pa_destroy(None)                                         # NULL-safe
    st = pa.Stats()
    assert L.pa_get_stats(None, C.byref(st), C.sizeof(st)) == pa.PA_ESTATE
    assert L.pa_search(None, None, 0, 10, 64, None, None, None) == pa.PA_ESTATE
    assert L.pa_search_device(C.c_void_p(12345), None, 0, 10, 64, None, None, None, None, None) == pa.PA_ESTATE


def _build(inst, **over):
    kw = dict(sub_offsets=inst["sub_offsets"], sub_neighbors=inst["sub_neighbors"], reduced=inst["reduced"],
              basis=inst["basis"], fes_centroids=inst["fes_centroids"], fes_cell_off=inst["fes_cell_off"],
              fes_pool_ids=inst["fes_pool_ids"], member_flags=inst["member_flags"], metric=inst["metric"],
              device=0)
    kw.update(over)
    return pa.Index(**kw)


def _expect(status, inst, **over):
    with pytest.raises(pa.PAError) as e:
        _build(inst, **over)
    assert e.value.status == status, str(e.value)
    return str(e.value)


@pytest.fixture(scope="module")
def inst():
    return tiny_instance(n=64, D=8, dp=4, R=6, m=4, seed=3, member_ratio=0.75)


def test_build_rejects_bad_graphs(L, inst):
    off, nb = inst["sub_offsets"].copy(), inst["sub_neighbors"].copy()
    bad = off.copy(); bad[0] = 1
    _expect(pa.PA_EGRAPH, inst, sub_offsets=bad)                                 # offsets[0] != 0
    u = int(np.flatnonzero(np.diff(off) > 1)[0])
    nb2 = nb.copy(); nb2[off[u]] = 1000
    _expect(pa.PA_EGRAPH, inst, sub_neighbors=nb2)                               # id out of range
    nb2 = nb.copy(); nb2[off[u]] = u
    _expect(pa.PA_EGRAPH, inst, sub_neighbors=nb2)                               # self-loop
    nb2 = nb.copy(); nb2[off[u] + 1] = nb2[off[u]]
    _expect(pa.PA_EGRAPH, inst, sub_neighbors=nb2)                               # duplicate
    _expect(pa.PA_EGRAPH, inst, max_degree=1)                                    # degree > max_degree
    nonmem = int(np.flatnonzero(inst["member_flags"] == 0)[0])
    nb2 = nb.copy(); nb2[off[u]] = nonmem
    if nonmem not in nb[off[u]:off[u + 1]]:
        _expect(pa.PA_EGRAPH, inst, sub_neighbors=nb2)                           # edge into non-member


def test_build_rejects_bad_basis_and_values(L, inst):
    V = inst["basis"].copy(); V[0, 0] += 1e-2
    _expect(pa.PA_EBASIS, inst, basis=V)
    V = inst["basis"].copy(); V[1, 1] = np.nan
    _expect(pa.PA_EINVAL, inst, basis=V)
    R = inst["reduced"].copy(); R[int(np.flatnonzero(inst["member_flags"])[0]), 0] = np.inf
    _expect(pa.PA_EINVAL, inst, reduced=R)
    _expect(pa.PA_EINVAL, inst, max_degree=65)


def test_build_rejects_bad_fes(L, inst):
    co = inst["fes_cell_off"].copy(); co[2] = co[1]
    _expect(pa.PA_EFES, inst, fes_cell_off=co)                                   # empty cell
    pool = inst["fes_pool_ids"].copy(); pool[1] = pool[0]
    _expect(pa.PA_EFES, inst, fes_pool_ids=pool)                                 # duplicate
    nonmem = int(np.flatnonzero(inst["member_flags"] == 0)[0])
    pool = inst["fes_pool_ids"].copy(); pool[0] = nonmem
    _expect(pa.PA_EFES, inst, fes_pool_ids=pool)                                 # not a member


def test_validation_then_device(L, inst):
    """A valid build passes validation; without a GPU it must fail at the device step (PA_ECUDA/PA_EINVAL
    for 'no device'), never silently fall back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by -m gpu tests")
    with pytest.raises(pa.PAError) as e:
        _build(inst)
    assert e.value.status in (pa.PA_ECUDA, pa.PA_EINVAL)


def test_binding_structs_match_the_header(tmp_path):
    """The ctypes mirrors in the binding have the header's sizes and field
    offsets (a C program compiled against include/pilotann.h prints them)."""
    import subprocess
    structs = {"pa_build_params": pa.BuildParams, "pa_search_opts": pa.SearchOpts, "pa_debug": pa.Debug,
               "pa_stats": pa.Stats, "pa_replica_meta": pa.ReplicaMeta, "pa_buffer": pa.Buffer}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "pilotann.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "abi"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = subprocess.check_output([str(exe)], text=True).split("\n")
    want = {}
    for ln in out:
        if ln:
            a, b, c = ln.split()
            want[(a, b)] = int(c)
    for cname, py in structs.items():
        assert C.sizeof(py) == want[(cname, "size")], cname
        for f, _ in py._fields_:
            assert getattr(py, f).offset == want[(cname, f)], (cname, f)


def test_replica_meta_rejected_before_device(L):
    """pa_build_replica validates the layout before touching a device."""
    m = pa.ReplicaMeta(n=100, pool_n=8, dim=16, rdim=8, rdim_pad=8, rdim_h=8, qlen=8, rstride=32, rstride_h=64,
                       ell_w=48, metric=0, fes_r=4, max_cell=4, proj_nb=32, pool_chunks=4)
    h = C.c_void_p()
    assert L.pa_build_replica(C.byref(m), 0, C.byref(h)) == pa.PA_EINVAL          # ell_w must be 32 or 64
    assert "inconsistent" in L.pa_last_error().decode()
    cnt = C.c_int32()
    assert L.pa_replica_buffers(None, None, 0, C.byref(cnt)) == pa.PA_ESTATE
