"""ctypes wrapper of the PilotANN ORACLE (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference arms.  The product package
(paper_2503_21206_b200) never imports this module and this module never
imports the product.  The ctypes structs below mirror oracle.cpp by hand.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
SRC = os.path.join(_HERE, "oracle.cpp")

NO_FES, NO_STAGE2, NO_STAGE1 = 1, 2, 4
COUNTERS = ("n_exp1", "n_dist1", "n_exp2", "n_dist2", "n_exp3", "n_dist3", "fes_work", "_pad")


def build(force: bool = False) -> str:
    """Compile the oracle (plain C++17, -O2, no fast-math, no intrinsics)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread", "-fno-fast-math",
               "-ffp-contract=off", SRC, "-o", LIB_PATH]
        subprocess.check_call(cmd)
    return LIB_PATH


class OrcIndex(C.Structure):
    _fields_ = [("n", C.c_int64), ("dim", C.c_int32), ("rdim", C.c_int32), ("metric", C.c_int32),
                ("sub_offsets", C.c_void_p), ("sub_neighbors", C.c_void_p), ("reduced", C.c_void_p),
                ("basis", C.c_void_p), ("fes_r", C.c_int32), ("fes_centroids", C.c_void_p),
                ("fes_cell_off", C.c_void_p), ("fes_pool_ids", C.c_void_p),
                ("full_offsets", C.c_void_p), ("full_neighbors", C.c_void_p), ("rotated", C.c_void_p),
                ("reduced_stride", C.c_int64)]


class OrcOpts(C.Structure):
    _fields_ = [("k", C.c_int32), ("ef1", C.c_int32), ("ef2", C.c_int32), ("ef3", C.c_int32),
                ("entries", C.c_int32), ("width", C.c_int32), ("refine_iters", C.c_int32),
                ("stages", C.c_int32), ("flags", C.c_uint32), ("threads", C.c_int32),
                ("trace_cap", C.c_int32), ("bloom_log2", C.c_int32), ("use_bloom", C.c_int32)]


class OrcOut(C.Structure):
    _fields_ = [("out_ids", C.c_void_p), ("out_d", C.c_void_p), ("cell", C.c_void_p),
                ("entries", C.c_void_p), ("entries_d", C.c_void_p),
                ("cand1_ids", C.c_void_p), ("cand1_d", C.c_void_p), ("counters", C.c_void_p),
                ("trace_expand", C.c_void_p), ("trace_visit", C.c_void_p),
                ("trace_nexp", C.c_void_p), ("trace_nvis", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.orc_search.restype = C.c_int
        _lib.orc_search.argtypes = [C.POINTER(OrcIndex), C.c_void_p, C.c_int64, C.POINTER(OrcOpts),
                                    C.POINTER(OrcOut)]
        _lib.orc_project.restype = None
        _lib.orc_project.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]
        _lib.orc_brute_force.restype = None
        _lib.orc_brute_force.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64,
                                         C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_int32,
                                         C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]
        _lib.orc_two_hop.restype = None
        _lib.orc_two_hop.argtypes = [C.POINTER(OrcIndex), C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                     C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_recall.restype = C.c_double
        _lib.orc_recall.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int64, C.c_int32,
                                    C.c_void_p, C.c_void_p]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


def default_budgets(k: int, ef: int):
    """Q21 / S:L469: ef1 = ef3 = ef, ef2 = max(k, ef/2); E = ef1; w = 1; 2 refine iterations."""
    return dict(ef1=ef, ef2=max(k, ef // 2), ef3=ef, entries=ef, width=1, refine_iters=2)


def _rows(a):
    """fp32 rows, possibly a column slice of a wider array (X̂[:, :d']) → (array, row stride)."""
    a = np.asarray(a)
    if a.ndim == 2 and a.dtype == np.float32 and a.strides[1] == 4 and a.strides[0] % 4 == 0:
        return a, a.strides[0] // 4
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.shape[1]


def make_index(inst: dict):
    """Keep contiguous copies alive inside the returned tuple (index struct, arrays)."""
    red, rstride = _rows(inst["reduced"])
    arrs = dict(
        sub_offsets=_c(inst["sub_offsets"], np.int64), sub_neighbors=_c(inst["sub_neighbors"], np.int32),
        reduced=red, basis=_c(inst["basis"], np.float32),
        fes_centroids=_c(inst["fes_centroids"], np.float32), fes_cell_off=_c(inst["fes_cell_off"], np.int64),
        fes_pool_ids=_c(inst["fes_pool_ids"], np.int32),
        full_offsets=_c(inst.get("full_offsets"), np.int64), full_neighbors=_c(inst.get("full_neighbors"), np.int32),
        rotated=_c(inst.get("rotated"), np.float32))
    N = arrs["sub_offsets"].shape[0] - 1
    ix = OrcIndex(n=N, dim=int(arrs["basis"].shape[0]), rdim=int(arrs["reduced"].shape[1]),
                  metric=1 if inst.get("metric", "l2") == "ip" else 0,
                  sub_offsets=_p(arrs["sub_offsets"]), sub_neighbors=_p(arrs["sub_neighbors"]),
                  reduced=_p(arrs["reduced"]), basis=_p(arrs["basis"]),
                  fes_r=int(arrs["fes_cell_off"].shape[0] - 1), fes_centroids=_p(arrs["fes_centroids"]),
                  fes_cell_off=_p(arrs["fes_cell_off"]), fes_pool_ids=_p(arrs["fes_pool_ids"]),
                  full_offsets=_p(arrs["full_offsets"]), full_neighbors=_p(arrs["full_neighbors"]),
                  rotated=_p(arrs["rotated"]), reduced_stride=rstride)
    return ix, arrs


def search(inst: dict, queries=None, k: int = 10, ef: int = 64, stages: int = 1, flags: int = 0,
           threads: int = 0, trace_cap: int = 0, bloom_log2=None, **budgets) -> dict:
    """Run O1-O9 over `queries` (default inst['queries']).  Returns numpy arrays.
    bloom_log2 = s selects the O13 bloom-filter visited set in stage ① (3 × 2^s bits)."""
    ix, keep = make_index(inst)
    Q = _c(inst["queries"] if queries is None else queries, np.float32)
    m = Q.shape[0]
    b = default_budgets(k, ef)
    b.update(budgets)
    o = OrcOpts(k=k, stages=stages, flags=flags, threads=threads, trace_cap=trace_cap,
                bloom_log2=0 if bloom_log2 is None else int(bloom_log2), use_bloom=0 if bloom_log2 is None else 1, **b)
    E, ef1 = b["entries"], b["ef1"]
    res = dict(ids=np.full((m, k), -1, np.int32), d=np.zeros((m, k)), cell=np.zeros(m, np.int32),
               entries=np.zeros((m, E), np.int32), entries_d=np.zeros((m, E)),
               cand1_ids=np.zeros((m, ef1), np.int32), cand1_d=np.zeros((m, ef1)),
               counters=np.zeros((m, 8), np.int64))
    if trace_cap:
        res.update(trace_expand=np.full((m, trace_cap), -1, np.int32),
                   trace_visit=np.full((m, trace_cap), -1, np.int32),
                   trace_nexp=np.zeros(m, np.int32), trace_nvis=np.zeros(m, np.int32))
    out = OrcOut(out_ids=_p(res["ids"]), out_d=_p(res["d"]), cell=_p(res["cell"]),
                 entries=_p(res["entries"]), entries_d=_p(res["entries_d"]),
                 cand1_ids=_p(res["cand1_ids"]), cand1_d=_p(res["cand1_d"]), counters=_p(res["counters"]),
                 trace_expand=_p(res.get("trace_expand")), trace_visit=_p(res.get("trace_visit")),
                 trace_nexp=_p(res.get("trace_nexp")), trace_nvis=_p(res.get("trace_nvis")))
    rc = lib().orc_search(C.byref(ix), _p(Q), m, C.byref(o), C.byref(out))
    if rc != 0:
        raise RuntimeError(f"orc_search failed: {rc}")
    del keep
    for i, name in enumerate(COUNTERS[:7]):
        res[name] = res["counters"][:, i]
    return res


def two_hop(inst: dict, e0: int, beam: int, E: int, queries=None, threads: int = 0) -> dict:
    """O14: two-hop entry selection from the fixed entry e0 (the FES baseline of
    P:L986-989).  → ids [m][E] int32, d [m][E] fp64 (ascending keys), n_dist [m]."""
    ix, keep = make_index(inst)
    Q = _c(inst["queries"] if queries is None else queries, np.float32)
    m = Q.shape[0]
    res = dict(ids=np.zeros((m, E), np.int32), d=np.zeros((m, E)), n_dist=np.zeros(m, np.int64))
    lib().orc_two_hop(C.byref(ix), _p(Q), m, int(e0), int(beam), int(E), threads, _p(res["ids"]), _p(res["d"]),
                      _p(res["n_dist"]))
    del keep
    return res


def project(Q: np.ndarray, V: np.ndarray) -> np.ndarray:
    Q = _c(Q, np.float32)
    V = _c(V, np.float32)
    out = np.zeros((Q.shape[0], V.shape[1]), np.float64)
    lib().orc_project(_p(Q), Q.shape[0], V.shape[0], _p(V), _p(out))
    return out


def brute_force(Qh: np.ndarray, X: np.ndarray, k: int, metric: str = "l2", ids=None, dim=None,
                threads: int = 0):
    """Exact top-k by (δ, id).  Qh fp64 [m][≥dim], X fp32 [n][≥dim]."""
    Qh = _c(Qh, np.float64)
    X = _c(X, np.float32)
    d = dim or X.shape[1]
    m = Qh.shape[0]
    ids_c = _c(ids, np.int32)
    oi = np.zeros((m, k), np.int32)
    od = np.zeros((m, k), np.float64)
    lib().orc_brute_force(_p(Qh), m, Qh.shape[1], _p(X), X.shape[0], X.shape[1], d, _p(ids_c),
                          0 if ids_c is None else ids_c.shape[0], k, 1 if metric == "ip" else 0,
                          threads, _p(oi), _p(od))
    return oi, od


def recall(ret, gt, k: int, ret_d=None, gt_d=None) -> float:
    ret = _c(ret, np.int32)
    gt = _c(gt, np.int32)
    rd = _c(ret_d, np.float64)
    gd = _c(gt_d, np.float64)
    return lib().orc_recall(_p(ret), ret.shape[1], _p(gt), gt.shape[1], ret.shape[0], k, _p(rd), _p(gd))
