"""Python binding of the B200-native PilotANN GPU stage (arXiv 2503.21206).

Argument marshalling only: every step of the search runs in the CUDA kernels /
C++ runtime of libpilotann.so behind include/pilotann.h.  There is no Python
or CPU fallback for the GPU stage: if the shared library is missing, importing
works (so the package can be inspected / built) but constructing an Index
raises immediately.

    import paper_2503_21206_b200 as pa
    ix = pa.Index(n=..., dim=..., rdim=..., sub_offsets=..., ...)   # pa_build
    ix.attach_host(full_offsets, full_neighbors, rotated)             # pa_attach_host (stages 2-3)
    ids, d = ix.search(queries, k=10, ef=64)                          # pa_search (host buffers)
    ix.search_device(q_dev, k, ef, out_ids_dev, out_d_dev)            # pa_search_device (torch tensors)
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpilotann.so")

PA_OK, PA_EINVAL, PA_EGRAPH, PA_EBASIS, PA_EFES, PA_ENOMEM, PA_ECUDA, PA_ESTATE, PA_ENOTSUP = 0, -1, -2, -3, -4, -5, -6, -7, -8
STATUS_NAMES = {0: "PA_OK", -1: "PA_EINVAL", -2: "PA_EGRAPH", -3: "PA_EBASIS", -4: "PA_EFES",
                -5: "PA_ENOMEM", -6: "PA_ECUDA", -7: "PA_ESTATE", -8: "PA_ENOTSUP"}
PA_L2, PA_IP = 0, 1
PA_STAGES_GPU, PA_STAGES_FULL, PA_STAGES_FULL_GPU = 1, 3, 7
PA_NO_FES, PA_NO_STAGE2, PA_NO_STAGE1, PA_NO_PIPELINE = 1, 2, 4, 8
PA_CHECK_SIMT, PA_CHECK_WIDE_VISITED = 1, 2
PA_ENTRIES_FES, PA_ENTRIES_TWO_HOP = 0, 1

# Symbols declared in include/pilotann.h (checked by tests/test_abi.py).
EXPORTS = ("pa_build", "pa_attach_host", "pa_search", "pa_search_device", "pa_search_candidates",
           "pa_get_stats", "pa_destroy", "pa_last_error", "pa_version",
           "pa_replica_meta_of", "pa_build_replica", "pa_replica_buffers", "pa_entries_device")


class PAError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class BuildParams(C.Structure):
    _fields_ = [("n", C.c_int64), ("dim", C.c_int32), ("rdim", C.c_int32), ("max_degree", C.c_int32),
                ("metric", C.c_int32), ("sub_offsets", C.c_void_p), ("sub_neighbors", C.c_void_p),
                ("member_flags", C.c_void_p), ("reduced", C.c_void_p), ("basis", C.c_void_p),
                ("fes_r", C.c_int32), ("fes_centroids", C.c_void_p), ("fes_cell_off", C.c_void_p),
                ("fes_pool_ids", C.c_void_p), ("device", C.c_int32), ("reduced_fp16", C.c_int32),
                ("reduced_stride", C.c_int64)]


class SearchOpts(C.Structure):
    _fields_ = [("stages", C.c_int32), ("ef1", C.c_int32), ("ef2", C.c_int32), ("ef3", C.c_int32),
                ("entries", C.c_int32), ("width", C.c_int32), ("refine_iters", C.c_int32),
                ("flags", C.c_uint32), ("hash_slots_log2", C.c_int32), ("host_threads", C.c_int32),
                ("bloom_log2", C.c_int32), ("check_path", C.c_uint32)]


class ReplicaMeta(C.Structure):
    _fields_ = [("n", C.c_int64), ("pool_n", C.c_int64)] + [(f, C.c_int32) for f in (
        "dim", "rdim", "rdim_pad", "rdim_h", "qlen", "rstride", "rstride_h", "ell_w", "metric", "fes_r",
        "max_cell", "proj_nb", "pool_chunks", "fes_fold_norm", "reduced_fp16", "has_full", "full_w", "xstride")]

    def to_list(self):
        return [getattr(self, f) for f, _ in self._fields_]

    @classmethod
    def from_list(cls, vals):
        return cls(**{f: int(v) for (f, _), v in zip(cls._fields_, vals)})


class Buffer(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("bytes", C.c_int64)]


class Debug(C.Structure):
    _fields_ = [("cell", C.c_void_p), ("entries", C.c_void_p), ("cand_ids", C.c_void_p),
                ("cand_dists", C.c_void_p), ("counters", C.c_void_p), ("trace_cap", C.c_int32),
                ("trace_expand", C.c_void_p), ("trace_visit", C.c_void_p), ("trace_nexp", C.c_void_p),
                ("trace_nvis", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [("queries", C.c_int64), ("kernel_launches", C.c_int64),
                ("ms_project", C.c_double), ("ms_fes", C.c_double), ("ms_traverse", C.c_double),
                ("ms_total_gpu", C.c_double), ("ms_h2d", C.c_double), ("ms_d2h", C.c_double),
                ("ms_host_stages", C.c_double), ("ms_wall", C.c_double),
                ("sum_n_exp", C.c_int64), ("sum_n_dist", C.c_int64), ("sum_spill", C.c_int64),
                ("overflow_queries", C.c_int64), ("sum_n_dist2", C.c_int64), ("sum_n_dist3", C.c_int64),
                ("ms_refine", C.c_double)]

    def asdict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def lib():
    """Load libpilotann.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback for the GPU stage)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.pa_build.restype = C.c_int
        L.pa_build.argtypes = [C.POINTER(BuildParams), C.POINTER(vp)]
        L.pa_attach_host.restype = C.c_int
        L.pa_attach_host.argtypes = [vp, vp, vp, vp]
        L.pa_search.restype = C.c_int
        L.pa_search.argtypes = [vp, vp, i64, i32, i32, C.POINTER(SearchOpts), vp, vp]
        L.pa_search_device.restype = C.c_int
        L.pa_search_device.argtypes = [vp, vp, i64, i32, i32, C.POINTER(SearchOpts), vp, vp, C.POINTER(Debug), vp]
        L.pa_search_candidates.restype = C.c_int
        L.pa_search_candidates.argtypes = [vp, vp, i64, i32, C.POINTER(SearchOpts), vp, vp]
        L.pa_entries_device.restype = C.c_int
        L.pa_entries_device.argtypes = [vp, vp, i64, i32, i32, i32, i32, vp, vp, vp, vp]
        L.pa_get_stats.restype = C.c_int
        L.pa_get_stats.argtypes = [vp, C.POINTER(Stats), C.c_size_t]
        L.pa_destroy.restype = None
        L.pa_destroy.argtypes = [vp]
        L.pa_replica_meta_of.restype = C.c_int
        L.pa_replica_meta_of.argtypes = [vp, C.POINTER(ReplicaMeta)]
        L.pa_build_replica.restype = C.c_int
        L.pa_build_replica.argtypes = [C.POINTER(ReplicaMeta), i32, C.POINTER(vp)]
        L.pa_replica_buffers.restype = C.c_int
        L.pa_replica_buffers.argtypes = [vp, C.POINTER(Buffer), i32, C.POINTER(i32)]
        L.pa_last_error.restype = C.c_char_p
        L.pa_version.restype = C.c_char_p
        _lib = L
    return _lib


def version() -> str:
    return lib().pa_version().decode()


def _check(rc):
    if rc != PA_OK:
        raise PAError(rc, lib().pa_last_error().decode())


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


def _ptr(a):
    return None if a is None else a.ctypes.data


def _rows(a):
    """fp32 row-major rows, possibly a column slice of a wider array (e.g. the
    first d' columns of X̂): → (array whose .ctypes.data is row 0, row stride in floats)."""
    a = np.asarray(a)
    if a.ndim == 2 and a.dtype == np.float32 and a.strides[1] == 4 and a.strides[0] % 4 == 0 \
            and a.strides[0] >= 4 * a.shape[1]:
        return a, a.strides[0] // 4
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.shape[1] if a.ndim == 2 else 0


def _host_rows(x, cols, dtype, name):
    """A host [m][cols] array of `dtype` from numpy or a CPU torch tensor → (pointer, m, keep-alive)."""
    if hasattr(x, "data_ptr"):
        if x.device.type != "cpu":
            raise ValueError(f"{name}: expected a CPU tensor (got {x.device}); use search_device for device buffers")
        want = {np.float32: "torch.float32", np.int32: "torch.int32"}[dtype]
        if str(x.dtype) != want or not x.is_contiguous() or x.dim() != 2 or (cols and x.shape[1] != cols):
            raise ValueError(f"{name}: expected a contiguous {want} tensor [m][{cols}], got {tuple(x.shape)} {x.dtype}")
        return x.data_ptr(), int(x.shape[0]), x
    a = np.asarray(x)
    if a.ndim != 2 or (cols and a.shape[1] != cols):
        raise ValueError(f"{name}: expected [m][{cols}], got {a.shape}")
    a = np.ascontiguousarray(a, dtype=dtype)
    return _ptr(a), a.shape[0], a


def _dev_rows(x, rows, cols, dtype, device, name):
    want = {np.float32: "torch.float32", np.int32: "torch.int32"}[dtype]
    if x.device.type != "cuda" or x.device.index != device:
        raise ValueError(f"{name}: expected a tensor on cuda:{device}, got {x.device}")
    if str(x.dtype) != want or not x.is_contiguous() or x.dim() != 2 or x.shape[1] != cols \
            or (rows is not None and x.shape[0] != rows):
        raise ValueError(f"{name}: expected a contiguous {want} tensor [{rows}][{cols}], got {tuple(x.shape)} {x.dtype}")


def make_opts(stages=PA_STAGES_GPU, ef1=0, ef2=0, ef3=0, entries=0, width=0, refine_iters=0, flags=0,
              hash_slots_log2=0, host_threads=0, bloom_log2=0, check_path=0) -> SearchOpts:
    return SearchOpts(stages=stages, ef1=ef1, ef2=ef2, ef3=ef3, entries=entries, width=width,
                      refine_iters=refine_iters, flags=flags, hash_slots_log2=hash_slots_log2,
                      host_threads=host_threads, bloom_log2=bloom_log2, check_path=check_path)


class Index:
    """One device replica (pa_build).  Arrays are host numpy arrays (copied)."""

    def __init__(self, *, sub_offsets, sub_neighbors, reduced, basis, fes_centroids, fes_cell_off,
                 fes_pool_ids, member_flags=None, metric="l2", max_degree=None, device=0, n=None,
                 reduced_fp16=False):
        so = _c(sub_offsets, np.int64)
        sn = _c(sub_neighbors, np.int32)
        red, rstride = _rows(reduced)
        bas = _c(basis, np.float32)
        cen = _c(fes_centroids, np.float32)
        coff = _c(fes_cell_off, np.int64)
        pool = _c(fes_pool_ids, np.int32)
        mf = _c(member_flags, np.uint8)
        n = int(so.shape[0] - 1) if n is None else int(n)
        if max_degree is None:
            max_degree = int(np.diff(so).max()) if so.shape[0] > 1 else 1
            max_degree = max(1, max_degree)
        p = BuildParams(n=n, dim=int(bas.shape[0]), rdim=int(red.shape[1]), max_degree=int(max_degree),
                        metric=PA_IP if metric in ("ip", PA_IP) else PA_L2,
                        sub_offsets=_ptr(so), sub_neighbors=_ptr(sn), member_flags=_ptr(mf),
                        reduced=_ptr(red), basis=_ptr(bas), fes_r=int(coff.shape[0] - 1),
                        fes_centroids=_ptr(cen), fes_cell_off=_ptr(coff), fes_pool_ids=_ptr(pool),
                        device=int(device), reduced_fp16=1 if reduced_fp16 else 0, reduced_stride=int(rstride))
        h = C.c_void_p()
        _check(lib().pa_build(C.byref(p), C.byref(h)))
        self._h = h
        self.n, self.dim, self.rdim, self.device = n, p.dim, p.rdim, int(device)
        self.metric = "ip" if p.metric == PA_IP else "l2"
        self._host_keep = None

    @classmethod
    def from_instance(cls, inst: dict, device=0, max_degree=None, reduced_fp16=False):
        return cls(sub_offsets=inst["sub_offsets"], sub_neighbors=inst["sub_neighbors"],
                   reduced=inst["reduced"], basis=inst["basis"], fes_centroids=inst["fes_centroids"],
                   fes_cell_off=inst["fes_cell_off"], fes_pool_ids=inst["fes_pool_ids"],
                   member_flags=inst.get("member_flags"), metric=inst.get("metric", "l2"),
                   max_degree=max_degree, device=device, reduced_fp16=reduced_fp16)

    # -- replication (pa_replica_meta_of / pa_build_replica / pa_replica_buffers) --
    def replica_meta(self) -> ReplicaMeta:
        m = ReplicaMeta()
        _check(lib().pa_replica_meta_of(self._h, C.byref(m)))
        return m

    @classmethod
    def empty_replica(cls, meta: ReplicaMeta, device: int) -> "Index":
        """An unfilled replica with `meta`'s layout on `device` (fill every buffer, e.g. by broadcast)."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        _check(lib().pa_build_replica(C.byref(meta), int(device), C.byref(h)))
        self._h = h
        self.n, self.dim, self.rdim, self.device = int(meta.n), int(meta.dim), int(meta.rdim), int(device)
        self.metric = "ip" if meta.metric == PA_IP else "l2"
        self._host_keep = None
        return self

    def replica_buffers(self) -> list[tuple[int, int]]:
        """[(device pointer, bytes)] of the replica's device arrays, in the fixed ABI order."""
        cnt = C.c_int32()
        _check(lib().pa_replica_buffers(self._h, None, 0, C.byref(cnt)))
        arr = (Buffer * cnt.value)()
        _check(lib().pa_replica_buffers(self._h, arr, cnt.value, C.byref(cnt)))
        return [(int(b.ptr or 0), int(b.bytes)) for b in arr]

    # -- pa_attach_host -----------------------------------------------------
    def attach_host(self, full_offsets, full_neighbors, rotated):
        keep = (_c(full_offsets, np.int64), _c(full_neighbors, np.int32), _c(rotated, np.float32))
        _check(lib().pa_attach_host(self._h, _ptr(keep[0]), _ptr(keep[1]), _ptr(keep[2])))
        self._host_keep = keep          # borrowed by the library until destroy

    # -- pa_search ------------------------------------------------------------
    def search(self, queries, k=10, ef=64, opts: SearchOpts | None = None, out=None, **kw):
        """pa_search on HOST buffers.  `queries`/`out` may be numpy arrays or
        (pinned) CPU torch tensors; results are written into `out`."""
        qp, m, _keep = _host_rows(queries, self.dim, np.float32, "queries")
        if out is None:
            out = (np.empty((m, k), np.int32), np.empty((m, k), np.float32))
        op = []
        for o_, dt, nm in zip(out, (np.int32, np.float32), ("out ids", "out dists")):
            if not hasattr(o_, "data_ptr") and not (isinstance(o_, np.ndarray) and o_.flags.c_contiguous
                                                    and o_.dtype == dt):
                raise ValueError(f"{nm}: expected a C-contiguous {np.dtype(dt).name} array [m][k]")
            p_, mo, _ = _host_rows(o_, k, dt, nm)
            if mo != m:
                raise ValueError(f"{nm}: {mo} rows for {m} queries")
            op.append(p_)
        o = opts if opts is not None else make_opts(**kw)
        _check(lib().pa_search(self._h, qp, m, k, ef, C.byref(o), op[0], op[1]))
        return out

    def search_candidates(self, queries, ef=64, opts: SearchOpts | None = None, **kw):
        qp, m, q = _host_rows(queries, self.dim, np.float32, "queries")
        ids = np.empty((m, ef), np.int32)
        d = np.empty((m, ef), np.float32)
        o = opts if opts is not None else make_opts(**kw)
        _check(lib().pa_search_candidates(self._h, qp, m, ef, C.byref(o), _ptr(ids), _ptr(d)))
        return ids, d

    # -- pa_search_device (torch CUDA tensors; pointers only) ----------------
    def search_device(self, q, k, ef, out_ids, out_d, opts: SearchOpts | None = None, debug: Debug | None = None,
                      stream=None, **kw):
        o = opts if opts is not None else make_opts(**kw)
        _dev_rows(q, None, self.dim, np.float32, self.device, "queries")
        m = int(q.shape[0])
        _dev_rows(out_ids, m, k, np.int32, self.device, "out_ids")
        _dev_rows(out_d, m, k, np.float32, self.device, "out_d")
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(q.device).cuda_stream
        _check(lib().pa_search_device(self._h, C.c_void_p(q.data_ptr()), int(q.shape[0]), k, ef, C.byref(o),
                                      C.c_void_p(out_ids.data_ptr()), C.c_void_p(out_d.data_ptr()),
                                      C.byref(debug) if debug is not None else None, C.c_void_p(stream)))

    def entries_device(self, q, E, method=PA_ENTRIES_FES, e0=0, beam=0, out=None, out_d=None, n_dist=None,
                       stream=None):
        """pa_entries_device: the E entries of every DEVICE query row (FES or the
        two-hop baseline, NEXT-f4).  `out` [m][E] int32 device tensor (allocated if
        None); `out_d` [m][E] fp32 and `n_dist` [m] int32 optional (two-hop only)."""
        _dev_rows(q, None, self.dim, np.float32, self.device, "queries")
        m = int(q.shape[0])
        if out is None:
            import torch
            out = torch.empty(m, E, dtype=torch.int32, device=q.device)
        _dev_rows(out, m, E, np.int32, self.device, "entries")
        if out_d is not None:
            _dev_rows(out_d, m, E, np.float32, self.device, "entry dists")
        if n_dist is not None:
            _dev_rows(n_dist.view(-1, 1), m, 1, np.int32, self.device, "n_dist")
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(q.device).cuda_stream
        _check(lib().pa_entries_device(self._h, C.c_void_p(q.data_ptr()), m, int(E), int(method), int(e0), int(beam),
                                       C.c_void_p(out.data_ptr()),
                                       C.c_void_p(out_d.data_ptr()) if out_d is not None else None,
                                       C.c_void_p(n_dist.data_ptr()) if n_dist is not None else None,
                                       C.c_void_p(stream)))
        return out

    def stats(self) -> dict:
        s = Stats()
        _check(lib().pa_get_stats(self._h, C.byref(s), C.sizeof(Stats)))
        return s.asdict()

    def close(self):
        if getattr(self, "_h", None):
            lib().pa_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def debug_buffers(m, ef, E, trace_cap=0, device="cuda"):
    """Allocate torch device buffers for pa_debug and return (Debug struct, dict of tensors)."""
    import torch
    t = dict(cell=torch.empty(m, dtype=torch.int32, device=device),
             entries=torch.empty(m, E, dtype=torch.int32, device=device),
             cand_ids=torch.empty(m, ef, dtype=torch.int32, device=device),
             cand_dists=torch.empty(m, ef, dtype=torch.float32, device=device),
             counters=torch.zeros(m, 4, dtype=torch.int32, device=device))
    if trace_cap:
        t.update(trace_expand=torch.full((m, trace_cap), -1, dtype=torch.int32, device=device),
                 trace_visit=torch.full((m, trace_cap), -1, dtype=torch.int32, device=device),
                 trace_nexp=torch.zeros(m, dtype=torch.int32, device=device),
                 trace_nvis=torch.zeros(m, dtype=torch.int32, device=device))
    d = Debug(cell=t["cell"].data_ptr(), entries=t["entries"].data_ptr(), cand_ids=t["cand_ids"].data_ptr(),
              cand_dists=t["cand_dists"].data_ptr(), counters=t["counters"].data_ptr(), trace_cap=trace_cap)
    if trace_cap:
        d.trace_expand = t["trace_expand"].data_ptr()
        d.trace_visit = t["trace_visit"].data_ptr()
        d.trace_nexp = t["trace_nexp"].data_ptr()
        d.trace_nvis = t["trace_nvis"].data_ptr()
    return d, t
