#!/usr/bin/env python
"""PilotANN GPU-stage benchmark (BASELINE.json metric: QPS at Recall@10 = 0.90).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1] [--impl ours|reference]

One step = one pass of the whole GPU stage (a1 projection → a2/a4 FES → a5/a6
traversal → a7 candidate/top-k output) over one batch of this rank's queries
(10K at C1), inputs resident in HBM.  The operating point is the smallest ef
of a sweep whose Recall@10 against the subgraph ground truth (GT_sub, exact
top-10 over members in the reduced space) is ≥ 0.90.
Multi-GPU (torchrun): every rank builds a replica of the same index and
searches its own shard of the global query set; no data-path collective
 — only a barrier and a MAX all-reduce of the timings.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

EF_SWEEP = (16, 24, 32, 40, 48, 56, 64, 72, 80, 88, 96, 112, 128, 160, 192, 224, 256)   # smallest ef reaching the target
TARGET_RECALL = 0.90


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and "Active" in r[5 + i]
                          and "Not" not in r[5 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def ncu_traffic(workload, ef, bloom=0, kernel="k_traverse"):
    """DRAM bytes per launch of `kernel` from a committed `ncu --set full` capture
    (profiles/ncu_traffic.json), when one exists for this workload, ef and visited set."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(workload, {}).get(str(ef) + (f"_bloom{bloom}" if bloom else ""))
        return (e["dram_bytes"], e["source"]) if e and e.get("kernel") == kernel else (None, None)
    except (OSError, ValueError, KeyError):
        return None, None


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# --------------------------------------------------------------- instance --
def parse_overrides(items):
    """--set key=value pairs → typed Config overrides (NEXT-f2 operating points)."""
    out = {}
    for it in items or []:
        k, v = it.split("=", 1)
        out[k] = float(v) if "." in v else int(v)
    return out


def make_instance(cfg_name, world, rank, m_per_rank, cache=None, overrides=None):
    import torch
    import datagen as dg
    ov = dict(overrides or {})
    cfg = dg.get_config(cfg_name, m=m_per_rank * world, **ov)
    if ov:
        cfg.name += "[" + ",".join(f"{k}={v}" for k, v in sorted(ov.items())) + "]"
    t0 = time.time()
    tag = "_".join(f"{k}{v}" for k, v in sorted(ov.items()))
    path = os.path.join(cache, f"inst_{cfg_name}{tag}_{world}_{rank}_{m_per_rank}.npz") if cache else None
    if path and os.path.exists(path):
        z = np.load(path, allow_pickle=False)
        inst = {k: z[k] for k in z.files}
        inst["cfg"], inst["metric"] = cfg, cfg.metric
        log(f"[rank {rank}] instance loaded from {path} in {time.time() - t0:.1f}s")
        return cfg, inst
    inst = dg.build_instance(cfg, device=f"cuda:{torch.cuda.current_device()}", gt=False)
    from paper_2503_21206_b200.dist import shard_bounds
    Q = inst["queries"]
    lo, hi = shard_bounds(Q.shape[0], rank, world)
    inst["queries"] = np.ascontiguousarray(Q[lo:hi])
    # ground truths for this rank's shard (exhaustive scan; recall measurement only)
    dev = f"cuda:{torch.cuda.current_device()}"
    V = torch.from_numpy(inst["V64"]).to(dev)
    Qh = torch.from_numpy(inst["queries"]).to(dev).double() @ V
    Xh = torch.from_numpy(inst["rotated"]).to(dev)
    inst["gt_ids"], _ = dg.ground_truth(Qh, Xh, cfg.k, cfg.metric)
    mem = torch.from_numpy(np.flatnonzero(inst["member_flags"])).to(dev)
    Xr = Xh[:, :cfg.dp].contiguous()
    inst["gt_sub_ids"], _ = dg.ground_truth(Qh[:, :cfg.dp], Xr, cfg.k, cfg.metric, ids=mem)
    del Xh, Xr, mem
    torch.cuda.empty_cache()
    log(f"[rank {rank}] instance {cfg.name}: N={cfg.N} D={cfg.D} d'={cfg.dp} members={int(inst['member_flags'].sum())}"
        f" m={m_per_rank} built in {time.time() - t0:.1f}s")
    if path:
        os.makedirs(cache, exist_ok=True)
        np.savez(path, **{k: v for k, v in inst.items() if isinstance(v, np.ndarray)})
    return cfg, inst


def recall_at(ids, gt, k):
    ids = np.asarray(ids)[:, :k]
    gt = np.asarray(gt)[:, :k]
    hit = sum(len(set(a.tolist()) & set(b.tolist())) for a, b in zip(ids, gt))
    return hit / (k * ids.shape[0])


# ------------------------------------------------------------- reference --
def run_reference(args, rank, world):
    """--impl reference: the ORACLE (plain fp64 C++) on the host cores, on a
    bounded sample of this workload per step."""
    if rank != 0:
        return
    import torch
    import oracle as orc
    orc.build()
    torch.cuda.set_device(0) if torch.cuda.is_available() else None
    cfg, inst = make_instance(args.config, 1, 0, args.m, args.cache, parse_overrides(args.set)) \
        if torch.cuda.is_available() else make_cpu_instance(args)
    cores = os.cpu_count()
    sample = args.ref_sample
    Q = inst["queries"]
    ef = args.ef
    if not ef:                       # same operating-point rule as the GPU arm, on a sample
        probe = min(len(Q), 500)
        for e in EF_SWEEP:
            rr = orc.search(inst, queries=Q[:probe], k=cfg.k, ef=e, stages=1, bloom_log2=args.bloom or None)
            if recall_at(rr["ids"], inst["gt_sub_ids"][:probe], cfg.k) >= TARGET_RECALL:
                ef = e
                break
        ef = ef or EF_SWEEP[-1]
    for _ in range(args.warmup):
        orc.search(inst, queries=Q[:min(sample, 64)], k=cfg.k, ef=ef, stages=1, bloom_log2=args.bloom or None)
    times = []
    for s in range(args.steps):
        qs = Q[(s * sample) % len(Q):][:sample]
        t = time.perf_counter()
        r = orc.search(inst, queries=qs, k=cfg.k, ef=ef, stages=1, bloom_log2=args.bloom or None)
        times.append(time.perf_counter() - t)
    qps = sample * len(times) / sum(times)
    rec = recall_at(r["ids"], inst["gt_sub_ids"][(s * sample) % len(Q):][:sample], cfg.k)
    line = {"impl": "reference", "metric": "QPS at Recall@10=0.90 (GPU stage, GT_sub)", "value": qps,
            "unit": "queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "ef": ef, "k": cfg.k, "sample_queries_per_step": sample},
            "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": cores, "kind": "oracle",
                             "sample": f"{sample} queries per step of {cfg.name}, stage 1, ef={ef}"
                                       + (f", bloom 3x2^{args.bloom}" if args.bloom else "")},
            "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "recall_at_10_sample": rec}
    print(json.dumps(line), flush=True)


def make_cpu_instance(args):
    import datagen as dg
    cfg = dg.get_config(args.config, m=args.m, **parse_overrides(args.set))
    return cfg, dg.build_instance(cfg)


# ------------------------------------------------------------------ ours --
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import __graft_entry__ as ge
    ge.build_library()
    import paper_2503_21206_b200 as pa

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg, inst = make_instance(args.config, world, rank, args.m, args.cache, parse_overrides(args.set))
    k = cfg.k
    m = inst["queries"].shape[0]
    t0 = time.time()
    ix = pa.Index.from_instance(inst, device=local_rank, reduced_fp16=args.reduced == "fp16")
    ix.attach_host(inst["full_offsets"], inst["full_neighbors"], inst["rotated"])
    log(f"[rank {rank}] pa_build {time.time() - t0:.1f}s")

    if args.repeat_queries > 1:      # experiment: same queries tiled R times (tail-effect probe)
        inst = dict(inst, queries=np.tile(inst["queries"], (args.repeat_queries, 1)),
                    gt_sub_ids=np.tile(inst["gt_sub_ids"], (args.repeat_queries, 1)),
                    gt_ids=np.tile(inst["gt_ids"], (args.repeat_queries, 1)))
        m = inst["queries"].shape[0]
    qd = torch.from_numpy(inst["queries"]).to(dev)
    out_i = torch.empty(m, k, dtype=torch.int32, device=dev)
    out_d = torch.empty(m, k, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    gt_key = "gt_sub_ids" if args.gt == "sub" else "gt_ids"     # operating-point rule's ground truth

    def step(ef):
        ix.search_device(qd, k, ef, out_i, out_d, stream=stream.cuda_stream, bloom_log2=args.bloom)

    # ---- operating point: smallest ef with Recall@10 (vs GT_sub) ≥ 0.90
    sweep = []
    chosen = None
    for ef in ([args.ef] if args.ef else EF_SWEEP):
        step(ef)
        torch.cuda.synchronize()
        rec = recall_at(out_i.cpu().numpy(), inst[gt_key], k)
        st = ix.stats()
        sweep.append({"ef": ef, "recall_at_10": round(rec, 4), "gpu_ms": round(st["ms_total_gpu"], 3),
                      "n_dist_per_q": st["sum_n_dist"] / m, "n_exp_per_q": st["sum_n_exp"] / m})
        log(f"[rank {rank}] ef={ef} recall@10={rec:.4f} gpu {st['ms_total_gpu']:.3f} ms "
            f"n_dist/q {st['sum_n_dist'] / m:.1f} n_exp/q {st['sum_n_exp'] / m:.1f}")
        if chosen is None and rec >= TARGET_RECALL:
            chosen = ef
            if not args.full_sweep:
                break
    if chosen is None:
        chosen = sweep[-1]["ef"]
    if world > 1:
        t = torch.tensor([chosen], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        chosen = int(t.item())
    ef = chosen

    # ---- timed region: W warm-up, K steps; L2 flushed between steps (512 MB write)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    ell_w = 32 if int(np.diff(inst["sub_offsets"]).max()) <= 32 else 64

    def timed(step_fn, ixv, ef_, fp16, clk=None):
        for _ in range(args.warmup):
            step_fn(ef_)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        acc = dict(trav=[], proj=[], fes=[], launches=0, bytes=0.0)
        row_bytes = 2 * ((cfg.dp + 7) // 8 * 8) if fp16 else 4 * cfg.dp
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.fill_(float(i))
            ev[i][0].record(stream)
            step_fn(ef_)
            ev[i][1].record(stream)
            st = ixv.stats()                      # syncs the traversal events of this step (outside the events)
            acc["trav"].append(st["ms_traverse"])
            acc["proj"].append(st["ms_project"])
            acc["fes"].append(st["ms_fes"])
            acc["launches"] += st["kernel_launches"]
            acc["bytes"] = st["sum_n_exp"] * 4 * ell_w + st["sum_n_dist"] * row_bytes
            acc["n_exp"], acc["n_dist"] = st["sum_n_exp"], st["sum_n_dist"]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        step_ms = [a.elapsed_time(b) for a, b in ev]
        ms_, trav_ = sum(step_ms) / len(step_ms), sum(acc["trav"]) / len(acc["trav"])
        if world > 1:
            t = torch.tensor([ms_, trav_], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_, trav_ = float(t[0]), float(t[1])
        acc.update(ms=ms_, trav_ms=trav_)
        return acc

    with ClockSampler(local_rank) as clk:
        main = timed(step, ix, ef, args.reduced == "fp16")
    ms, trav, launches, bytes_alg = main["ms"], main["trav_ms"], main["launches"], main["bytes"]
    trav_ms, proj_ms, fes_ms = main["trav"], main["proj"], main["fes"]
    rec = recall_at(out_i.cpu().numpy(), inst["gt_sub_ids"], k)
    rec_full = recall_at(out_i.cpu().numpy(), inst["gt_ids"], k)
    qps = m * world / (ms / 1e3)

    # ---- variants beside the headline: exact visited set and/or binary16-stored
    # reduced rows (NEXT-f1), each at its own smallest ef with Recall@10 (GT_sub) >= 0.90
    def variant(name, what, fp16, bloom):
        ixv = pa.Index.from_instance(inst, device=local_rank, reduced_fp16=fp16) if fp16 else ix

        def stepv(e):
            ixv.search_device(qd, k, e, out_i, out_d, stream=stream.cuda_stream, bloom_log2=bloom)
        efv = None
        for e in EF_SWEEP:
            stepv(e)
            torch.cuda.synchronize()
            if recall_at(out_i.cpu().numpy(), inst[gt_key], k) >= TARGET_RECALL:
                efv = e
                break
        efv = efv or EF_SWEEP[-1]
        if world > 1:
            t = torch.tensor([efv], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            efv = int(t.item())
        v = timed(stepv, ixv, efv, fp16)
        rv = recall_at(out_i.cpu().numpy(), inst[gt_key], k)
        pk, _ = measured_peaks()
        ach = v["bytes"] / (v["trav_ms"] / 1e3) / 1e9
        if fp16:
            ixv.close()
        return {"what": what, "reduced_storage": "fp16" if fp16 else "fp32", "bloom_log2": bloom,
                "value": round(m * world / (v["ms"] / 1e3), 1), "unit": "queries/s", "ef": efv,
                "recall_at_10_gt_sub": round(rv, 4), "ms_per_step": round(v["ms"], 4),
                "traverse_ms": round(v["trav_ms"], 4), "alg_bytes_per_launch": v["bytes"],
                "n_dist_per_q": v["n_dist"] / m, "n_exp_per_q": v["n_exp"] / m,
                "roofline_frac": round(ach / pk, 4), "achieved_gbs": round(ach, 1)}

    variants = {}
    if not args.no_f1:
        want = [x for x in args.variants.split(",") if x]
        specs = {
            "exact": ("exact visited set (smem hash + global spill) instead of the paper's bloom filter; "
                      "fp32 rows", False, 0),
            "fp16": ("NEXT-f1: reduced rows stored as binary16 (rounded once at build; fp32 arithmetic; parity "
                     f"vs the oracle on the same rounded values), bloom 3 x 2^{args.bloom_bits}", True, args.bloom_bits),
            "exact_fp16": ("exact visited set + binary16 rows", True, 0),
        }
        for name in want:
            if name in specs and args.reduced == "fp32" and not (name == "exact" and not args.bloom):
                variants[name] = variant(name, *specs[name])
                log(f"[rank {rank}] variant {name}: {variants[name]['value']:.0f} q/s ef={variants[name]['ef']} "
                    f"trav {variants[name]['traverse_ms']:.3f} ms")

    # ---- e2e through the public host API: pinned host queries in, host results out
    hq = torch.from_numpy(inst["queries"]).pin_memory()
    ho = (torch.empty(m, k, dtype=torch.int32).pin_memory(), torch.empty(m, k, dtype=torch.float32).pin_memory())
    for _ in range(2):
        ix.search(hq, k=k, ef=ef, out=ho, bloom_log2=args.bloom)
    e2e_t = []
    for _ in range(max(3, args.steps)):
        t = time.perf_counter()
        ix.search(hq, k=k, ef=ef, out=ho, bloom_log2=args.bloom)
        e2e_t.append(time.perf_counter() - t)
    e2e_s = sum(e2e_t) / len(e2e_t)
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])
    e2e_qps = m * world / e2e_s

    # ---- end-to-end with host stages ②③ (M1, full-space GT), optional
    full = None
    if not args.no_full:
        full = measure_full(ix, inst, cfg, args, rank)
    # ---- NEXT-f3: all three stages on the GPU (X̂ and the full graph in HBM), device-timed
    full_gpu = None
    if not args.no_full:
        sw = []
        for e in (16, 32, 48, 64, 96, 128, 192, 256):
            def stepf(ee=e):
                ix.search_device(qd, k, ee, out_i, out_d, stream=stream.cuda_stream, bloom_log2=args.bloom,
                                 stages=pa.PA_STAGES_FULL_GPU)
            for _ in range(args.warmup):
                stepf()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                flush.fill_(1.0)
                stepf()
            e1.record(stream)
            torch.cuda.synchronize()
            st = ix.stats()
            msf = e0.elapsed_time(e1) / args.steps
            rf = recall_at(out_i.cpu().numpy(), inst["gt_ids"], k)
            sw.append({"ef": e, "recall_at_10": round(rf, 4), "qps": round(m * world / (msf / 1e3), 1),
                       "ms_per_step": round(msf, 4), "refine_ms": round(st["ms_refine"], 4),
                       "n_dist23_per_q": (st["sum_n_dist2"] + st["sum_n_dist3"]) / m})
            log(f"[rank {rank}] FULL_GPU ef={e} recall@10={rf:.4f} qps {sw[-1]['qps']:.0f} refine {st['ms_refine']:.3f} ms")
            if rf >= TARGET_RECALL:
                break
        ok = [x for x in sw if x["recall_at_10"] >= TARGET_RECALL]
        full_gpu = {"metric": "QPS at Recall@10=0.90 (stages 1-3 all on the GPU, full-space GT; NEXT-f3)",
                    "unit": "queries/s", "value": ok[0]["qps"] if ok else None, "ef": ok[0]["ef"] if ok else None,
                    "timing": "device (CUDA events), inputs resident, L2 flushed per step", "sweep": sw}
    # ---- NEXT-f4: Table 6 ablation — components removed cumulatively
    ablation = None
    if args.ablation:
        ablation = []
        fl = 0
        for name, bit in (("full", 0), ("-pipelining", pa.PA_NO_PIPELINE), ("-FES", pa.PA_NO_FES),
                          ("-stage2", pa.PA_NO_STAGE2), ("-stage1", pa.PA_NO_STAGE1)):
            fl |= bit
            r_ = measure_full(ix, inst, cfg, args, rank, flags=fl)
            ablation.append({"removed": name, "flags": fl, "qps_at_0.90": r_["value"], "ef": r_["ef"],
                             "sweep": r_["sweep"]})
            log(f"[rank {rank}] ablation {name}: {r_['value']} q/s ef={r_['ef']}")

    peak, peak_src = measured_peaks()
    achieved = bytes_alg / (trav / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(cfg.name, ef, args.bloom)
    line = None
    if rank == 0:
        oinst = inst if args.reduced == "fp32" else dict(inst, reduced=inst["reduced"].astype(np.float16).astype(np.float32))
        cpu = None if args.no_cpu_baseline else cpu_baseline(oinst, cfg, ef, args)
        clocks = clk.summary()
        line = {
            "metric": "QPS at Recall@10=0.90 (GPU stage: projection+FES+subgraph traversal, "
                      + ("GT_sub)" if args.gt == "sub" else "full-space GT)"),
            "value": round(qps, 1), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "N": cfg.N, "D": cfg.D, "d_reduced": cfg.dp, "metric": cfg.metric,
                       "sampling_ratio": cfg.ratio, "queries_per_gpu": m, "k": k, "ef": ef,
                       "recall_at_10_gt_sub": round(rec, 4), "recall_at_10_full_gt_gpu_only": round(rec_full, 4),
                       "l2": "flushed between steps (512 MB write), per-step CUDA events",
                       "reduced_storage": args.reduced,
                       "visited": f"bloom 3x2^{args.bloom} bits" if args.bloom else "exact",
                       "parallelism": f"query-sharded x{world}, replicated index"},
            "ef_sweep": sweep,
            "roofline": {"bound": "hbm", "kernel": "k_traverse", "achieved": round(achieved, 1),
                         "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "traffic_source": traffic_src,
                         "traverse_ms": round(trav, 4), "alg_bytes_per_launch": bytes_alg,
                         "kernel_ms": {"project": round(sum(proj_ms) / len(proj_ms), 4),
                                       "fes": round(sum(fes_ms) / len(fes_ms), 4), "traverse": round(trav, 4)},
                         "bytes_model": "sum_q n_exp*4*ELLW + n_dist*row_bytes (4*d' fp32 / 2*round8(d') fp16)",
                         "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_qps, 1), "unit": "queries/s", "h2d_bytes_per_step": m * cfg.D * 4,
                    "d2h_bytes_per_step": m * k * 8},
            "end_to_end_full": full,
            "full_gpu": full_gpu,
            "ablation_table6": ablation,
            "variants": variants,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    ix.close()


def measure_full(ix, inst, cfg, args, rank, flags=0):
    """M1: pa_search(PA_STAGES_FULL) — GPU stage ① + host ② ③ — against full-space GT."""
    import paper_2503_21206_b200 as pa
    k = cfg.k
    m = inst["queries"].shape[0]
    chosen = None
    sweep = []
    hq = inst["queries"]
    for ef in (16, 32, 64, 128, 192, 256):
        kw = dict(stages=pa.PA_STAGES_FULL, bloom_log2=args.bloom, flags=flags)
        ix.search(hq, k=k, ef=ef, **kw)                                 # warm-up (pinned buffers, pools)
        t = time.perf_counter()
        ids, _ = ix.search(hq, k=k, ef=ef, **kw)
        dt = time.perf_counter() - t
        rec = recall_at(ids, inst["gt_ids"], k)
        st = ix.stats()
        sweep.append({"ef": ef, "recall_at_10": round(rec, 4), "qps": round(m / dt, 1),
                      "host_ms": round(st["ms_host_stages"], 2), "gpu_ms": round(st["ms_total_gpu"], 3)})
        log(f"[rank {rank}] FULL ef={ef} recall@10={rec:.4f} qps {m / dt:.0f} host {st['ms_host_stages']:.1f} ms")
        if rec >= TARGET_RECALL:
            chosen = sweep[-1]
            break
    return {"metric": "QPS at Recall@10=0.90 (stages 1-3, full-space GT)", "unit": "queries/s",
            "value": chosen["qps"] if chosen else None, "ef": chosen["ef"] if chosen else None,
            "host_threads": os.cpu_count(), "sweep": sweep}


def cpu_baseline(inst, cfg, ef, args):
    """The oracle (plain fp64 C++, untuned) on the host cores, on a bounded
    sample of the same workload at the same ef."""
    import oracle as orc
    orc.build()
    Q = inst["queries"]
    cal = Q[:64]
    t = time.perf_counter()
    orc.search(inst, queries=cal, k=cfg.k, ef=ef, stages=1, bloom_log2=args.bloom or None)
    per_q = (time.perf_counter() - t) / len(cal)
    n = int(min(len(Q), max(256, args.cpu_seconds / max(per_q, 1e-6))))
    t = time.perf_counter()
    r = orc.search(inst, queries=Q[:n], k=cfg.k, ef=ef, stages=1, bloom_log2=args.bloom or None)
    dt = time.perf_counter() - t
    return {"value": round(n / dt, 1), "unit": "queries/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"first {n} queries of {cfg.name}, stage 1 (projection+FES+traversal), ef={ef}, fp64"
                      + (f", bloom 3x2^{args.bloom}" if args.bloom else ""),
            "recall_at_10_gt_sub": round(recall_at(r["ids"], inst["gt_sub_ids"][:n], cfg.k), 4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C1")
    ap.add_argument("--m", type=int, default=10_000, help="queries per GPU")
    ap.add_argument("--ef", type=int, default=0, help="fix ef (0 = sweep to Recall@10 >= 0.90)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-sample", type=int, default=500)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--full-sweep", action="store_true")
    ap.add_argument("--no-full", action="store_true")
    ap.add_argument("--gt", default="sub", choices=["sub", "full"],
                    help="ground truth of the Recall@10 >= 0.90 rule: the sampled subgraph's (stage-1 target) or "
                         "full-space (GPU-only operating points, NEXT-f2)")
    ap.add_argument("--set", action="append", default=[], metavar="KEY=VALUE",
                    help="override a datagen Config field (e.g. ratio=1.0, dp=96: NEXT-f2 operating points)")
    ap.add_argument("--ablation", action="store_true", help="NEXT-f4: Table 6 cumulative ablation of the full pipeline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-f1", action="store_true", help="skip the binary16-storage (NEXT-f1) variant")
    ap.add_argument("--cache", default=None, help="dir to cache the generated instance (same-call reuse only)")
    ap.add_argument("--repeat-queries", type=int, default=1, help="experiment only: tile the query batch R times")
    ap.add_argument("--reduced", default="fp32", choices=["fp32", "fp16"],
                    help="storage of the reduced rows on the GPU (fp16 = NEXT-f1; parity on the rounded values)")
    ap.add_argument("--bloom", type=int, default=12,
                    help="visited set of the headline path: the paper's shared-memory bloom filter (P:L392-395) "
                         "of 3 x 2^BLOOM bits per query; 0 = exact set")
    ap.add_argument("--bloom-bits", type=int, default=12, help="bloom size of the binary16 variant")
    ap.add_argument("--variants", default="exact,fp16,exact_fp16", help="variants measured beside the headline")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1 and args.impl == "ours":
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
