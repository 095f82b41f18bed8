"""NEXT-f4: FES vs the two-hop baseline (§6.3 "FES analysis", Fig
"FES benefit" P:L946-970): entry quality as Recall@1000 of the entry set against
the subgraph's exact top-1000 (reduced space), and entry-selection throughput on
the GPU (projection + selection, CUDA events, inputs resident, L2 flushed).

usage: python scripts/f4_fes_vs_twohop.py [C3S] > profiles/r2_f4_fes_vs_twohop.json
"""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen as dg  # noqa: E402
import paper_2503_21206_b200 as pa  # noqa: E402
import __graft_entry__ as ge  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3S"
ge.build_library()
cfg = dg.get_config(name)
t0 = time.time()
inst = dg.build_instance(cfg, device="cuda", gt=False)
print(f"[f4] instance {cfg.name} in {time.time() - t0:.1f}s", file=sys.stderr, flush=True)
dev = torch.device("cuda")
V = torch.from_numpy(inst["V64"]).to(dev)
Qh = torch.from_numpy(inst["queries"]).to(dev).double() @ V
mem = torch.from_numpy(np.flatnonzero(inst["member_flags"])).to(dev)
Xr = torch.from_numpy(np.ascontiguousarray(inst["reduced"])).to(dev)
gt1000, _ = dg.ground_truth(Qh[:, :cfg.dp], Xr, 1000, cfg.metric, ids=mem)
# the fixed entry e0: the member nearest the mean member row (the graph's "medoid", HNSW-style fixed entry)
mu = Xr[mem].double().mean(0)
e0 = int(mem[torch.argmin(((Xr[mem].double() - mu) ** 2).sum(1))].item())
del Xr, V
torch.cuda.empty_cache()
ix = pa.Index.from_instance(inst)
q = torch.from_numpy(inst["queries"]).to(dev)
m = q.shape[0]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
gts = [set(r.tolist()) for r in gt1000]


def run(E, method, beam=0, reps=10):
    out = torch.empty(m, E, dtype=torch.int32, device=dev)
    nd = torch.empty(m, dtype=torch.int32, device=dev) if method == pa.PA_ENTRIES_TWO_HOP else None
    for _ in range(3):
        ix.entries_device(q, E, method=method, e0=e0, beam=beam, out=out, n_dist=nd)
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ix.entries_device(q, E, method=method, e0=e0, beam=beam, out=out, n_dist=nd)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    ids = out.cpu().numpy()
    rec = float(np.mean([len(set(r[r >= 0].tolist()) & g) / 1000.0 for r, g in zip(ids, gts)]))
    row = {"E": E, "ms": round(ms, 4), "qps": round(m / ms * 1e3, 1), "recall_at_1000": round(rec, 5)}
    if nd is not None:
        row["beam"] = beam
        row["visited_per_q"] = float(nd.float().mean().item())
    print(f"[f4] {row}", file=sys.stderr, flush=True)
    return row


fes = [run(E, pa.PA_ENTRIES_FES) for E in (1, 2, 4, 8, 16, 32, 64, 128, 256)]
two = [run(256, pa.PA_ENTRIES_TWO_HOP, beam=b) for b in (0, 1, 2, 4, 8, 16, 32)]
two_e = [run(E, pa.PA_ENTRIES_TWO_HOP, beam=32) for E in (1, 4, 16, 64)]
ix.close()
print(json.dumps({"experiment": "NEXT-f4 FES vs two-hop entry selection (P:L986-989)", "workload": cfg.name,
                  "queries": m, "e0": e0, "gt": "exact top-1000 over subgraph members in the reduced space",
                  "timing": "CUDA events around pa_entries_device (projection + selection), median of 10, "
                            "L2 flushed (256 MB write) before each",
                  "fes_by_E": fes, "two_hop_by_beam_E256": two, "two_hop_beam32_by_E": two_e}))
