"""Diagnostic at 100M: is stage-1 recall (GT_sub) limited by the graph or by the FES entries?
GPU ef sweep, then the oracle with a PERFECT entry (the GT_sub top-1 as the only entry)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen as dg
from datagen import large as lg
import paper_2503_21206_b200 as pa
import __graft_entry__ as ge
import oracle as orc

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = dg.get_config(name)
ge.build_library()
orc.build()
t = time.time()
inst = lg.build_instance_large(cfg, device="cuda", cache=os.environ.get("PA_CACHE"), gt_k=10)
torch.cuda.empty_cache()
print(f"instance {time.time() - t:.1f}s  sub degree mean {np.diff(inst['sub_offsets']).sum() / inst['member_flags'].sum():.2f}"
      f" full degree mean {inst['full_neighbors'].size / cfg.N:.2f}", flush=True)
ix = pa.Index.from_instance(inst)
q = torch.from_numpy(inst["queries"]).cuda()
m = q.shape[0]
oi = torch.empty(m, 10, dtype=torch.int32, device="cuda")
od = torch.empty(m, 10, dtype=torch.float32, device="cuda")
rec = lambda ids, gt: sum(len(set(a) & set(b)) for a, b in zip(ids[:, :10].tolist(), gt[:, :10].tolist())) / (10 * len(ids))
for ef in (64, 96, 128, 160, 192, 256):
    for bl in (0, 12, 13, 14):
        try:
            ix.search_device(q, 10, ef, oi, od, bloom_log2=bl)
        except pa.PAError as e:
            print(f"GPU ef={ef} bloom={bl}: {e}", flush=True)
            continue
        torch.cuda.synchronize()
        st = ix.stats()
        print(f"GPU ef={ef} bloom={bl} GT_sub {rec(oi.cpu().numpy(), inst['gt_sub_ids']):.4f} trav {st['ms_traverse']:.3f} ms "
              f"gpu {st['ms_total_gpu']:.3f} ms n_dist/q {st['sum_n_dist'] / m:.0f} n_exp/q {st['sum_n_exp'] / m:.0f}", flush=True)
ix.close()
if os.environ.get("DIAG_ORACLE", "1") != "1":
    sys.exit(0)
# oracle, perfect entry: one query at a time with pool = [GT_sub top-1]
sel = np.arange(0, m, m // 40)[:40]
for ef in (64, 256, 1024):
    hits = 0
    for qi in sel:
        top1 = int(inst["gt_sub_ids"][qi, 0])
        sub = dict(inst, queries=inst["queries"][qi:qi + 1], fes_cell_off=np.array([0, 1], np.int64),
                   fes_pool_ids=np.array([top1], np.int32), fes_centroids=inst["fes_centroids"][:1])
        r = orc.search(sub, k=10, ef=ef, stages=1, entries=1, threads=1)
        hits += len(set(r["ids"][0].tolist()) & set(inst["gt_sub_ids"][qi, :10].tolist()))
    print(f"oracle perfect-entry ef={ef}: GT_sub recall {hits / (10 * len(sel)):.4f}", flush=True)
# oracle with FES entries at large ef
for ef in (256, 1024):
    r = orc.search(inst, queries=inst["queries"][sel], k=10, ef=ef, stages=1)
    print(f"oracle FES ef={ef}: GT_sub recall {rec(r['ids'], inst['gt_sub_ids'][sel]):.4f}", flush=True)
