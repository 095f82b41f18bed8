"""Diagnostic: build a large instance with datagen/large.py on the GPU, then measure
the product's GPU-stage Recall@10 (GT_sub) and the all-GPU three-stage recall
(full-space GT) over an ef sweep — is the graph good enough, and how fast is the tool?"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen as dg
from datagen import large as lg
import paper_2503_21206_b200 as pa
import __graft_entry__ as ge

name = sys.argv[1] if len(sys.argv) > 1 else "C2S"
cfg = dg.get_config(name)
ge.build_library()
t = time.time()
inst = lg.build_instance_large(cfg, device="cuda", cache=os.environ.get("PA_CACHE"))
print(f"instance {time.time() - t:.1f}s", flush=True)
X = inst["rotated"]
t = time.time()
ix = pa.Index.from_instance(inst)
ix.attach_host(inst["full_offsets"], inst["full_neighbors"], inst["rotated"])
print(f"pa_build {time.time() - t:.1f}s", flush=True)
q = torch.from_numpy(inst["queries"]).cuda()
m = q.shape[0]
oi = torch.empty(m, 10, dtype=torch.int32, device="cuda")
od = torch.empty(m, 10, dtype=torch.float32, device="cuda")


def rec(ids, gt):
    ids = ids[:, :10]; gt = gt[:, :10]
    return sum(len(set(a) & set(b)) for a, b in zip(ids.tolist(), gt.tolist())) / (10 * len(ids))


for ef in (32, 64, 96, 128, 192, 256):
    ix.search_device(q, 10, ef, oi, od, bloom_log2=12)
    torch.cuda.synchronize()
    st = ix.stats()
    print(f"ef={ef} GT_sub recall {rec(oi.cpu().numpy(), inst['gt_sub_ids']):.4f} "
          f"full-GT {rec(oi.cpu().numpy(), inst['gt_ids']):.4f} gpu {st['ms_total_gpu']:.3f} ms "
          f"trav {st['ms_traverse']:.3f} n_dist/q {st['sum_n_dist'] / m:.0f}", flush=True)
t = time.time()
for ef in (32, 64, 96, 128, 192):
    ix.search_device(q, 10, ef, oi, od, bloom_log2=12, stages=pa.PA_STAGES_FULL_GPU)
    torch.cuda.synchronize()
    st = ix.stats()
    print(f"FULL_GPU ef={ef} full-GT recall {rec(oi.cpu().numpy(), inst['gt_ids']):.4f} gpu {st['ms_total_gpu']:.3f} ms "
          f"(first call incl. X-hat upload {time.time() - t:.1f}s)", flush=True)
for ef in (64, 128, 256):
    t = time.time()
    ids, _ = ix.search(inst["queries"], k=10, ef=ef, stages=pa.PA_STAGES_FULL, bloom_log2=12)
    print(f"FULL host ef={ef} full-GT recall {rec(ids, inst['gt_ids']):.4f} {m / (time.time() - t):.0f} q/s", flush=True)
