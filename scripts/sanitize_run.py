"""Small searches through every kernel path (C0, 64 queries) for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): tcgen05 projection + FES, the
pipelined traversal with the bloom and the exact (forced-spill) visited sets,
binary16 rows, the v1 traversal, the SIMT fallbacks and stages 2-3 on the GPU."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen as dg  # noqa: E402
import paper_2503_21206_b200 as pa  # noqa: E402

cfg = dg.get_config("C0", m=64)
inst = dg.build_instance(cfg, device="cpu", gt=False)
for fp16 in (False, True):
    ix = pa.Index.from_instance(inst, reduced_fp16=fp16)
    ix.attach_host(inst["full_offsets"], inst["full_neighbors"], inst["rotated"])
    for kw in (dict(bloom_log2=12), dict(), dict(hash_slots_log2=5), dict(ef=256, entries=1024)):
        ef = kw.pop("ef", cfg.ef)
        ix.search(inst["queries"], k=cfg.k, ef=ef, **kw)
    ix.search(inst["queries"], k=cfg.k, ef=cfg.ef, stages=pa.PA_STAGES_FULL_GPU, bloom_log2=12)
    ix.search(inst["queries"], k=cfg.k, ef=cfg.ef, stages=pa.PA_STAGES_FULL)
    ix.close()
os.environ["PA_TRAVERSE"] = "v1"
os.environ["PA_PROJECT"] = "simt"
os.environ["PA_FES"] = "simt"
ix = pa.Index.from_instance(inst)
ix.search(inst["queries"], k=cfg.k, ef=cfg.ef)
ix.close()
print("sanitize run done")
