"""Diagnostic: kNN-candidate accuracy of the graph tool at full C1 scale (GPU)."""
import sys, time, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen as dg

cfg = dg.get_config("C1")
dev = "cuda"
X, labels = dg.gen_base(cfg, dev)
rng = np.random.default_rng(0)
sample = torch.from_numpy(np.sort(rng.choice(cfg.N, 1000, replace=False))).to(dev)
d = dg._sqdist(X[sample], X)
d[torch.arange(1000, device=dev), sample] = float("inf")
true64 = torch.topk(d, 64, dim=1, largest=False).indices.cpu().numpy()
del d
lab = dg.partition_labels(X, cfg.N // 1000, cfg.seeds["graph"])
for P in [int(p) for p in os.environ.get("PS", "32 64").split()]:
    t = time.time()
    rows = dg.knn_graph(X, 64, labels=lab, P=P)
    torch.cuda.synchronize()
    tt = time.time() - t
    r = rows[sample].cpu().numpy()
    acc10 = np.mean([len(set(r[i, :10]) & set(true64[i, :10])) / 10 for i in range(1000)])
    acc64 = np.mean([len(set(r[i]) & set(true64[i])) / 64 for i in range(1000)])
    print(f"P={P}: {tt:.1f}s  10-NN acc {acc10:.3f}  64-NN acc {acc64:.3f}", flush=True)
    if os.environ.get("REFINE"):
        t = time.time()
        rr = dg.refine_knn(X, rows, torch.arange(cfg.N, device=dev), iters=1)
        torch.cuda.synchronize()
        r = rr[sample].cpu().numpy()
        acc10 = np.mean([len(set(r[i, :10]) & set(true64[i, :10])) / 10 for i in range(1000)])
        acc64 = np.mean([len(set(r[i]) & set(true64[i])) / 64 for i in range(1000)])
        print(f"  +refine1: {time.time() - t:.1f}s  10-NN acc {acc10:.3f}  64-NN acc {acc64:.3f}", flush=True)
