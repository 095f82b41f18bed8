"""Run the product's GPU stage through the C ABI (pa_search_device) with debug/trace outputs."""
import numpy as np

import paper_2503_21206_b200 as pa


def run_gpu(ix, inst, k, ef, trace_cap=0, queries=None, **opts):
    import torch
    q = inst["queries"] if queries is None else queries
    m = q.shape[0]
    qd = torch.from_numpy(np.ascontiguousarray(q, np.float32)).cuda()
    ids = torch.full((m, k), -7, dtype=torch.int32, device="cuda")
    d = torch.full((m, k), -7.0, dtype=torch.float32, device="cuda")
    o = pa.make_opts(**opts)
    ef1 = o.ef1 or ef
    E = o.entries or ef1
    dbg, t = pa.debug_buffers(m, ef1, E, trace_cap=trace_cap)
    ix.search_device(qd, k, ef, ids, d, opts=o, debug=dbg)
    torch.cuda.synchronize()
    out = {name: v.cpu().numpy() for name, v in t.items()}
    out["ids"], out["d"] = ids.cpu().numpy(), d.cpu().numpy()
    out["n_exp1"], out["n_dist1"] = out["counters"][:, 0], out["counters"][:, 1]
    out["spill"], out["status"] = out["counters"][:, 2], out["counters"][:, 3]
    return out
