"""Few unknowns against a large database: fused top-k time per formulation
as the batch shrinks (the tensor image path streams the whole 4-bit image
whatever the batch; the CUDA-core path reads packed rows).

usage: small_batch.py [N_R] [L]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

n_r, L = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (20_000_000, 1024)))
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, -(-L // 64)), dtype=torch.int64, device="cuda", generator=g)
if L % 64:
    r[:, -1] &= ~((1 << (64 - L % 64)) - 1)
panel = m.DevicePanel.from_words(r, L)
dbs = {f: KnownDatabase(panel, formulation=f) for f in ("tensor_f4", "popc")}
for n_q in (1, 2, 4, 8, 16, 32, 64, 256):
    q = r[torch.randint(0, n_r, (n_q,), device="cuda", generator=g)].clone()
    dq = m.DevicePanel.from_words(q, L)
    line = []
    res = {}
    for f, db in dbs.items():
        ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, 16, f), dtype=torch.uint8, device="cuda")
        s, x = db.topk_device(dq, 16, None, ws)
        res[f] = (s.clone(), x.clone())
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            db.topk_device(dq, 16, None, ws)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        line.append(f"{f} {np.median(ts):8.3f} ms")
    same = all(torch.equal(res["popc"][i], res["tensor_f4"][i]) for i in range(2))
    print(f"N_Q {n_q:4d}: " + "  ".join(line) + f"  same={same}", flush=True)
