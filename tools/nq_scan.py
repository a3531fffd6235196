"""Fused top-16 time of the prepared mxf4 image against 20M x 1024-locus knowns
as the number of unknowns grows, next to the two bounds (the image read at the
measured HBM copy rate, the MMA work at the probe rate): anomalies show up as
points far above both.

usage: nq_scan.py [N_R] [L] [NQ,...]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

n_r = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
L = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
nqs = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 128, 256, 384, 512, 768, 1024, 1536,
                                                                             2048, 3072, 4096, 8192]
g = torch.Generator(device="cuda").manual_seed(0)
nw = -(-L // 64)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, nw), dtype=torch.int64, device="cuda", generator=g)
db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation="tensor_f4")
image_gb = n_r * (-(-L // 256) * 256) / 2 / 1e9
for n_q in nqs:
    q = r[torch.randint(0, n_r, (n_q,), device="cuda", generator=g)].clone()
    dq = m.DevicePanel.from_words(q, L)
    ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, 16, "tensor_f4"), dtype=torch.uint8, device="cuda")
    db.topk_device(dq, 16, None, ws)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        db.topk_device(dq, 16, None, ws)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = float(np.median(ts))
    hbm = image_gb / 6.5e3 * 1e3  # ms at 6.5 TB/s
    mma = n_r * n_q * L / 4.43e15 * 1e3
    print(f"N_Q {n_q:5d}: {t:8.3f} ms   bounds: image {hbm:.2f} ms, MMA {mma:.2f} ms -> {t / max(hbm, mma):.2f}x",
          flush=True)
