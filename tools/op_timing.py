"""Fused top-k (and full-matrix) time per operator on one database shape:
AND-NOT (Eq. 1), AND and XOR through the prepared image, plus the
CUDA-core scan for one unknown.  XOR adds the row-popcount pass (per
query batch) and an epilogue transform; AND-NOT / AND differ only in the
unknown-side complement.

usage: op_timing.py [N_R] [N_Q] [L]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (20_000_000, 2048, 1024)))
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, -(-L // 64)), dtype=torch.int64, device="cuda", generator=g)
if L % 64:
    r[:, -1] &= ~((1 << (64 - L % 64)) - 1)
panel = m.DevicePanel.from_words(r, L)
q = r[torch.randint(0, n_r, (n_q,), device="cuda", generator=g)].clone()
dq = m.DevicePanel.from_words(q, L)
dq1 = m.DevicePanel.from_words(q[:1].clone(), L)


def timed(fn, reps=10):
    fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for op in ("andnot", "and", "xor"):
    db = KnownDatabase(panel, op=op)
    ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, 16, "auto"), dtype=torch.uint8, device="cuda")
    t_img = timed(lambda: db.topk_device(dq, 16, None, ws))
    ws1 = torch.empty(m.compare.topk_workspace_bytes(n_r, 1, 16, "auto"), dtype=torch.uint8, device="cuda")
    t_one = timed(lambda: db.topk_device(dq1, 16, None, ws1))
    print(f"{n_r}x{n_q}x{L} op={op:6s}: top-16 {t_img:8.3f} ms ({n_r * n_q / t_img / 1e9:.3f}e12 cmp/s)"
          f"   one unknown (scan) {t_one:6.3f} ms", flush=True)
    del db
    torch.cuda.empty_cache()
