"""One-unknown (and few-unknown) CUDA-core scan over a large packed panel:
time per grid size (FASTID_SCAN_CTAS) against a plain read of the same bytes
(torch int64 sum) -- is the scan HBM-, latency- or issue-bound?

usage: scan_timing.py [N_R] [L]
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1707_00516_b200 as m

n_r, L = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (20_000_000, 1024)))
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, -(-L // 64)), dtype=torch.int64, device="cuda", generator=g)
if L % 64:
    r[:, -1] &= ~((1 << (64 - L % 64)) - 1)
panel = m.DevicePanel.from_words(r, L)
nbytes = panel.rows.numel() * panel.rows.element_size()


def timed(fn, reps=20):
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


flat = panel.rows.view(torch.int64).view(-1)
t = timed(lambda: flat.sum())
print(f"torch int64 sum of {nbytes / 1e9:.2f} GB: {t:.3f} ms = {nbytes / t / 1e6:.0f} GB/s", flush=True)
ws = torch.empty(m.compare.topk_workspace_bytes(n_r, 16, 16, "auto"), dtype=torch.uint8, device="cuda")
for n_q in (1, 4):
    q = m.DevicePanel.from_words(r[:n_q].clone(), L)
    ref = None
    for ctas in ("", "148", "296", "444", "592"):
        os.environ["FASTID_SCAN_CTAS"] = ctas
        t = timed(lambda: m.topk_device(panel, q, 16, formulation="popc", workspace=ws))
        s, x = m.topk_device(panel, q, 16, formulation="popc", workspace=ws)
        cur = (s.cpu(), x.cpu())
        same = ref is None or all(torch.equal(a, b) for a, b in zip(ref, cur))
        ref = ref or cur
        print(f"n_q {n_q} ctas {ctas or 'default':>7}: {t:.3f} ms = {nbytes / t / 1e6:.0f} GB/s same={same}",
              flush=True)
os.environ.pop("FASTID_SCAN_CTAS", None)
# the same scan with (almost) no list insertions: max_score 0 admits only exact copies
for n_q in (1, 4):
    q = m.DevicePanel.from_words(r[:n_q].clone(), L)
    for ctas in ("", "296"):
        os.environ["FASTID_SCAN_CTAS"] = ctas
        t = timed(lambda: m.topk_device(panel, q, 16, max_score=0, formulation="popc", workspace=ws))
        print(f"n_q {n_q} ctas {ctas or 'default':>7} max_score 0: {t:.3f} ms = {nbytes / t / 1e6:.0f} GB/s",
              flush=True)
    os.environ.pop("FASTID_SCAN_CTAS", None)
    t = timed(lambda: m.threshold_hits(panel, q, 0, formulation="popc"))
    print(f"n_q {n_q} threshold 0 (host call): {t:.3f} ms", flush=True)
