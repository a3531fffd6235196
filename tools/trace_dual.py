"""Per-stage timeline of the dual-tile CTA-pair MMA issuer (CTA 0, debug flag 8)
on a C4-shaped job: where the tensor pipe waits (accumulator, A stage, B stage).

usage: trace_dual.py [N_R] [N_Q] [L] [TILES]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1707_00516_b200 import _native

lib = _native.diag_lib()
import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L, tiles = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (20_000_000, 512, 5000, 1200)))
g = torch.Generator(device="cuda").manual_seed(0)
nw = -(-L // 64)
r = torch.randint(-(2**62), 2**62, (n_r, nw), dtype=torch.int64, device="cuda", generator=g)
q = torch.randint(-(2**62), 2**62, (n_q, nw), dtype=torch.int64, device="cuda", generator=g)
if L % 64:
    r[:, -1] &= ~((1 << (64 - L % 64)) - 1)
    q[:, -1] &= ~((1 << (64 - L % 64)) - 1)
db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation="tensor_f4")
del r
dq = m.DevicePanel.from_words(q, L)
db.topk_device(dq, 16)
torch.cuda.synchronize()
buf = torch.zeros((tiles, 67), dtype=torch.int64, device="cuda")
n_kst = (L + 255) // 256
ideal = 8 * 256 * 192 * 64 / (4.43e15 / 74) * 1.965e9  # cycles per dual stage at the probe rate
import os

# CONFIGS="sa:lag,...": A ring depth and lag per run (diag overrides FASTID_DUAL_SA / FASTID_DUAL_LAG)
runs = [(8, f"pair dual, A ring {c.split(':')[0]}, lag {c.split(':')[1]}", c)
        for c in os.environ.get("CONFIGS", "").split(",") if c] or [(8, "pair dual", None)]
for flags, name, cfg in runs:
    if cfg is not None:
        os.environ["FASTID_DUAL_SA"], os.environ["FASTID_DUAL_LAG"] = cfg.split(":")
    lib.fastid_debug_flags(flags)
    buf.zero_()
    lib.fastid_debug_trace(buf.data_ptr(), tiles)
    db.topk_device(dq, 16)
    torch.cuda.synchronize()
    lib.fastid_debug_trace(None, 0)
    torch.cuda.synchronize()
    ts = []
    lib.fastid_debug_flags(0)
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); db.topk_device(dq, 16); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"   {name}: untraced launch median {np.median(ts):.3f} ms")
    t = buf.cpu().numpy().astype(np.int64)
    t = t[200:][t[200:, 1] != 0]  # the MMA trace fills every second tile (the dual step's first)
    go, wait0 = t[:, 1], t[:, 0]
    pre, post = t[:, 35:35 + min(n_kst, 16)], t[:, 51:51 + min(n_kst, 16)]
    per = np.diff(go)
    print(f"== {name}: median dual-step period {np.median(per):.0f} cyc (ideal {ideal * n_kst:.0f}); "
          f"accumulator wait {np.median(go - wait0):.0f}")
    print("   A wait + prev issue (pre[k]-post[k-1]):", np.median(pre[:, 1:] - post[:, :-1], axis=0).astype(int).tolist())
    print("   B wait (post[k]-pre[k]):             ", np.median(post - pre, axis=0).astype(int).tolist())
    print(f"   stage-to-stage median {np.median(np.diff(post, axis=1)):.0f} cyc (ideal {ideal:.0f})")
lib.fastid_debug_flags(0)
