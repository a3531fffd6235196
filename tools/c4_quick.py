"""Quick C4-shaped timing (512 x N x 5000 top-16, tensor_f4 prepared image) for A/B between builds.
usage: c4_quick.py [N_R] [N_Q] [L]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path.cwd()))
import numpy as np, torch
import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase
n_r, n_q, L = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (5_000_000, 512, 5000)))
import os
from paper_1707_00516_b200 import _native
_native.diag_lib().fastid_debug_flags(int(os.environ.get("FASTID_FLAGS", "0")))
g = torch.Generator(device="cuda").manual_seed(0)
nw = -(-L // 64)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, nw), dtype=torch.int64, device="cuda", generator=g)
tail = L % 64
if tail:
    r[:, -1] &= ~((1 << (64 - tail)) - 1)
q = r[torch.randint(0, n_r, (n_q,), device="cuda", generator=g)].clone()
db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation="tensor_f4")
dq = m.DevicePanel.from_words(q, L)
ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, 16, "tensor_f4"), dtype=torch.uint8, device="cuda")
for _ in range(2):
    db.topk_device(dq, 16, None, ws)
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); db.topk_device(dq, 16, None, ws); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{Path.cwd().name} flags={os.environ.get('FASTID_FLAGS', '0')}: {n_r}x{n_q}x{L} top-16 median {np.median(ts):.3f} ms", flush=True)
