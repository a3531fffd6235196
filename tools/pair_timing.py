"""Device timing of the prepared-image top-k kernel: CTA pairs vs single CTA.

usage: pair_timing.py [N_R] [N_Q] [L] [REPS]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1707_00516_b200 as m
from paper_1707_00516_b200 import _native
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (20_000_000, 2048, 1024)))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
g = torch.Generator(device="cuda").manual_seed(0)
nw = L // 64
rw = torch.randint(-2**62, 2**62, (n_r, nw), dtype=torch.int64, device="cuda", generator=g)
qw = torch.randint(-2**62, 2**62, (n_q, nw), dtype=torch.int64, device="cuda", generator=g)
db = KnownDatabase(m.DevicePanel.from_words(rw, L), formulation="tensor_f4")
dq = m.DevicePanel.from_words(qw, L)
del rw
lib = _native.diag_lib()
for flags, name in ((0, "pair"), (2, "single"), (1, "pair-noepi"), (4, "pair-noload")):
    lib.fastid_debug_flags(flags)
    out = db.topk_device(dq, 16)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); db.topk_device(dq, 16); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts) / 1e3
    print(f"{name:6s} {n_r}x{n_q}x{L}: {t*1e3:8.3f} ms (median {sorted(ts)[len(ts)//2]:.3f})  "
          f"{2*n_r*n_q*L/t/1e12:8.1f} TFLOP/s-equiv", flush=True)
lib.fastid_debug_flags(0)
