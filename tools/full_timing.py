"""Device timing of the full-matrix (u32 N_R x N_Q) comparison through the prepared database.

usage: full_timing.py [N_R] [N_Q] [L] [REPS]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1707_00516_b200 as m
from paper_1707_00516_b200 import _native
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1_000_000, 2048, 1024)))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
g = torch.Generator(device="cuda").manual_seed(0)
nw = L // 64
rw = torch.randint(-2**62, 2**62, (n_r, nw), dtype=torch.int64, device="cuda", generator=g)
qw = torch.randint(-2**62, 2**62, (n_q, nw), dtype=torch.int64, device="cuda", generator=g)
lib = _native.diag_lib()
import os
lib.fastid_debug_flags(int(os.environ.get("FASTID_FLAGS", "0")))
for form in (os.environ.get("FASTID_FORMS", "tensor_f4,tensor_i8")).split(","):
    db = KnownDatabase(m.DevicePanel.from_words(rw, L), formulation=form)
    dq = m.DevicePanel.from_words(qw, L)
    out = torch.empty((n_r, n_q), dtype=torch.int32, device="cuda")
    db.full_device(dq, out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); db.full_device(dq, out); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts) / 1e3
    print(f"{form} full {n_r}x{n_q}x{L}: {t*1e3:8.3f} ms  out {n_r*n_q*4/t/1e9:7.1f} GB/s  "
          f"{2*n_r*n_q*L/t/1e12:8.1f} TFLOP/s-equiv", flush=True)
    del db, out
    torch.cuda.empty_cache()
