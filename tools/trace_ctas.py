"""Per-CTA start/finish times of the top-k tensor kernel (debug flag 64, %globaltimer ns).

usage: trace_ctas.py [N_R] [N_Q] [L]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1707_00516_b200 as m
from paper_1707_00516_b200 import _native
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (20_000_000, 2048, 1024)))
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-2**62, 2**62, (n_r, L // 64), dtype=torch.int64, device="cuda", generator=g)
q = torch.randint(-2**62, 2**62, (n_q, L // 64), dtype=torch.int64, device="cuda", generator=g)
db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation="tensor_f4")
del r
dq = m.DevicePanel.from_words(q, L)
lib = _native.diag_lib()
db.topk_device(dq, 16); torch.cuda.synchronize()
buf = torch.zeros((148 * 4,), dtype=torch.int64, device="cuda")
lib.fastid_debug_flags(64)
lib.fastid_debug_trace(buf.data_ptr(), 0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); db.topk_device(dq, 16); e1.record(); e1.synchronize()
lib.fastid_debug_trace(None, 0)
lib.fastid_debug_flags(0)
t = buf.cpu().numpy().reshape(148, 4)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t - t0) / 1e3  # us
print(f"CTAs: {len(t)}; event time {e0.elapsed_time(e1)*1e3:.0f} us")
print(f"entry spread {rel[:, 0].max():.1f} us; setup (entry->roles) median {np.median(rel[:, 1] - rel[:, 0]):.1f} us")
print(f"roles done: min {rel[:, 2].min():.0f} median {np.median(rel[:, 2]):.0f} max {rel[:, 2].max():.0f} us")
print(f"exit: min {rel[:, 3].min():.0f} median {np.median(rel[:, 3]):.0f} max {rel[:, 3].max():.0f} us")
print("slowest CTAs (roles done us):", np.sort(rel[:, 2])[-8:].round(0).tolist())
print("fastest CTAs (roles done us):", np.sort(rel[:, 2])[:8].round(0).tolist())
import time
ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, 16, "tensor_f4"), dtype=torch.uint8, device="cuda")
out = (torch.empty((n_q, 16), dtype=torch.int32, device="cuda"), torch.empty((n_q, 16), dtype=torch.int64, device="cuda"))
torch.cuda.synchronize()
for trial in range(3):
    h0 = time.perf_counter()
    e0.record()
    db.topk_device(dq, 16, None, ws, out)
    h1 = time.perf_counter()
    e1.record(); e1.synchronize()
    print(f"host enqueue {1e6*(h1-h0):.0f} us; device event span {e0.elapsed_time(e1)*1e3:.0f} us")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(5):
    db.topk_device(dq, 16, None, ws, out)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
