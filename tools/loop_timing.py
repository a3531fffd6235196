"""Per-launch kernel times of the top-k path: back-to-back launches vs a sync after each.

usage: loop_timing.py [N_R] [N_Q] [L] [STEPS]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L, steps = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (20_000_000, 2048, 1024, 20)))
g = torch.Generator(device="cuda").manual_seed(0)
full = len(sys.argv) > 6 and sys.argv[6] == "full64"  # all 64 bits uniform (bench.py's generator)
lo, hi = (-(2**63), 2**63 - 1) if full else (-2**62, 2**62)
r = torch.randint(lo, hi, (n_r, L // 64), dtype=torch.int64, device="cuda", generator=g)
q = torch.randint(lo, hi, (n_q, L // 64), dtype=torch.int64, device="cuda", generator=g)
if len(sys.argv) > 5 and sys.argv[5] == "planted":
    # unknowns = copies of random knowns with a few flipped bits (bench.py's workload)
    src = torch.randint(0, n_r, (n_q,), device="cuda", generator=g)
    q = r[src].clone()
    flip = torch.randint(0, L, (n_q, 8), device="cuda", generator=g)
    for j in range(8):
        w, b = flip[:, j] // 64, flip[:, j] % 64
        q[torch.arange(n_q, device="cuda"), w] ^= (1 << b)
db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation="tensor_f4")
del r
dq = m.DevicePanel.from_words(q, L)
ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, 16, "tensor_f4"), dtype=torch.uint8, device="cuda")
out = (torch.empty((n_q, 16), dtype=torch.int32, device="cuda"), torch.empty((n_q, 16), dtype=torch.int64, device="cuda"))
for _ in range(3):
    db.topk_device(dq, 16, None, ws, out)
torch.cuda.synchronize()
for mode in ("back-to-back", "sync-each", "back-to-back"):
    evs = []
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        db.topk_device(dq, 16, None, ws, out, events=(e0, e1))
        evs.append((e0, e1))
        if mode == "sync-each":
            torch.cuda.synchronize()
    t1.record()
    torch.cuda.synchronize()
    ks = np.array([a.elapsed_time(b) for a, b in evs])
    print(f"{mode:13s}: total {t0.elapsed_time(t1)/steps:.3f} ms/step; kernel min {ks.min():.3f} med {np.median(ks):.3f} "
          f"max {ks.max():.3f} ms", flush=True)
