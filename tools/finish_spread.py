"""Per-CTA finish times of the C3 top-k comparison (debug flag 64), grouped by unknown group
and slice: where the finishing spread comes from."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1707_00516_b200 as m
from paper_1707_00516_b200 import _native
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L = 20_000_000, 2048, 1024
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, L // 64), dtype=torch.int64, device="cuda", generator=g)
q = r[torch.randint(0, n_r, (n_q,), device="cuda", generator=g)].clone()
db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation="tensor_f4")
del r
dq = m.DevicePanel.from_words(q, L)
lib = _native.diag_lib()
for _ in range(3):
    db.topk_device(dq, 16)
torch.cuda.synchronize()
buf = torch.zeros((148 * 4,), dtype=torch.int64, device="cuda")
runs = []
for rep in range(3):
    buf.zero_()
    lib.fastid_debug_flags(64)
    lib.fastid_debug_trace(buf.data_ptr(), 0)
    db.topk_device(dq, 16); torch.cuda.synchronize()
    lib.fastid_debug_trace(None, 0)
    lib.fastid_debug_flags(0)
    t = buf.cpu().numpy().reshape(148, 4)[:144]  # regular grid: blockIdx < 144
    t0 = t[:, 0].min()
    runs.append((t[:, 2] - t0) / 1e3)
d = np.mean(runs, axis=0)  # per regular CTA, us
pair = d.reshape(72, 2).max(1)
by = pair.reshape(8, 9)  # [group][slice]
np.set_printoptions(precision=0, suppress=True, linewidth=160)
print("finish (us) by group (rows) x slice (cols):\n", by)
print("group means:", by.mean(1).round(0), " slice means:", by.mean(0).round(0))
print(f"min {d.min():.0f} median {np.median(d):.0f} max {d.max():.0f}; run-to-run corr of per-CTA times: "
      f"{np.corrcoef(runs[0], runs[1])[0,1]:.2f}")
