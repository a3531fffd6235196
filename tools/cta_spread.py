"""Per-CTA start / finish times of one prepared-image top-k launch (diag build,
debug flag 64: %globaltimer at entry, roles start, roles done, exit) for any
shape: is a slow launch every CTA being slow, or a few CTAs finishing late?

usage: cta_spread.py N_R N_Q L
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

n_r, n_q, L = (int(x) for x in sys.argv[1:4])
g = torch.Generator(device="cuda").manual_seed(0)
nw = -(-L // 64)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, nw), dtype=torch.int64, device="cuda", generator=g)
if L % 64:
    r[:, -1] &= ~((1 << (64 - L % 64)) - 1)
q = r[torch.randint(0, n_r, (n_q,), device="cuda", generator=g)].clone()
db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation="tensor_f4")
del r
dq = m.DevicePanel.from_words(q, L)
for _ in range(3):
    db.topk_device(dq, 16)
torch.cuda.synchronize()
n_cta = 2 * (_native.lib() and 74)
buf = torch.zeros((160 * 4,), dtype=torch.int64, device="cuda")
lib.fastid_debug_flags(64)
lib.fastid_debug_trace(buf.data_ptr(), 0)
db.topk_device(dq, 16)
torch.cuda.synchronize()
lib.fastid_debug_trace(None, 0)
lib.fastid_debug_flags(0)
t = buf.cpu().numpy().reshape(160, 4)
t = t[t[:, 0] != 0]
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
np.set_printoptions(precision=0, suppress=True, linewidth=200)
print(f"{n_r}x{n_q}x{L}: {len(t)} CTAs; entry max {rel[:, 0].max():.0f} us; roles start median "
      f"{np.median(rel[:, 1]):.0f}; roles done min {rel[:, 2].min():.0f} median {np.median(rel[:, 2]):.0f} "
      f"max {rel[:, 2].max():.0f} us")
print("roles done per CTA (us):", np.sort(rel[:, 2]))
