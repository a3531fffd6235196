"""A/B: CTA-pair top-k with debug flags 0 vs FLAG (see common.cuh for the flag bits), alternating
rounds, plus per-CTA finish times (debug flag 64) for each.  usage: spare_ab.py [FLAG] (default 16: no top-k insertions)"""
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
ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, 16, "tensor_f4"), dtype=torch.uint8, device="cuda")
lib = _native.diag_lib()
FLAG = int(sys.argv[1]) if len(sys.argv) > 1 else 16
res = {0: [], FLAG: []}
for rd in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    for flags in (0, FLAG):
        lib.fastid_debug_flags(flags)
        db.topk_device(dq, 16, None, ws)
        evs = []
        for _ in range(8):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            db.topk_device(dq, 16, None, ws, events=(e0, e1))
            evs.append((e0, e1))
        torch.cuda.synchronize()
        res[flags].append(np.median([a.elapsed_time(b) for a, b in evs]))
for flags, v in res.items():
    print(f"flags {flags:5d}: {[round(x, 3) for x in v]} mean {np.mean(v):.3f} ms")
buf = torch.zeros((148 * 4,), dtype=torch.int64, device="cuda")
for flags in (0, FLAG):
    buf.zero_()
    lib.fastid_debug_flags(64 | flags)
    lib.fastid_debug_trace(buf.data_ptr(), 0)
    db.topk_device(dq, 16, None, ws); torch.cuda.synchronize()
    lib.fastid_debug_trace(None, 0)
    t = buf.cpu().numpy().reshape(148, 4)
    live = t[:, 0] > 0
    rel = (t[live] - t[live, 0].min()) / 1e3
    done = rel[:, 2]
    print(f"flags {flags}: CTAs {live.sum()}, done min {done.min():.0f} med {np.median(done):.0f} max {done.max():.0f} us; "
          f"last 4 CTAs (blockIdx): {np.argsort(t[:, 2])[-4:].tolist()}")
lib.fastid_debug_flags(0)
