"""A/B of the mxf4 image encodings (uniform 1.0 x 1.0 vs weighted 0.5/1/2 pairs): alternating
rounds of back-to-back top-16 launches on the same inputs, kernel time per round.

usage: encoding_ab.py [N_R] [ROUNDS] [STEPS]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1707_00516_b200 as m
from paper_1707_00516_b200 import _native
from paper_1707_00516_b200.search import KnownDatabase

n_r, rounds, steps = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (20_000_000, 4, 10)))
n_q, L = 2048, 1024
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, L // 64), dtype=torch.int64, device="cuda", generator=g)
src = torch.randint(0, n_r, (n_q,), device="cuda", generator=g)
q = r[src].clone()
lib = _native.diag_lib()
dq = m.DevicePanel.from_words(q, L)
panel = m.DevicePanel.from_words(r, L)
del r
dbs = {}
for name, flags in (("uniform", 0), ("weighted", 512)):
    lib.fastid_debug_flags(flags)
    dbs[name] = (KnownDatabase(panel, formulation="tensor_f4"), flags)
ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, 16, "tensor_f4"), dtype=torch.uint8, device="cuda")
res = {k: [] for k in dbs}
ref = None
for rd in range(rounds):
    for name, (db, flags) in dbs.items():
        lib.fastid_debug_flags(flags)
        s, x = db.topk_device(dq, 16, None, ws)
        torch.cuda.synchronize()
        got = (s.cpu(), x.cpu())
        if ref is None:
            ref = got
        assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1]), name
        evs = []
        for _ in range(steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            db.topk_device(dq, 16, None, ws, events=(e0, e1))
            evs.append((e0, e1))
        torch.cuda.synchronize()
        res[name].append(np.median([a.elapsed_time(b) for a, b in evs]))
lib.fastid_debug_flags(0)
for name, v in res.items():
    print(f"{name:9s} per-round median kernel ms: {[round(x, 3) for x in v]}  mean {np.mean(v):.3f}")
