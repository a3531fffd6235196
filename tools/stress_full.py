"""Repeat the tensor full-matrix compare and diff against the popc kernel (race hunt)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1707_00516_b200 as m

n_r, n_q, L, reps = (int(x) for x in sys.argv[2:6])
g = torch.Generator(device="cuda").manual_seed(1)
rw = torch.randint(-2**62, 2**62, (n_r, L // 64), dtype=torch.int64, device="cuda", generator=g)
qw = torch.randint(-2**62, 2**62, (n_q, L // 64), dtype=torch.int64, device="cuda", generator=g)
dr = m.DevicePanel.from_words(rw, L); dq = m.DevicePanel.from_words(qw, L)
ref = m.compare_device(dr, dq, formulation="popc").clone()
for form in sys.argv[1].split(","):
    bad_runs = 0
    for i in range(reps):
        out = torch.full((n_r, n_q), -7, dtype=torch.int32, device="cuda")
        m.compare_device(dr, dq, out, formulation=form)
        diff = (out != ref)
        nb = int(diff.sum())
        if nb:
            bad_runs += 1
            idx = torch.nonzero(diff)[:8].tolist()
            rows = torch.nonzero(diff.any(1)).flatten()
            cols = torch.nonzero(diff.any(0)).flatten()
            print(f"{form} run {i}: {nb} bad cells; rows {rows.numel()} [{int(rows.min())}..{int(rows.max())}], "
                  f"cols {cols.numel()} [{int(cols.min())}..{int(cols.max())}] first {idx}; "
                  f"vals {[int(out[a,b]) for a,b in idx[:4]]} exp {[int(ref[a,b]) for a,b in idx[:4]]}", flush=True)
    print(f"{form}: {bad_runs}/{reps} runs with mismatches", flush=True)
