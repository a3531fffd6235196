"""Configuration A/B timed by ncu (gpu__time_duration per launch, kernels
serialised with idle gaps, so the board's power limiter does not engage and
variants compare at the same clock).  Each variant (environment knobs read per
launch by the library; results identical) runs WARM untimed launches and REPS
timed launches of the prepared-image top-k; run under

    ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tensor_kernel \\
        --csv --log-file out.csv python tools/ncu_ab.py N_R N_Q L VAR=v[,VAR=v] ...

then `python tools/ncu_ab.py --parse out.csv N_R N_Q L VARIANTS...` prints the
median duration per variant (regular grid; a spare grid is listed apart).
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
WARM, REPS = 2, 5


def variants_env(variants):
    keys = {kv.split("=")[0] for v in variants if v != "-" for kv in v.split(",")}
    for v in variants:
        env = {k: None for k in keys}
        if v != "-":
            env.update(dict(kv.split("=") for kv in v.split(",")))
        yield v, env


if sys.argv[1] == "--parse":
    import csv
    import statistics

    rows = [r for r in csv.reader(open(sys.argv[2])) if r]
    hdr = next(r for r in rows if r[0] == "ID")
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    regular = [float(r[iv].replace(",", "")) for r in rows[rows.index(hdr) + 1:]
               if len(r) == len(hdr) and "tensor_kernel" in r[ik] and r[ik].rstrip(")").split(",")[6].strip() != "1"
               and ", 1>" not in r[ik]]
    variants = sys.argv[6:]
    per = WARM + REPS
    for n, v in enumerate(variants):
        ts = regular[n * per + WARM:(n + 1) * per]
        print(f"[{v}] {sys.argv[3]}x{sys.argv[4]}x{sys.argv[5]}: median {statistics.median(ts) / 1e3:.3f} ms "
              f"min {min(ts) / 1e3:.3f} ({len(ts)} launches)")
    sys.exit(0)

import torch

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
ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, 16, "tensor_f4"), dtype=torch.uint8, device="cuda")
for v, env in variants_env(sys.argv[4:] or ["-"]):
    for k, val in env.items():
        if val is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = val
    for _ in range(WARM + REPS):
        db.topk_device(dq, 16, None, ws)
    torch.cuda.synchronize()
