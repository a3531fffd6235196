"""A/B of scheduling environment knobs (read per launch by the library; results
are identical) on the prepared-image top-k, alternating rounds on one box.

usage: env_ab.py N_R N_Q L VAR=val[,VAR=val] ...      ('-' = no override)
"""
import os
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import pynvml
import torch

import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L = (int(x) for x in sys.argv[1:4])
variants = sys.argv[4:] or ["-"]
reps, rounds = int(os.environ.get("REPS", "10")), int(os.environ.get("ROUNDS", "3"))
pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(0)


class Sampler:
    def __enter__(self):
        self.clk, self.run = [], True

        def loop():
            while self.run:
                self.clk.append(pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM))
                threading.Event().wait(0.005)

        self.t = threading.Thread(target=loop)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.run = False
        self.t.join()


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
keys = {kv.split("=")[0] for v in variants if v != "-" for kv in v.split(",")}
ref = None
for rnd in range(rounds):
    for v in variants:
        for k in keys:
            os.environ.pop(k, None)
        if v != "-":
            for kv in v.split(","):
                k, val = kv.split("=")
                os.environ[k] = val
        s, x = db.topk_device(dq, 16, None, ws)
        torch.cuda.synchronize()
        if ref is None:
            ref = (s.clone(), x.clone())
        assert torch.equal(s, ref[0]) and torch.equal(x, ref[1]), v
        ts = []
        with Sampler() as smp:
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                db.topk_device(dq, 16, None, ws)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
        print(f"round {rnd} [{v}] {n_r}x{n_q}x{L}: median {np.median(ts):.3f} ms min {min(ts):.3f} "
              f"sm {np.median(smp.clk):.0f} MHz", flush=True)
