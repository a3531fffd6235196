"""A/B of dual-tile CTA-pair ring configurations (FASTID_DUAL_SA /
FASTID_DUAL_LAG, read per launch), alternating rounds on one box, C4-shaped job, with the SM
clock and board power sampled during each measurement.

usage: CONFIGS=sa:lag,... dual_ab.py [N_R] [N_Q] [L] [ROUNDS] [REPS]
"""
import os
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import pynvml
import torch

import paper_1707_00516_b200 as m  # product build: the ring knobs are read per launch
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L, rounds, reps = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (20_000_000, 512, 5000, 3, 10)))
configs = [c for c in os.environ.get("CONFIGS", "0:-1").split(",") if c]
pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(0)


class Sampler:
    def __enter__(self):
        self.clk, self.pw, self.run = [], [], True

        def loop():
            while self.run:
                self.clk.append(pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM))
                self.pw.append(pynvml.nvmlDeviceGetPowerUsage(hdl) / 1e3)
                threading.Event().wait(0.005)

        self.t = threading.Thread(target=loop)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.run = False
        self.t.join()


import bench  # C4 generator

panel = bench.c4_shard_panel(m, 1707, 0, n_r, L, torch.device("cuda"))
dq = m.DevicePanel.from_words(bench.mixture_unknowns(panel, n_q, np.random.default_rng(1707)), L)
db = KnownDatabase(panel, formulation="tensor_f4")
ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, 16, "tensor_f4"), dtype=torch.uint8, device="cuda")
ref = None
for rnd in range(rounds):
    for c in configs:
        sa, lag = c.split(":")
        os.environ["FASTID_DUAL_SA"], os.environ["FASTID_DUAL_LAG"] = sa, lag
        s, x = db.topk_device(dq, 16, None, ws)
        torch.cuda.synchronize()
        if ref is None:
            ref = (s.clone(), x.clone())
        assert torch.equal(s, ref[0]) and torch.equal(x, ref[1]), c
        ts = []
        with Sampler() as smp:
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                db.topk_device(dq, 16, None, ws)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
        print(f"round {rnd} A ring {sa} lag {lag}: median {np.median(ts):.3f} ms min {min(ts):.3f} "
              f"sm {np.median(smp.clk):.0f} MHz power {np.median(smp.pw):.0f} W", flush=True)
