"""A/B of prepared-database execution options on the product library, alternating
rounds on one box (device time, CUDA events, median of REPS) with SM clock and
board power sampled during each measurement.

usage: opt_ab.py MODE N_R N_Q L OPTSETS...
  MODE    full | topk
  OPTSETS comma-separated option names per variant ('-' = defaults), e.g.
          - no_spare_pairs no_tma_store,no_spare_pairs
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
from paper_1707_00516_b200.search import DB_OPTIONS, KnownDatabase

mode, n_r, n_q, L = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
variants = sys.argv[5:] or ["-"]
reps, rounds = int(os.environ.get("REPS", "10")), int(os.environ.get("ROUNDS", "3"))
pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())


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


g = torch.Generator(device="cuda").manual_seed(0)
nw = -(-L // 64)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, nw), dtype=torch.int64, device="cuda", generator=g)
if L % 64:
    r[:, -1] &= ~((1 << (64 - L % 64)) - 1)
q = r[torch.randint(0, n_r, (n_q,), device="cuda", generator=g)].clone()
db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation="tensor_f4")
del r
dq = m.DevicePanel.from_words(q, L)
if mode == "full":
    out = torch.empty((n_r, n_q), dtype=torch.int32, device="cuda")
    fn = lambda: db.full_device(dq, out)  # noqa: E731
else:
    ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, 16, "tensor_f4"), dtype=torch.uint8, device="cuda")
    fn = lambda: db.topk_device(dq, 16, None, ws)  # noqa: E731
for rnd in range(rounds):
    for v in variants:
        for name in DB_OPTIONS:
            db.set_option(name, False)
        if v != "-":
            for name in v.split(","):
                db.set_option(name, True)
        fn()
        torch.cuda.synchronize()
        ts = []
        with Sampler() as smp:
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
        extra = f" out {n_r * n_q * 4 / np.median(ts) / 1e6:.0f} GB/s" if mode == "full" else ""
        print(f"round {rnd} [{v}] {mode} {n_r}x{n_q}x{L}: median {np.median(ts):.3f} ms min {min(ts):.3f}{extra} "
              f"sm {np.median(smp.clk):.0f} MHz power {np.median(smp.pw):.0f} W", flush=True)
        if os.environ.get("ALL"):
            print("   ", " ".join(f"{t:.3f}" for t in ts), flush=True)
