"""A/B of the host-buffer search loops on one box, alternating rounds: device-
resident steps (topk_device back to back), synchronous search_words per step,
and the pipelined search_many; SM clock / board power sampled in each.

usage: e2e_ab.py [N_R] [N_Q] [L] [STEPS] [ROUNDS]
"""
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import pynvml
import torch

import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L, steps, rounds = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (20_000_000, 2048, 1024, 20, 3)))
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


g = torch.Generator(device="cuda").manual_seed(0)
nw = L // 64
r = torch.randint(-(2**63), 2**63 - 1, (n_r, nw), dtype=torch.int64, device="cuda", generator=g)
qw = r[torch.randint(0, n_r, (n_q,), device="cuda", generator=g)].cpu().numpy().view(np.uint64)
db = KnownDatabase(m.DevicePanel.from_words(r, L))
del r
dq = m.DevicePanel.from_words(qw, L)
ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, 16, "auto"), dtype=torch.uint8, device="cuda")


def device_loop():
    for _ in range(steps):
        db.topk_device(dq, 16, None, ws)
    torch.cuda.synchronize()


def sync_loop():
    for _ in range(steps):
        db.search_words(qw, 16)


def pipe_loop():
    for _ in db.search_many((qw for _ in range(steps)), 16):
        pass


for fn in (device_loop, sync_loop, pipe_loop):
    fn()
for rnd in range(rounds):
    for name, fn in (("device", device_loop), ("sync", sync_loop), ("pipelined", pipe_loop)):
        torch.cuda.synchronize()
        with Sampler() as smp:
            t0 = time.perf_counter()
            fn()
            t = (time.perf_counter() - t0) / steps
        print(f"round {rnd} {name:9s}: {t * 1e3:7.3f} ms/step  sm {np.median(smp.clk):.0f} MHz "
              f"(min {min(smp.clk)}) power {np.median(smp.pw):.0f} W", flush=True)
