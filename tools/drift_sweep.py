"""C4-shaped drift-window sweep (diag build): 512 x 20M x 5000 top-16 on the
prepared mxf4 image, timed per FASTID_DRIFT_TILES value.
usage: drift_sweep.py [N_R] [N_Q] [L] [values...]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path.cwd()))
import numpy as np
import torch

from paper_1707_00516_b200 import _native

_native.diag_lib()
import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L = (int(x) for x in sys.argv[1:4])
vals = [int(v) for v in sys.argv[4:]] or [0, 2, 4, 6, 8, 12, 20, 40]
# FLAGS="0,4": alternate debug-flag values instead of drift values (drift stays auto)
flag_vals = [int(v) for v in os.environ["FLAGS"].split(",")] if "FLAGS" in os.environ else None
import threading
import pynvml
pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())


class Sampler:
    """SM clock (MHz) and board power (W) every 5 ms while active."""
    def __enter__(self):
        self.clk, self.pw, self.run = [], [], True
        def loop():
            while self.run:
                self.clk.append(pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM))
                self.pw.append(pynvml.nvmlDeviceGetPowerUsage(hdl) / 1e3)
                threading.Event().wait(0.005)
        self.t = threading.Thread(target=loop); self.t.start(); return self
    def __exit__(self, *a):
        self.run = False; self.t.join()
if os.environ.get("C4DATA", "1") == "1":
    # bench.py's C4 generator: per-locus presence p ~ U(0.1, 0.5), OR-mixtures of 2-5 knowns
    import bench
    panel = bench.c4_shard_panel(m, 1707, 0, n_r, L, torch.device("cuda"))
    dq = m.DevicePanel.from_words(bench.mixture_unknowns(panel, n_q, np.random.default_rng(1707)), L)
    db = KnownDatabase(panel, formulation="tensor_f4")
    del panel
else:
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
for rnd in range(int(os.environ.get('ROUNDS', '2'))):
    for v in (flag_vals if flag_vals is not None else vals):
        if flag_vals is not None:
            _native.lib().fastid_debug_flags(v)
        elif v:
            os.environ["FASTID_DRIFT_TILES"] = str(v)
        else:
            os.environ.pop("FASTID_DRIFT_TILES", None)
        for _ in range(2):
            db.topk_device(dq, 16, None, ws)
        ts = []
        with Sampler() as smp:
            for _ in range(int(os.environ.get("REPS", "10"))):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); db.topk_device(dq, 16, None, ws); e1.record(); e1.synchronize()
                ts.append(e0.elapsed_time(e1))
        what = f"flags={v}" if flag_vals is not None else f"drift={v or 'auto'}"
        print(f"round {rnd} {what}: {n_r}x{n_q}x{L} top-16 median {np.median(ts):.3f} ms min {min(ts):.3f} "
              f"sm {np.median(smp.clk):.0f} MHz power {np.median(smp.pw):.0f} W", flush=True)
