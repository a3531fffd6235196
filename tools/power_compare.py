"""Board power and SM clock while (a) the tcgen05 mxf4 probe and (b) the C3 top-k comparison run
back to back for ~3 s each (nvidia-smi at 20 ms): where the clock headroom goes."""
import ctypes, subprocess, sys, time, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1707_00516_b200 as m
from paper_1707_00516_b200 import _native
from paper_1707_00516_b200.search import KnownDatabase

L = _native.diag_lib()
n_r, n_q, Lc = 20_000_000, 2048, 1024
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, Lc // 64), dtype=torch.int64, device="cuda", generator=g)
q = r[torch.randint(0, n_r, (n_q,), device="cuda", generator=g)].clone()
db = KnownDatabase(m.DevicePanel.from_words(r, Lc), formulation="tensor_f4")
del r
dq = m.DevicePanel.from_words(q, Lc)
ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, 16, "tensor_f4"), dtype=torch.uint8, device="cuda")
scratch = torch.zeros(4096, dtype=torch.int32, device="cuda")
work = ctypes.c_double(0)
stream = torch.cuda.current_stream().cuda_stream


def sample(fn, seconds, label):
    log = f"/tmp/pw_{label}.csv"
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm,clocks_event_reasons.active",
                          "--format=csv,noheader,nounits", "-lms", "20"], stdout=open(log, "w"))
    time.sleep(0.5)
    t0 = time.time(); n = 0
    while time.time() - t0 < seconds:
        fn(); n += 1
        if n % 5 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    p.terminate(); p.wait()
    rows = [l.split(",") for l in open(log).read().splitlines() if l.count(",") >= 2]
    pw = np.array([float(x[0]) for x in rows]); clk = np.array([float(x[1]) for x in rows])
    busy = pw > 300
    print(f"{label:10s}: power median {np.median(pw[busy]):.0f} W (max {pw.max():.0f}), SM clock median "
          f"{np.median(clk[busy]):.0f} MHz, reasons {sorted(set(x[2].strip() for x in rows))}", flush=True)


sample(lambda: L.fastid_probe_peak(3, 20000, scratch.data_ptr(), ctypes.byref(work), stream), 3, "probe")
sample(lambda: db.topk_device(dq, 16, None, ws), 3, "c3-topk")
sample(lambda: L.fastid_probe_peak(3, 20000, scratch.data_ptr(), ctypes.byref(work), stream), 3, "probe")

for flags, label in ((4096, "c3-spin"), (0, "c3-sleep"), (4096, "c3-spin"), (0, "c3-sleep")):
    L.fastid_debug_flags(flags)
    sample(lambda: db.topk_device(dq, 16, None, ws), 3, label)
    evs = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        db.topk_device(dq, 16, None, ws, events=(e0, e1)); evs.append((e0, e1))
    torch.cuda.synchronize()
    print(f"   {label}: kernel median {np.median([a.elapsed_time(b) for a, b in evs]):.3f} ms", flush=True)
L.fastid_debug_flags(0)
