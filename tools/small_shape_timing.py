"""Where the time of a small full-matrix call goes (C5 mixture-to-mixture
4096 x 4096): CUDA-event time of one call, host wall time per call (enqueue
cost), and the same call captured once in a CUDA graph and replayed.

usage: small_shape_timing.py [N_R] [N_Q] [L]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 1024)))
g = torch.Generator(device="cuda").manual_seed(0)
nw = -(-L // 64)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, nw), dtype=torch.int64, device="cuda", generator=g)
q = torch.randint(-(2**63), 2**63 - 1, (n_q, nw), dtype=torch.int64, device="cuda", generator=g)
if L % 64:
    r[:, -1] &= ~((1 << (64 - L % 64)) - 1)
    q[:, -1] &= ~((1 << (64 - L % 64)) - 1)
db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation="tensor_f4")
dq = m.DevicePanel.from_words(q, L)
out = torch.empty((n_r, n_q), dtype=torch.int32, device="cuda")
ref = None


def ev(fn, reps=20):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return np.median(ts), min(ts)


def call():
    db.full_device(dq, out)


call()
torch.cuda.synchronize()
ref = out.clone()
med, mn = ev(call)
print(f"{n_r}x{n_q}x{L} full: one call, event time median {med:.1f} us min {mn:.1f} us")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    call()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"  200 back-to-back calls: host enqueue {1e6 * (t1 - t0) / 200:.1f} us/call, "
      f"wall {1e6 * (t2 - t0) / 200:.1f} us/call")
# the same call in a CUDA graph
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    call()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
try:
    out.zero_()
    # capture on the stream the warm-up ran on: the library keeps its launch
    # scratch per stream, and a first use inside the capture would have to allocate
    with torch.cuda.graph(graph, stream=s):
        call()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref), "graph replay result differs"
    med, mn = ev(graph.replay)
    print(f"  CUDA graph replay: event time median {med:.1f} us min {mn:.1f} us (result identical)")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        graph.replay()
    torch.cuda.synchronize()
    print(f"  200 graph replays: wall {1e6 * (time.perf_counter() - t0) / 200:.1f} us/replay")
except Exception as e:  # report, do not hide
    print(f"  CUDA graph capture failed: {type(e).__name__}: {e}")
