"""End-to-end full-matrix timing through the host-buffer drop-in (run_b200_kernel = fastid_run_kernel):
numpy knowns/unknowns in, numpy u32 (N_R, N_Q) out -- the reference's run_naive_kernel call shape.

usage: host_full_timing.py [N_R] [N_Q] [L] [REPS]
"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import numpy as np
import oracle
import paper_1707_00516_b200 as m

n_r, n_q, L = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1_000_000, 2048, 1024)))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
rng = np.random.default_rng(5)
r = rng.integers(0, 2**64, (n_r, L // 64), dtype=np.uint64)
q = rng.integers(0, 2**64, (n_q, L // 64), dtype=np.uint64)
out = np.empty((n_r, n_q), np.uint32)
out.fill(0)  # first touch outside the timed region
m.run_b200_kernel(r, q, out)
ts = []
for _ in range(reps):
    t0 = time.perf_counter()
    m.run_b200_kernel(r, q, out)
    ts.append(time.perf_counter() - t0)
t = min(ts)
pick = rng.integers(0, n_r, 32)
ok = np.array_equal(out[pick], oracle.naive(r[pick], q))
print(f"run_b200_kernel {n_r}x{n_q}x{L}: {t*1e3:.1f} ms  ({n_r*n_q*4/t/1e9:.1f} GB/s of u32 output, "
      f"{n_r*n_q/t:.3e} cmp/s)  oracle rows ok={ok}", flush=True)

# the same matrix streamed into a packed-binary (FIDM) score file
import os, tempfile
R = m.Panel(tuple(range(n_r)), r, L)
Q = m.Panel(tuple(range(n_q)), q, L)
with tempfile.TemporaryDirectory(dir=os.environ.get("FASTID_FIDM_DIR")) as d:
    path = os.path.join(d, "scores.fidm")
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        m.compare_to_fidm(R, Q, path)
        ts.append(time.perf_counter() - t0)
        os.unlink(path)
    t = min(ts)
    print(f"compare_to_fidm {n_r}x{n_q}x{L}: {t*1e3:.1f} ms  ({n_r*n_q*4/t/1e9:.1f} GB/s into {d})", flush=True)
