"""Out-of-core top-k timing (fastid_run_topk): a host-resident known panel
streamed through the device, pinned and pageable, auto chunking; the result
is checked against oracle.scan over the whole panel for every unknown.

usage: streamed_timing.py [N_R] [N_Q] [L] [REPS]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np
import torch

import oracle  # checker only
import paper_1707_00516_b200 as m

n_r, n_q, L = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (20_000_000, 2048, 1024)))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
nw = -(-L // 64)
g = torch.Generator().manual_seed(7)
host = torch.randint(-(2**63), 2**63 - 1, (n_r, nw), dtype=torch.int64, generator=g)
if L % 64:
    host[:, -1] &= ~((1 << (64 - L % 64)) - 1)
r = host.numpy().view(np.uint64)
rng = np.random.default_rng(7)
q = r[rng.integers(0, n_r, n_q)].copy()
Q = m.Panel(tuple(range(n_q)), q, L)
t0 = time.perf_counter()
(es, ex, _), _ = oracle.scan(r, q, 16, 0xFFFFFFFE)
oracle_s = time.perf_counter() - t0
pinned = host.pin_memory()
for what, arr in (("pageable", r), ("page-locked", pinned.numpy().view(np.uint64))):
    R = m.Panel(tuple(range(n_r)), arr, L) if n_r < 100_000 else type("P", (), dict(
        words=arr, bit_length=L, word_width=64, ids=None))()
    res = m.topk_streamed(R, Q, 16)  # warm-up (allocates staging)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        res = m.topk_streamed(R, Q, 16)
        ts.append(time.perf_counter() - t0)
    ok = np.array_equal(res.scores, es) and np.array_equal(res.index, ex)
    t = min(ts)
    print(f"{what:11s} {n_r}x{n_q}x{L} top-16 streamed: {t * 1e3:8.1f} ms  "
          f"{n_r * n_q / t:.3e} cmp/s  host rows {arr.nbytes / t / 1e9:6.1f} GB/s  "
          f"ok={ok} (oracle.scan over all {n_q} unknowns: {oracle_s:.1f} s)", flush=True)
