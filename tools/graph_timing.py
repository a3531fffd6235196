"""Host-buffer top-k per call: KnownDatabase.search_words (a dozen enqueues per
call) vs the same search captured as one CUDA graph (KnownDatabase.graphed_search).

usage: graph_timing.py [N_R] [L] [NQ,...]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

n_r = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
L = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
nqs = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 16, 256, 2048]
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, L // 64), dtype=torch.int64, device="cuda", generator=g)
db = KnownDatabase(m.DevicePanel.from_words(r, L))
for n_q in nqs:
    q = r[torch.randint(0, n_r, (n_q,), device="cuda", generator=g)].cpu().numpy().view(np.uint64)
    gs = db.graphed_search(n_q, 16)
    a = db.search_words(q, 16)
    b = gs.run(q)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    res = {}
    for name, fn in (("search_words", lambda: db.search_words(q, 16)), ("graphed", lambda: gs.run(q))):
        fn()
        ts = []
        for _ in range(20):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        res[name] = np.median(ts) * 1e3
    print(f"{n_r}x{n_q}x{L} top-16 per call: search_words {res['search_words']:.3f} ms, "
          f"graphed {res['graphed']:.3f} ms", flush=True)
