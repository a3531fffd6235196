"""Race / hang hunt: many back-to-back launches of several prepared-image shapes
(resident unknowns, dual-tile streamed unknowns, one unknown group, spare pairs,
full matrix, threshold), every result compared with the first run's.

usage: stress_runs.py [REPS]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
g = torch.Generator(device="cuda").manual_seed(3)
bad = 0
CASES = ((2_000_000, 2048, 1024, "topk", "andnot"), (1_000_000, 512, 5000, "topk", "andnot"),
         (3_000_000, 7, 1024, "topk", "andnot"), (500_000, 1000, 2000, "topk", "andnot"),
         (300_000, 2048, 1024, "full", "andnot"), (1_000_000, 300, 3500, "thr", "andnot"),
         # the CUDA-core scan (1, 2 and 4 unknowns: bulk list updates, 3 CTAs per SM) and
         # the operators (XOR's signed mxf4 operand, AND)
         (3_000_000, 1, 1024, "topk", "andnot"), (3_000_000, 2, 1024, "topk", "xor"),
         (3_000_000, 4, 1024, "topk", "and"), (1_000_000, 2048, 1024, "topk", "xor"),
         (300_000, 512, 1024, "full", "xor"))
for n_r, n_q, L, mode, op in CASES:
    nw = -(-L // 64)
    r = torch.randint(-(2**63), 2**63 - 1, (n_r, nw), dtype=torch.int64, device="cuda", generator=g)
    if L % 64:
        r[:, -1] &= ~((1 << (64 - L % 64)) - 1)
    q = r[torch.randint(0, n_r, (n_q,), device="cuda", generator=g)].clone()
    db = KnownDatabase(m.DevicePanel.from_words(r, L), op=op)
    dq = m.DevicePanel.from_words(q, L)
    qp = m.Panel(tuple(range(n_q)), q.cpu().numpy().view("uint64"), L)

    def run():
        if mode == "topk":
            s, x = db.topk_device(dq, 16)
            return s.clone(), x.clone()
        if mode == "full":
            return (db.full_device(dq).clone(),)
        h = db.threshold(qp, L // 8)  # planted copies (score 0) only: random pairs sit near L/4
        return tuple(torch.from_numpy(a.astype("int64")) for a in (h.query, h.ref, h.score))

    ref = run()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n_bad = 0
    for i in range(reps):
        got = run()
        if not all(torch.equal(a, b) for a, b in zip(got, ref)):
            n_bad += 1
    torch.cuda.synchronize()
    bad += n_bad
    print(f"{n_r}x{n_q}x{L} {mode} {op}: {reps} runs in {time.perf_counter() - t0:.1f} s, {n_bad} differing", flush=True)
    del db, r, q, dq
    torch.cuda.empty_cache()
print("stress ok" if bad == 0 else f"STRESS FAILED: {bad} differing runs")
