"""Randomised parity sweep on the GPU: random shapes (log-uniform sizes, loci
near tile / stage / word boundaries, u32 and u64 words), random formulations,
database options, chunked images, k, score caps, epilogues and operators
(AND-NOT / AND / XOR; AND and XOR against oracle.np_scores_op), each result
compared bit-exactly with the oracle.  Runs for SECONDS; prints every failure
with its seed so it can be replayed.

usage: fuzz_parity.py [SECONDS] [SEED]
"""
import os
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
from paper_1707_00516_b200.search import DB_OPTIONS, KnownDatabase

seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 600
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 1
workers = os.cpu_count() or 1


def rand_words(rng, n, L, width):
    nw = -(-L // width)
    dt = np.uint64 if width == 64 else np.uint32
    w = rng.integers(0, 2**width, (n, nw), dtype=dt)
    if L % width:
        w[:, -1] &= dt((2**width - 1) ^ ((1 << (width - L % width)) - 1))
    return w


def pick_L(rng):
    base = rng.choice([64, 128, 256, 512, 1024, 2048, 2304, 3072, 3200, 4096, 5000, 8192, 10000])
    return int(max(1, base + rng.integers(-70, 70))) if rng.random() < 0.6 else int(base)


def case(seed):
    rng = np.random.default_rng(seed)
    L = pick_L(rng)
    width = 64 if rng.random() < 0.7 else 32
    budget = 2e11 / max(L, 1)  # n_r * n_q cap so the oracle stays fast
    n_q = int(np.exp(rng.uniform(0, np.log(3000))))
    n_r = int(min(np.exp(rng.uniform(0, np.log(400_000))), max(1, budget / max(n_q, 1))))
    r = rand_words(rng, n_r, L, width)
    q = rand_words(rng, n_q, L, width)
    planted = min(n_q, max(1, n_q // 8))
    q[:planted] = r[rng.integers(0, n_r, planted)]
    if n_r > 4:
        r[-2:] = r[:2]  # ties across the ends
    form = rng.choice(["tensor_f4", "tensor_f4", "tensor_f4", "tensor_i8", "popc"])
    if not m._native.supports(form, L):
        form = "auto"
    chunk = None
    if form == "tensor_f4" and n_r > 400 and rng.random() < 0.2:
        chunk = int(192 * rng.integers(1, max(2, n_r // 192)))
    op = str(rng.choice(["andnot", "andnot", "andnot", "and", "xor"]))
    if op != "andnot" and n_r * n_q * r.shape[1] > 3e8:
        op = "andnot"  # the numpy operator oracle is for small cases

    def o_full():
        if op == "andnot":
            return oracle.blocked(r, np.ascontiguousarray(q.T), 64, 16, workers)
        return oracle.np_scores_op(r, q, op, block=max(1, int(5e7 // max(1, n_q * r.shape[1]))))

    def o_topk(k, ms):
        if op == "andnot":
            return oracle.topk(r, q, k, ms, workers)
        return oracle.topk_from_matrix(o_full(), k, ms)

    db = KnownDatabase(r, L, formulation=form, ref_base=int(rng.integers(0, 3)) * 1000, image_chunk_rows=chunk, op=op)
    if chunk:
        db.chunked_min_queries = 1
    for name in DB_OPTIONS:
        if rng.random() < 0.15:
            db.set_option(name, True)
    mode = rng.choice(["topk", "topk", "threshold", "full", "streamed", "graphed"])
    if mode == "streamed":  # host panel streamed through the device in random chunks
        k = int(rng.integers(1, 33))
        cr = int(rng.integers(1, n_r + 1)) if rng.random() < 0.8 else 0
        R = m.Panel(tuple(range(n_r)), r, L)
        Q = m.Panel(tuple(range(n_q)), q, L)
        res = m.topk_streamed(R, Q, k, formulation=form, chunk_rows=cr, ref_base=7, op=op)
        es, ex, _ = o_topk(k, 0xFFFFFFFE)
        ok = np.array_equal(res.scores, es) and np.array_equal(res.index, np.where(ex >= 0, ex + 7, -1))
        return ok, f"seed {seed}: {n_r}x{n_q}x{L} w{width} {form} op={op} streamed chunk_rows={cr} k={k}"
    if mode == "graphed":
        k = int(rng.integers(1, 33))
        g = db.graphed_search(n_q, k)
        s, x = g.run(q)
        es, ex, _ = o_topk(k, 0xFFFFFFFE)
        ok = np.array_equal(s, es) and np.array_equal(x, np.where(ex >= 0, ex + db.ref_base, -1))
        return ok, f"seed {seed}: {n_r}x{n_q}x{L} w{width} {form} op={op} chunk={chunk} graphed k={k}"
    desc = f"seed {seed}: {n_r}x{n_q}x{L} w{width} {form} op={op} chunk={chunk} opts={sorted(getattr(db.image, 'options', set()) or [])} {mode}"
    base = db.ref_base
    if mode == "topk":
        k = int(rng.integers(1, 33))
        ms = None if rng.random() < 0.6 else int(rng.integers(0, max(1, L // 2)))
        s, x = db.search_words(q, k, ms)
        es, ex, _ = o_topk(k, 0xFFFFFFFE if ms is None else ms)
        ok = np.array_equal(s, es) and np.array_equal(x, np.where(ex >= 0, ex + base, -1))
        return ok, desc + f" k={k} max={ms}"
    full = o_full()
    if mode == "threshold":
        t = int(np.percentile(full, rng.uniform(0, 3))) if full.size else 0
        h = db.threshold(m.Panel(tuple(range(n_q)), q, L), t)
        hq, hr, hs = oracle.threshold_from_matrix(full, t)
        ok = np.array_equal(h.query, hq) and np.array_equal(h.ref, hr + base) and np.array_equal(h.score, hs)
        return ok, desc + f" t={t}"
    got = db.full_device(m.DevicePanel.from_words(q, L)).cpu().numpy().view(np.uint32)
    return bool(np.array_equal(got, full)), desc


t_end = time.time() + seconds
n = fails = 0
seed = seed0
while time.time() < t_end:
    try:
        ok, desc = case(seed)
    except Exception as e:  # a crash is a failure too
        ok, desc = False, f"seed {seed}: {type(e).__name__}: {e}"
    n += 1
    if not ok:
        fails += 1
        print("FAIL", desc, flush=True)
    elif n % 50 == 0:
        print(f"{n} cases ok (last: {desc})", flush=True)
    seed += 1
    torch.cuda.empty_cache()
print(f"fuzz: {n} cases, {fails} failures")
