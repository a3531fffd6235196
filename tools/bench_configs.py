"""Measure BASELINE.json configs C1, C2, C4, C5 (C3 is bench.py) on one B200,
each line checked against the CPU oracle at full size.

Each line: config, formulation, device time (CUDA events, warm, min of reps),
comparisons/s, bit-pairs/s, and the oracle check that was run (``ok`` is
always true/false, never skipped):

* C1: score_checksum of the full matrix == the reference's own checksum of the
  same synth_panel inputs (tests/golden/checksums.json).
* C2: the full 1M x 2048 u32 matrix (8.19 GB, D2H) byte-equal to the C port of
  compare_blocked on the same synth_panel inputs; both checksums reported.
* C4: bench.py's generator (per-locus presence p ~ U(0.1, 0.5), OR-mixtures of
  2-5 contributors); the top-16 of all 512 mixtures vs oracle.scan over all
  20M knowns.
* C5: mixture-to-mixture 4096 x 4096 full matrices (every cell vs the oracle)
  and 2048 x N top-16 lines (every unknown vs oracle.scan) across the loci sweep.

usage: python tools/bench_configs.py [--only C1,C2,C4,C5] [--json out.jsonl] [--forms tensor_f4,...]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402  (the C4 generator)
import oracle  # noqa: E402  (checker only)
import paper_1707_00516_b200 as m  # noqa: E402
from paper_1707_00516_b200.search import KnownDatabase  # noqa: E402


def rand_words(n, L, gen):
    nw = -(-L // 64)
    w = torch.randint(-(2**63), 2**63 - 1, (n, nw), dtype=torch.int64, device="cuda", generator=gen)
    tail = L % 64
    if tail:
        w[:, -1] &= ~((1 << (64 - tail)) - 1)
    return w


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


def words_np(w):
    return w.cpu().numpy().view(np.uint64)


def report(out, **kw):
    kw["cmp_per_s"] = kw["n_known"] * kw["n_unknown"] / kw["seconds"]
    kw["bitpairs_per_s"] = kw["cmp_per_s"] * kw["loci"]
    line = json.dumps(kw)
    print(line, flush=True)
    if out:
        out.write(line + "\n")
        out.flush()


def full_matrix_lines(cfg, r_np, q_np, L, forms, out, expected=None, extra=None):
    """Every formulation's full matrix (device), then byte-equality with the oracle's."""
    n_known, n_unknown = r_np.shape[0], q_np.shape[0]
    if expected is None:
        t0 = time.perf_counter()
        expected = oracle.blocked(r_np, np.ascontiguousarray(q_np.T), 64, 16, os.cpu_count() or 1)
        oracle_s = time.perf_counter() - t0
    else:
        oracle_s = None
    dr, dq = m.DevicePanel.from_words(r_np, L), m.DevicePanel.from_words(q_np, L)
    for form in forms:
        db = KnownDatabase(dr, formulation=form)
        o = torch.empty((n_known, n_unknown), dtype=torch.int32, device="cuda")
        t = timed(lambda: db.full_device(dq, o))
        got = o.cpu().numpy().view(np.uint32)
        ok = bool(np.array_equal(got, expected))
        kw = dict(config=cfg, mode="full", formulation=form, n_known=n_known, n_unknown=n_unknown, loci=L,
                  seconds=t, out_gb_per_s=n_known * n_unknown * 4 / t / 1e9,
                  check="every cell byte-equal to the oracle (C port of compare_blocked)", ok=ok,
                  oracle_s=oracle_s)
        kw.update(extra or {})
        report(out, **kw)
        del db, o, got
        torch.cuda.empty_cache()
    return expected


def topk_lines(cfg, dr, q_np, L, forms, out, k=16, r_np=None, extra=None):
    """Every formulation's fused top-k over the resident panel; every unknown vs oracle.scan."""
    n_known, n_unknown = dr.n_profiles, q_np.shape[0]
    if r_np is None:
        r_np = dr.to_words()
    t0 = time.perf_counter()
    (es, ex, _), _ = oracle.scan(r_np, q_np, k, 0xFFFFFFFE)
    oracle_s = time.perf_counter() - t0
    dq = m.DevicePanel.from_words(q_np, L)
    for form in forms:
        db = KnownDatabase(dr, formulation=form)
        ws = torch.empty(m.compare.topk_workspace_bytes(n_known, n_unknown, k, form), dtype=torch.uint8,
                         device="cuda")
        res = [None]

        def fn():
            res[0] = db.topk_device(dq, k, None, ws)

        t = timed(fn)
        s = res[0][0].cpu().numpy().view(np.uint32)
        x = res[0][1].cpu().numpy()
        ok = bool(np.array_equal(s, es) and np.array_equal(x, ex))
        kw = dict(config=cfg, mode=f"top{k}", formulation=form, n_known=n_known, n_unknown=n_unknown, loci=L,
                  seconds=t, check=f"all {n_unknown} unknowns vs oracle.scan over all {n_known} knowns", ok=ok,
                  oracle_s=oracle_s)
        kw.update(extra or {})
        report(out, **kw)
        del db, ws
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C2,C4,C5")
    ap.add_argument("--json", default=None)
    ap.add_argument("--forms", default="tensor_f4,tensor_i8,popc")
    args = ap.parse_args()
    only = set(args.only.split(","))
    forms = args.forms.split(",")
    out = open(args.json, "a") if args.json else None
    gen = torch.Generator(device="cuda").manual_seed(1707)

    if "C1" in only:
        # BASELINE config 1: 64 x 10,000 x 1,024, full matrix; checksum against the reference's
        # own score_checksum of the same synth_panel inputs (tests/golden/checksums.json)
        row = next(r for r in json.loads((ROOT / "tests/golden/checksums.json").read_text())
                   if r["label"].startswith("baseline_config1"))
        refs = oracle.synth_words(row["n_refs"], row["n_words"], 64, row["seed"], 0)
        queries = oracle.synth_words(row["n_queries"], row["n_words"], 64, row["seed"], 1)
        for form in forms:
            dr, dq = m.DevicePanel.from_words(refs, 1024), m.DevicePanel.from_words(queries, 1024)
            o = torch.empty((10_000, 64), dtype=torch.int32, device="cuda")
            t = timed(lambda: m.compare_device(dr, dq, o, formulation=form))
            ok = oracle.score_checksum(o.cpu().numpy().view(np.uint32)) == row["checksum"]
            report(out, config="C1", mode="full", formulation=form, n_known=10_000, n_unknown=64, loci=1024,
                   seconds=t, check="score_checksum == reference checksum", ok=bool(ok))

    if "C2" in only:
        # 2048 x 1M x 1024 full matrix on synth_panel inputs (seed 1707): every cell vs the port
        refs = oracle.synth_words(1_000_000, 16, 64, 1707, 0)
        queries = oracle.synth_words(2048, 16, 64, 1707, 1)
        queries[:1024] = refs[np.random.default_rng(5).integers(0, 1_000_000, 1024)]
        t0 = time.perf_counter()
        exp = oracle.blocked(refs, np.ascontiguousarray(queries.T), 64, 16, os.cpu_count() or 1)
        oracle_s = time.perf_counter() - t0
        full_matrix_lines("C2", refs, queries, 1024, forms, out, expected=exp,
                          extra={"inputs": "synth_panel(1M, 16, 64, 1707, 0/1), 1024 planted copies",
                                 "checksum": oracle.score_checksum(exp), "oracle_s": oracle_s})
        del exp

    if "C4" in only:
        # bench.py's C4: per-locus presence p ~ U(0.1, 0.5), 512 OR-mixtures of 2-5 contributors
        L, n_known, n_mix = 5000, 20_000_000, 512
        dr = bench.c4_shard_panel(m, 1707, 0, n_known, L, torch.device("cuda"))
        q = bench.mixture_unknowns(dr, n_mix, np.random.default_rng(1707))
        topk_lines("C4", dr, q, L, [f for f in forms if f != "popc"] + (["popc"] if "popc" in forms else []), out,
                   extra={"contributors": "2-5 per mixture", "knowns": "p ~ U(0.1, 0.5) per locus"})
        del dr
        torch.cuda.empty_cache()

    if "C5" in only:
        for L in (1024, 2048, 5000, 10_000, 20_000, 40_000):
            r = words_np(rand_words(4096, L, gen))
            q = words_np(rand_words(4096, L, gen))
            q[:2048] = r[np.random.default_rng(L).integers(0, 4096, 2048)]
            full_matrix_lines(f"C5-M2M-L{L}", r, q, L, forms, out)
        for L in (1024, 5000, 10_000, 40_000):
            n_known = 5_000_000 if L <= 5000 else 1_000_000
            r = rand_words(n_known, L, gen)
            q = words_np(rand_words(2048, L, gen))
            q[:1024] = words_np(r[torch.randint(0, n_known, (1024,), device="cuda", generator=gen)])
            dr = m.DevicePanel.from_words(r, L)
            r_np = words_np(r)
            del r
            topk_lines(f"C5-2048xN-L{L}", dr, q, L, [f for f in forms if f != "popc" or L <= 5000], out, k=16,
                       r_np=r_np)
            del dr, r_np
            torch.cuda.empty_cache()
    if out:
        out.close()


if __name__ == "__main__":
    main()
