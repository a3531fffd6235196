"""Measure BASELINE.json configs C1, C2, C4, C5 (C3 is bench.py) on one B200.

Each line: config, formulation, device time (CUDA events, warm, min of reps),
comparisons/s, bit-pairs/s, and an oracle spot check.  Synthetic inputs are
generated on the device (torch RNG); knowns are uniform random bits, unknowns
planted near-copies (C1-C3, C5) or OR-mixtures of 2-5 knowns (C4).

usage: python tools/bench_configs.py [--only C2,C4] [--json out.jsonl]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (checker only)
import paper_1707_00516_b200 as m  # noqa: E402
from paper_1707_00516_b200.search import KnownDatabase  # noqa: E402


def rand_words(n, L, gen, density=None):
    nw = -(-L // 64)
    if density is None:
        w = torch.randint(-(2**63), 2**63 - 1, (n, nw), dtype=torch.int64, device="cuda", generator=gen)
    else:
        w = torch.zeros((n, nw), dtype=torch.int64, device="cuda")
        step = max(1, (1 << 28) // (nw * 64))  # rows per chunk: ~1 GiB of float draws
        for r0 in range(0, n, step):
            bits = (torch.rand((min(step, n - r0), nw * 64), device="cuda", generator=gen) < density).to(torch.int64)
            for b in range(64):
                w[r0:r0 + bits.shape[0]] |= bits[:, b::64] << (63 - b)
            del bits
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


def run_full(cfg, n_known, n_unknown, L, forms, out, gen, check_rows=64, planted=True):
    r = rand_words(n_known, L, gen)
    q = rand_words(n_unknown, L, gen)
    if planted:
        q[: n_unknown // 2] = r[torch.randint(0, n_known, (n_unknown // 2,), device="cuda", generator=gen)]
    for form in forms:
        db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation=form)
        dq = m.DevicePanel.from_words(q, L)
        o = torch.empty((n_known, n_unknown), dtype=torch.int32, device="cuda")
        t = timed(lambda: db.full_device(dq, o))
        rows = torch.randint(0, n_known, (check_rows,), device="cuda", generator=gen)
        got = o[rows].cpu().numpy().view(np.uint32)
        exp = oracle.naive(words_np(r[rows]), words_np(q))
        report(out, config=cfg, mode="full", formulation=form, n_known=n_known, n_unknown=n_unknown, loci=L,
               seconds=t, out_gb_per_s=n_known * n_unknown * 4 / t / 1e9,
               check=f"{check_rows} random rows vs oracle", ok=bool(np.array_equal(got, exp)))
        del db, o
        torch.cuda.empty_cache()


def run_topk(cfg, r, q, L, forms, out, k=16, check_q=4, max_score=None, extra=None):
    n_known, n_unknown = r.shape[0], q.shape[0]
    for form in forms:
        db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation=form)
        dq = m.DevicePanel.from_words(q, L)
        ws = torch.empty(m.compare.topk_workspace_bytes(n_known, n_unknown, k, form), dtype=torch.uint8,
                         device="cuda")
        res = [None]

        def fn():
            res[0] = db.topk_device(dq, k, max_score, ws)

        t = timed(fn)
        ok = None
        if check_q:
            pick = np.linspace(0, n_unknown - 1, check_q).astype(int)
            s = res[0][0].cpu().numpy().view(np.uint32)[pick]
            x = res[0][1].cpu().numpy()[pick]
            es, ex, _ = oracle.topk(words_np(r), words_np(q)[pick], k,
                                    0xFFFFFFFE if max_score is None else max_score)
            ok = bool(np.array_equal(s, es) and np.array_equal(x, ex))
        report(out, config=cfg, mode=f"top{k}", formulation=form, n_known=n_known, n_unknown=n_unknown, loci=L,
               seconds=t, check=f"{check_q} unknowns vs oracle over all knowns", ok=ok, **(extra or {}))
        del db
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
        run_full("C2", 1_000_000, 2048, 1024, forms, out, gen)

    if "C4" in only:
        # 512 mixtures of 2-5 contributors x 20M knowns x 5,000 loci, AND-NOT exclusion counts:
        # contributors score 0; report top-16 (contributors first) with a threshold.
        L, n_known, n_mix = 5000, 20_000_000, 512
        r = rand_words(n_known, L, gen, density=None)
        # per-locus minor-allele presence p ~ U(0.1, 0.5): resample knowns row-blockwise at lower density
        r[: n_known // 4] = rand_words(n_known // 4, L, gen, density=0.3)
        contrib = torch.randint(0, n_known // 4, (n_mix, 5), device="cuda", generator=gen)
        ncon = torch.randint(2, 6, (n_mix,), device="cuda", generator=gen)
        q = torch.zeros((n_mix, r.shape[1]), dtype=torch.int64, device="cuda")
        for c in range(5):
            use = (ncon > c).unsqueeze(1)
            q |= torch.where(use, r[contrib[:, c]], torch.zeros_like(q))
        run_topk("C4", r, q, L, [f for f in forms if f != "popc"] + (["popc"] if "popc" in forms else []), out,
                 k=16, check_q=2, extra={"contributors": "2-5 per mixture"})
        del r, q
        torch.cuda.empty_cache()

    if "C5" in only:
        for L in (1024, 2048, 5000, 10_000, 20_000, 40_000):
            r = rand_words(4096, L, gen)
            run_full(f"C5-M2M-L{L}", 4096, 4096, L, forms, out, gen, check_rows=16)
        for L in (1024, 5000, 10_000, 40_000):
            n_known = 5_000_000 if L <= 5000 else 1_000_000
            r = rand_words(n_known, L, gen)
            q = rand_words(2048, L, gen)
            q[:1024] = r[torch.randint(0, n_known, (1024,), device="cuda", generator=gen)]
            run_topk(f"C5-2048xN-L{L}", r, q, L, [f for f in forms if f != "popc" or L <= 5000], out, k=16,
                     check_q=2 if n_known * L <= 5e9 else 0)
            del r, q
            torch.cuda.empty_cache()
    if out:
        out.close()


if __name__ == "__main__":
    main()
