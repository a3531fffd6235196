"""Quick correctness probe of the tensor formulations on small shapes (diagnostic)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np, torch
import paper_1707_00516_b200 as m
import oracle

rng = np.random.default_rng(5)
for form in sys.argv[1].split(","):
    for (n_r, n_q, L) in ((224, 128, 256), (300, 70, 1024), (1000, 300, 512), (5000, 2048, 1024), (777, 129, 2048)):
        if not m._native.supports(form, L):
            print(form, L, "unsupported"); continue
        r = rng.integers(0, 2**64, (n_r, L // 64), dtype=np.uint64)
        q = rng.integers(0, 2**64, (n_q, L // 64), dtype=np.uint64)
        exp = oracle.naive(r, q)
        try:
            got = m.compare_b200(m.Panel(tuple(range(n_r)), r, L), m.Panel(tuple(range(n_q)), q, L), formulation=form).scores
        except Exception as e:
            print(form, (n_r, n_q, L), "ERROR", e); continue
        ok = np.array_equal(got, exp)
        print(form, (n_r, n_q, L), "OK" if ok else "MISMATCH", flush=True)
        if not ok:
            bad = np.argwhere(got != exp)
            print("  n_bad", len(bad), "first", bad[:5].tolist(), "got", got[tuple(bad[0])], "exp", exp[tuple(bad[0])])
            print("  got[0,:8]", got[0, :8], "exp[0,:8]", exp[0, :8])
            print("  ratio mean", (got.astype(float).mean() / exp.mean()))
