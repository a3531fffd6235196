"""Bulk panel ingest timing: native parser (csrc/ingest.cu) vs the reference's io.load_panel.

usage: ingest_timing.py [N_PROFILES] [L] [REF_SAMPLE]   (the reference is timed only if importable)
"""
import os, sys, tempfile, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1707_00516_b200.ingest import load_panel

n, L = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (1_000_000, 1024)))
ref_sample = int(sys.argv[3]) if len(sys.argv) > 3 else 50_000
rng = np.random.default_rng(3)
words = rng.integers(0, 2**64, (n, L // 64), dtype=np.uint64)
with tempfile.TemporaryDirectory() as d:
    path = os.path.join(d, "p.panel")
    hexw = np.char.zfill(np.char.mod("%x", words.reshape(-1)), 16).reshape(n, -1)
    with open(path, "w") as fh:
        fh.write(f"#bits={L}\n")
        for i in range(n):
            fh.write(f"P{i}\t{''.join(hexw[i])}\n")
    size = os.path.getsize(path)
    t0 = time.perf_counter()
    p = load_panel(path, 64)
    t = time.perf_counter() - t0
    assert np.array_equal(p.words, words)
    print(f"native load_panel: {n} profiles x {L} loci ({size/1e6:.0f} MB) in {t:.3f} s "
          f"({n/t:.3e} profiles/s, {size/t/1e9:.2f} GB/s, {os.cpu_count()} host threads)", flush=True)
    try:
        sys.path.insert(0, "/root/reference/pkg/src")
        os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp())
        from fastid.io import load_panel as ref_load
    except Exception:
        ref_load = None
    if ref_load is not None:
        sp = os.path.join(d, "s.panel")
        with open(path) as src, open(sp, "w") as dst:
            for i, line in enumerate(src):
                if i > ref_sample:
                    break
                dst.write(line)
        t0 = time.perf_counter()
        rp = ref_load(sp, 64)
        t = time.perf_counter() - t0
        assert np.array_equal(rp.words, words[:ref_sample])
        print(f"reference io.load_panel: {ref_sample} profiles in {t:.3f} s ({ref_sample/t:.3e} profiles/s)")
