"""Full-matrix writes stay inside the logical matrix: the output is a poisoned
view [n_refs rows, n_queries cols] of a larger buffer (row pitch 160, 100 extra
rows), and every cell outside the view must still hold the poison afterwards.
Checked for each formulation, with and without the prepared image, and with
each epilogue store variant (debug flags 0 / 256 / 2048)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1])); sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import numpy as np, torch, oracle
import paper_1707_00516_b200 as m
from paper_1707_00516_b200 import _native
from paper_1707_00516_b200.search import KnownDatabase
rng = np.random.default_rng(0)
bad_any = False
for L in (300, 1024):
    nw = -(-L // 64)
    for n_r, n_q in ((2500, 150), (2500, 152), (2431, 149), (700, 128)):
        r = rng.integers(0, 2**64, (n_r, nw), dtype=np.uint64); q = rng.integers(0, 2**64, (n_q, nw), dtype=np.uint64)
        if L % 64:
            r[:, -1] &= ~np.uint64(0) << np.uint64(64 - L % 64); q[:, -1] &= ~np.uint64(0) << np.uint64(64 - L % 64)
        exp = oracle.naive(r, q)
        dq = m.DevicePanel.from_words(q, L)
        for form in ("tensor_f4", "tensor_i8", "popc"):
            for img in (True, False):
                for flags in (0, 256, 2048):
                    _native.diag_lib().fastid_debug_flags(flags)
                    buf = torch.full((n_r + 100, 160), -1, dtype=torch.int32, device="cuda")
                    p = buf[:n_r, :n_q]
                    if img:
                        KnownDatabase(r, L, formulation=form).full_device(dq, p)
                    else:
                        m.compare.compare_device(m.DevicePanel.from_words(r, L), dq, p, form)
                    g = buf.cpu().numpy().view(np.uint32)
                    ok = np.array_equal(g[:n_r, :n_q], exp)
                    outside = g.copy(); outside[:n_r, :n_q] = 0xFFFFFFFF
                    bad_cols = sorted(set(np.nonzero(outside != 0xFFFFFFFF)[1].tolist()))
                    bad_rows = int((outside != 0xFFFFFFFF).any(1).sum())
                    if not ok or bad_cols:
                        bad_any = True
                        print(L, n_r, n_q, form, "image" if img else "plain", flags, "MISMATCH" if not ok else "ok",
                              "clobbered cols", bad_cols[:8], "rows", bad_rows)
_native.diag_lib().fastid_debug_flags(0)
print("pitch probe:", "FAIL" if bad_any else "all writes inside the view")
