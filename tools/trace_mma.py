"""Per-stage timeline of the MMA issuer of CTA 0 (debug flag 8): u_full waits per stage."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1707_00516_b200 as m
from paper_1707_00516_b200 import _native
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L, tiles = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (20_000_000, 2048, 1024, 2000)))
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-2**62, 2**62, (n_r, L // 64), dtype=torch.int64, device="cuda", generator=g)
q = torch.randint(-2**62, 2**62, (n_q, L // 64), dtype=torch.int64, device="cuda", generator=g)
db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation="tensor_f4")
del r
dq = m.DevicePanel.from_words(q, L)
lib = _native.diag_lib()
db.topk_device(dq, 16); torch.cuda.synchronize()
buf = torch.zeros((tiles, 67), dtype=torch.int64, device="cuda")
n_kst = (L + 255) // 256
for flags, name in ((8, "pair"), (8 | 4, "pair-noload"), (8 | 2, "single")):
    lib.fastid_debug_flags(flags)
    buf.zero_()
    lib.fastid_debug_trace(buf.data_ptr(), tiles)
    db.topk_device(dq, 16); torch.cuda.synchronize()
    lib.fastid_debug_trace(None, 0)
    t = buf.cpu().numpy().astype(np.int64)[200:]
    go, issued = t[:, 1], t[:, 2]
    pre, post = t[:, 35:35 + n_kst], t[:, 51:51 + n_kst]
    per = np.diff(go)
    print(f"== {name}: median tile period {np.median(per):.0f} cyc (ideal {128*224*L/15200*(2 if 'pair' in name else 1):.0f}); "
          f"t_empty wait {np.median(go - t[:, 0]):.0f}; issue span {np.median(issued - go):.0f}")
    print("   per-stage u_full wait (median):", np.median(post - pre, axis=0).astype(int).tolist(),
          " stage-to-stage:", np.median(np.diff(post, axis=1), axis=0).astype(int).tolist())
lib.fastid_debug_flags(0)
