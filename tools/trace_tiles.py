"""Per-tile timeline of CTA 0 of the top-k tensor kernel (fastid_debug_trace).

usage: trace_tiles.py [N_R] [N_Q] [L] [TILES]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1707_00516_b200 as m
from paper_1707_00516_b200 import _native
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L, tiles = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (20_000_000, 2048, 1024, 8000)))
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-2**62, 2**62, (n_r, L // 64), dtype=torch.int64, device="cuda", generator=g)
q = torch.randint(-2**62, 2**62, (n_q, L // 64), dtype=torch.int64, device="cuda", generator=g)
db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation="tensor_f4")
del r
dq = m.DevicePanel.from_words(q, L)
lib = _native.diag_lib()
lib.fastid_debug_flags(int(sys.argv[5]) if len(sys.argv) > 5 else 0)
db.topk_device(dq, 16); torch.cuda.synchronize()
buf = torch.zeros((tiles * 68,), dtype=torch.int64, device="cuda")
lib.fastid_debug_trace(buf.data_ptr(), tiles)
db.topk_device(dq, 16); torch.cuda.synchronize()
lib.fastid_debug_trace(None, 0)
full = buf.cpu().numpy().astype(np.int64)
ins = full[tiles * 67:]
t = full[:tiles * 67].reshape(tiles, 67)[200:]
if ins.any():
    print("insertions per tile index (all CTAs):", [int(ins[i]) for i in (0, 1, 2, 5, 10, 20, 50, 100, 200, 500, 1000, 2000, 4000, 7000) if i < tiles])
    print("total insertions:", int(ins.sum()))
acq, rel, ld, done = t[:, 3:19], t[:, 19:35], t[:, 35:51], t[:, 51:67]
w = [i for i in range(16) if acq[:, i].any()]
acq, rel, ld, done = acq[:, w], rel[:, w], ld[:, w], done[:, w]
wait, go, issued = t[:, 0], t[:, 1], t[:, 2]
med = lambda x: int(np.median(x))
print(f"epilogue warps traced: {len(w)}")
print(f"MMA tile period {med(np.diff(go))}; t_empty wait (go-wait) {med(go - wait)}; issue span {med(issued - go)}")
print(f"commit(issued) -> first acquire {med(acq.min(1) - issued)}; -> last acquire {med(acq.max(1) - issued)}")
print(f"acquire -> loaded (per warp median) {med(ld - acq)}; loaded -> processed {med(done - ld)}; release - loaded {med(rel - ld)}")
print(f"last release of tile i -> MMA go of tile i+2 {med(go[2:] - rel.max(1)[:-2])}")
print(f"per-warp processed(i) -> acquire(i+1) {med(acq[1:] - done[:-1])}")
for pct in (50, 90, 99):
    print(f"  p{pct}: loaded->processed {int(np.percentile(done - ld, pct))}, acquire spread {int(np.percentile(acq.max(1) - acq.min(1), pct))}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); db.topk_device(dq, 16); e1.record(); e1.synchronize()
print(f"kernel+merge {e0.elapsed_time(e1):.3f} ms")
pt = done - ld
for lo, hi in ((0, 200), (500, 700), (1100, 1300)):
    x = pt[lo:hi]
    print(f"tiles {lo+200}-{hi+200}: loaded->processed p50 {int(np.percentile(x, 50))} p90 {int(np.percentile(x, 90))} "
          f"p99 {int(np.percentile(x, 99))}; MMA wait p50 {med((go - wait)[lo:hi])}")
for lo in (2000, 4000, 7000):
    x = pt[lo:lo + 500]
    print(f"tiles {lo+200}-{lo+700}: loaded->processed p50 {int(np.percentile(x, 50))} p90 {int(np.percentile(x, 90))} "
          f"p99 {int(np.percentile(x, 99))}; MMA wait p50 {med((go - wait)[lo:lo+500])}")
