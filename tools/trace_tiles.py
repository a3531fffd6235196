"""Per-tile timeline of CTA 0 of the top-k tensor kernel (fastid_debug_trace)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1707_00516_b200 as m
from paper_1707_00516_b200 import _native
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L, tiles = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-2**62, 2**62, (n_r, L // 64), dtype=torch.int64, device="cuda", generator=g)
q = torch.randint(-2**62, 2**62, (n_q, L // 64), dtype=torch.int64, device="cuda", generator=g)
db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation="tensor_f4")
dq = m.DevicePanel.from_words(q, L)
db.topk_device(dq, 16); torch.cuda.synchronize()
buf = torch.zeros((tiles, 67), dtype=torch.int64, device="cuda")
_native.lib().fastid_debug_trace(buf.data_ptr(), tiles)
db.topk_device(dq, 16); torch.cuda.synchronize()
_native.lib().fastid_debug_trace(None, 0)
t = buf.cpu().numpy().astype(np.int64)
t0 = t[0, 0]
print("tile  mma_wait  mma_go  mma_issued | epi_acq(min,max)  epi_rel(min,max) | epi_busy(max)")
for i in range(0, tiles, max(1, tiles // 40)):
    row = t[i] - t0
    acq, rel = row[3:19], row[19:35]
    print(f"{i:5d} {row[0]:9d} {row[1]:8d} {row[2]:10d} | {acq.min():8d} {acq.max():8d}  {rel.min():8d} {rel.max():8d} | {(rel - acq).max():6d}")
d = np.diff(t[:, 1])
print("median MMA tile period (cycles):", np.median(d[d > 0]) if len(d) else None)
print("median MMA wait (go - wait):", np.median(t[:, 1] - t[:, 0]))
print("median epilogue span (max rel - min acq):", np.median(t[:, 19:35].max(1) - t[:, 3:19].min(1)))
print("median lag commit->epi acquire:", np.median(t[:, 3:19].min(1) - t[:, 2]))
acq, b0l, b0d, rel = t[:, 3:19], t[:, 35:51], t[:, 51:67], t[:, 19:35]
sl = slice(200, None)
print("per-warp medians (cycles) over tiles 200..:")
print("  acquire -> batch0 loaded:", np.median((b0l - acq)[sl], axis=0).astype(int).tolist())
print("  batch0 loaded -> processed:", np.median((b0d - b0l)[sl], axis=0).astype(int).tolist())
print("  batch0 processed -> release (batch1 loaded):", np.median((rel - b0d)[sl], axis=0).astype(int).tolist())
print("  acquire spread (max-min):", int(np.median((acq.max(1) - acq.min(1))[sl])))

# same run with the epilogue's TMEM loads switched off (results invalid; timing only)
_native.lib().fastid_debug_flags(1)
buf.zero_()
_native.lib().fastid_debug_trace(buf.data_ptr(), tiles)
db.topk_device(dq, 16); torch.cuda.synchronize()
_native.lib().fastid_debug_trace(None, 0)
_native.lib().fastid_debug_flags(0)
t = buf.cpu().numpy().astype(np.int64)
d = np.diff(t[:, 1])
print("NO-TMEM-LOAD epilogue: median MMA tile period:", np.median(d[d > 0]),
      "median issue span (issued-go):", np.median(t[:, 2] - t[:, 1]))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for flags in (0, 1):
    _native.lib().fastid_debug_flags(flags)
    e0.record(); db.topk_device(dq, 16); e1.record(); e1.synchronize()
    print(f"flags={flags}: kernel+merge {e0.elapsed_time(e1):.3f} ms")
_native.lib().fastid_debug_flags(0)
