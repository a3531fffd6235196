"""A database whose mxf4 image cannot fit in HBM (20M x 16384 loci: 41 GB packed, 164 GB image)
falls back to packed operands and still answers exactly (1 unknown checked against the oracle)."""
import sys, time, warnings
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import numpy as np, torch
import oracle
import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

n_r, L, n_q = 20_000_000, 16384, 64
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, L // 64), dtype=torch.int64, device="cuda", generator=g)
panel = m.DevicePanel.from_words(r, L)
q = r[torch.randint(0, n_r, (n_q,), device="cuda", generator=g)].clone()
del r
torch.cuda.empty_cache()
with warnings.catch_warnings(record=True) as w:
    warnings.simplefilter("always")
    db = KnownDatabase(panel, formulation="tensor_f4")
print("image:", db.image is not None, "| warnings:", [str(x.message)[:100] for x in w])
dq = m.DevicePanel.from_words(q, L)
t0 = time.perf_counter(); s, x = db.topk_device(dq, 16); torch.cuda.synchronize(); t = time.perf_counter() - t0
print(f"top-16 of {n_r} x {n_q} x {L}: {t*1e3:.1f} ms ({n_r*n_q*L/t:.3e} bit-pairs/s)")
rows = panel.rows.view(torch.int64).cpu().numpy().view(np.uint64)[:, : L // 64]
qq = q[:1].cpu().numpy().view(np.uint64)
es, ex, _ = oracle.topk(rows, qq, 16)
ok = np.array_equal(s[:1].cpu().numpy().view(np.uint32), es) and np.array_equal(x[:1].cpu().numpy(), ex)
print("oracle check (unknown 0 over all knowns):", ok)
