"""C3-shaped threshold search (2048 planted unknowns x N knowns x 1024): hits with score <= T,
through KnownDatabase.threshold (device kernel + hit compaction + host copy), oracle-checked.
usage: threshold_timing.py [N_R] [T]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import numpy as np, torch
import oracle
import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

n_r = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
T = int(sys.argv[2]) if len(sys.argv) > 2 else 64
n_q, L = 2048, 1024
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, L // 64), dtype=torch.int64, device="cuda", generator=g)
src = torch.randint(0, n_r, (n_q,), device="cuda", generator=g)
q = r[src].clone()
db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation="tensor_f4")
qp = m.Panel(tuple(range(n_q)), q.cpu().numpy().view(np.uint64), L)
hits = db.threshold(qp, T)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter(); hits = db.threshold(qp, T); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
t = min(ts)
print(f"threshold <= {T}: {len(hits.query)} hits over {n_r}x{n_q}x{L} in {t*1e3:.2f} ms ({n_r*n_q/t:.3e} cmp/s)")
# every planted copy must be found with score 0
srcn = src.cpu().numpy()
found = set(zip(hits.query.tolist(), hits.ref.tolist()))
assert all((j, int(srcn[j])) in found for j in range(n_q))
assert (hits.score <= T).all()
print("planted copies all found; scores within threshold")
