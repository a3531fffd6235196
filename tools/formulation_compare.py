"""One top-16 launch per formulation on the same 2048 x N x 1024 job (for ncu):
CUDA-core LOP3+POPC vs tcgen05 i8 vs tcgen05 mxf4 (prepared image, CTA pairs).

usage: formulation_compare.py [N_R]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

n_r = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
n_q, L = 2048, 1024
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, L // 64), dtype=torch.int64, device="cuda", generator=g)
q = torch.randint(-(2**63), 2**63 - 1, (n_q, L // 64), dtype=torch.int64, device="cuda", generator=g)
dq = m.DevicePanel.from_words(q, L)
for form in ("popc", "tensor_i8", "tensor_f4"):
    db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation=form)
    db.topk_device(dq, 16)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); db.topk_device(dq, 16); e1.record(); e1.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    print(f"{form:10s} {n_r}x{n_q}x{L} top-16: {t*1e3:8.3f} ms  {n_r*n_q*L/t:.3e} bit-pairs/s", flush=True)
    del db
    torch.cuda.empty_cache()
