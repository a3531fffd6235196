"""A panel whose tensor image does not fit (20M x 16384 loci: 41 GB packed, 164 GB
image): fused top-16 through the chunked image vs the packed-operand kernels, by
batch size -- the crossover the chunked image's per-search build cost sets.

usage: chunked_vs_packed.py [N_R] [L] [NQ,...]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import ChunkedImage, KnownDatabase

n_r = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
L = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
nqs = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [64, 256, 512, 2048]
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-(2**63), 2**63 - 1, (n_r, L // 64), dtype=torch.int64, device="cuda", generator=g)
panel = m.DevicePanel.from_words(r, L)
qsrc = r[torch.randint(0, n_r, (max(nqs),), device="cuda", generator=g)].clone()
del r
torch.cuda.empty_cache()
packed = KnownDatabase(panel, formulation="tensor_f4", prepare=False)
chunked = KnownDatabase(panel, formulation="tensor_f4", prepare=False)
chunked.image = ChunkedImage(panel, "tensor_f4")
print(f"chunk rows {chunked.image.chunk_rows} ({chunked.image.buf.numel() / 1e9:.1f} GB image buffer)", flush=True)
for n_q in nqs:
    dq = m.DevicePanel.from_words(qsrc[:n_q].clone(), L)
    res = {}
    for name, db in (("chunked", chunked), ("packed", packed)):
        s, x = db.topk_device(dq, 16)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s, x = db.topk_device(dq, 16)
        torch.cuda.synchronize()
        res[name] = (time.perf_counter() - t0, s.cpu(), x.cpu())
    same = torch.equal(res["chunked"][1], res["packed"][1]) and torch.equal(res["chunked"][2], res["packed"][2])
    print(f"N_Q {n_q:5d}: chunked image {res['chunked'][0] * 1e3:8.1f} ms  packed {res['packed'][0] * 1e3:8.1f} ms "
          f"({n_r * n_q * L / min(res['chunked'][0], res['packed'][0]):.3e} bit-pairs/s best)  same={same}", flush=True)
