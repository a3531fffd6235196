"""Kernel timing on bench.py's exact inputs (host-generated knowns, planted unknowns) vs device-generated ones."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench
import paper_1707_00516_b200 as m
from paper_1707_00516_b200.search import KnownDatabase

n_r, n_q, L, k = 20_000_000, 2048, 1024, 16
g = torch.Generator().manual_seed(1707 * 1000)
host = torch.randint(-(2**63), 2**63 - 1, (n_r, L // 64), dtype=torch.int64, generator=g)
host_np = host.numpy().view(np.uint64)
qh, _ = bench.planted_unknowns(host_np, n_q, L, np.random.default_rng(1707))
gd = torch.Generator(device="cuda").manual_seed(0)
qr = torch.randint(-(2**63), 2**63 - 1, (n_q, L // 64), dtype=torch.int64, device="cuda", generator=gd)


def run(name, db, dq, steps=10):
    ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, k, "tensor_f4"), dtype=torch.uint8, device="cuda")
    out = (torch.empty((n_q, k), dtype=torch.int32, device="cuda"), torch.empty((n_q, k), dtype=torch.int64, device="cuda"))
    for _ in range(3):
        db.topk_device(dq, k, None, ws, out)
    ks = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        db.topk_device(dq, k, None, ws, out, events=(e0, e1))
        ks.append((e0, e1))
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) for a, b in ks]
    print(f"{name:40s} kernel med {np.median(t):.3f} ms", flush=True)


db = KnownDatabase(m.DevicePanel.from_words(host.cuda(), L), formulation="tensor_f4")
run("bench knowns + bench planted unknowns", db, m.DevicePanel.from_words(qh, L))
run("bench knowns + random unknowns", db, m.DevicePanel.from_words(qr, L))
src = torch.randint(0, n_r, (n_q,), generator=torch.Generator().manual_seed(5))
run("bench knowns + exact copies", db, m.DevicePanel.from_words(host[src].numpy().view(np.uint64), L))
