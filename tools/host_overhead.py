import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_1707_00516_b200 as m
from paper_1707_00516_b200 import _native
from paper_1707_00516_b200.search import KnownDatabase
n_r, n_q, L = 2_000_000, 2048, 1024
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randint(-2**62, 2**62, (n_r, L // 64), dtype=torch.int64, device="cuda", generator=g)
q = torch.randint(-2**62, 2**62, (n_q, L // 64), dtype=torch.int64, device="cuda", generator=g)
db = KnownDatabase(m.DevicePanel.from_words(r, L), formulation="tensor_f4")
dq = m.DevicePanel.from_words(q, L)
ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, 16, "tensor_f4"), dtype=torch.uint8, device="cuda")
out = (torch.empty((n_q, 16), dtype=torch.int32, device="cuda"), torch.empty((n_q, 16), dtype=torch.int64, device="cuda"))
db.topk_device(dq, 16, None, ws, out); torch.cuda.synchronize()
lib = _native.diag_lib()
lib.fastid_debug_flags(128)
for i in range(3):
    h0 = time.perf_counter()
    db.topk_device(dq, 16, None, ws, out)
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"call {i}: host {1e6*(h1-h0):.0f} us", file=sys.stderr, flush=True)
lib.fastid_debug_flags(0)
