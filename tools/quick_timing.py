"""Ad-hoc device timing of one formulation/mode (CUDA events, warm).

usage: quick_timing.py FORMS [MODE] [N_R] [N_Q] [L] [REPS]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1707_00516_b200 as m


def run(form, mode, n_r, n_q, L, k=16, reps=5):
    g = torch.Generator(device="cuda").manual_seed(0)
    nw = L // 64
    rw = torch.randint(-2**62, 2**62, (n_r, nw), dtype=torch.int64, device="cuda", generator=g)
    qw = torch.randint(-2**62, 2**62, (n_q, nw), dtype=torch.int64, device="cuda", generator=g)
    dr = m.DevicePanel.from_words(rw, L); dq = m.DevicePanel.from_words(qw, L)
    del rw, qw
    if mode == "full":
        out = torch.empty((n_r, n_q), dtype=torch.int32, device="cuda")
        fn = lambda: m.compare_device(dr, dq, out, formulation=form)
    else:
        ws = torch.empty(m.compare.topk_workspace_bytes(n_r, n_q, k, form), dtype=torch.uint8, device="cuda")
        o = (torch.empty((n_q, k), dtype=torch.int32, device="cuda"), torch.empty((n_q, k), dtype=torch.int64, device="cuda"))
        fn = lambda: m.topk_device(dr, dq, k, None, 0, form, ws, o)
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    t = min(ts) / 1e3
    print(f"{form:10s} {mode:5s} {n_r}x{n_q}x{L}: {t*1e3:9.3f} ms  {n_r*n_q/t:.3e} cmp/s  {n_r*n_q*L/t:.3e} bitpairs/s", flush=True)


if __name__ == "__main__":
    forms = sys.argv[1].split(",") if len(sys.argv) > 1 else ["popc"]
    if len(sys.argv) > 2:
        mode = sys.argv[2]
        n_r, n_q, L = (int(x) for x in sys.argv[3:6])
        reps = int(sys.argv[6]) if len(sys.argv) > 6 else 5
        for f in forms:
            run(f, mode, n_r, n_q, L, reps=reps)
    else:
        for f in forms:
            run(f, "full", 1_000_000, 2048, 1024)
            run(f, "topk", 2_000_000, 2048, 1024)
            run(f, "topk", 20_000_000, 2048, 1024, reps=2)
