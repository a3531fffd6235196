"""Tensor-pipe probe: single-CTA vs CTA-pair mxf4 MMA throughput (resident operands)."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1707_00516_b200 import _native

L = _native.lib()
scratch = torch.zeros(4096, dtype=torch.int32, device="cuda")
src = torch.zeros(1 << 30, dtype=torch.uint8, device="cuda")
B = 268
names = {}
for nflag, n in ((128, "N=192"), (1024, "N=144"), (8192, "N=96")):
    for extra, nm in ((0, "plain"), (64 + 512, "wait+commit/4"), (64 + 512 + 2048, "wait+commit/8"),
                      (64 + 512 + 4096, "wait+commit/4 3buf"), (64 + 512 + 2048 + 4096, "wait+commit/8 3buf")):
        if nflag == 128 and extra & 4096:
            continue
        if nflag == 8192 and extra not in (0, 64 + 512):
            continue
        names[B + nflag + extra] = f"pair {n} tiled {nm}"
for nflag, n in ((128, "N=192"), (8192, "N=96"), (16, "N=256")):
    names[8 + 4 + 32 + nflag] = f"pair {n} 2 accumulators alternating, random operands"
for variant, name in names.items():
    best = 0
    for rep in range(4):
        work = ctypes.c_double(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _native.check(L.fastid_probe_variant(_native.formulation_code("tensor_f4"), variant, 40000,
                                             scratch.data_ptr(), src.data_ptr(), src.numel(), ctypes.byref(work),
                                             torch.cuda.current_stream().cuda_stream), "probe")
        e1.record(); e1.synchronize()
        if rep:
            best = max(best, work.value / (e0.elapsed_time(e1) / 1e3))
    print(f"{name:28s}: {2*best/1e12:8.1f} TFLOP/s-equiv", flush=True)
