"""Tensor-pipe probe variants: alternating vs single accumulator, with/without bulk-copy smem traffic."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1707_00516_b200 import _native

L = _native.lib()
scratch = torch.zeros(4096, dtype=torch.int32, device="cuda")
src = torch.zeros(2 << 30, dtype=torch.uint8, device="cuda")
for form in ("tensor_f4", "tensor_i8"):
    for variant in (0, 1, 4, 5, 6):
        work = ctypes.c_double(0)
        best = 0
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _native.check(L.fastid_probe_variant(_native.formulation_code(form), variant, 20000, scratch.data_ptr(),
                                                 src.data_ptr(), src.numel(), ctypes.byref(work),
                                                 torch.cuda.current_stream().cuda_stream), "probe")
            e1.record(); e1.synchronize()
            if rep:
                best = max(best, work.value / (e0.elapsed_time(e1) / 1e3))
        print(f"{form} variant {variant}: {2*best/1e12:8.1f} TFLOP/s-equiv ({best:.3e} MAC/s)", flush=True)
