"""TMEM read throughput (bytes/clk/SM) for tcgen05.ld 32x32b at several widths and warp counts."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1707_00516_b200 import _native
L = _native.lib()
scratch = torch.zeros(4096, dtype=torch.int32, device="cuda")
clk = torch.cuda.clock_rate() if hasattr(torch.cuda, "clock_rate") else 1965
for x in (8, 32, 64):
    for warps in (4, 8, 16):
        work = ctypes.c_double(0); best = 0
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _native.check(L.fastid_probe_tmem_read(x, warps, 20000, scratch.data_ptr(), ctypes.byref(work),
                                                   torch.cuda.current_stream().cuda_stream), "probe")
            e1.record(); e1.synchronize()
            if rep: best = max(best, work.value / (e0.elapsed_time(e1) / 1e3))
        print(f"x{x:<3d} warps {warps:2d}: {best/1e12:7.2f} TB/s total = {best/148/1.965e9:7.1f} B/clk/SM @1965MHz", flush=True)
