"""MMA stream + concurrent TMEM reads: MMA efficiency and TMEM-read B/clk per SM."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1707_00516_b200 import _native
L = _native.lib()
iters = 20000
for readers in (0, 4, 8, 15):
    sink = torch.zeros(2 * 148, dtype=torch.int64, device="cuda")
    _native.check(L.fastid_probe_contention(iters, readers, sink.data_ptr(), torch.cuda.current_stream().cuda_stream), "p")
    torch.cuda.synchronize()
    s = sink.cpu().numpy().reshape(148, 2)
    cyc = s[:, 1].astype(float)
    mma_eff = (iters * 112.0) / cyc  # 112 cycles per 128x224x64 mxf4 MMA at peak
    print(f"readers {readers:2d}: MMA efficiency {mma_eff.mean():.3f}  TMEM read {(s[:,0]/cyc).mean():7.1f} B/clk/SM", flush=True)
