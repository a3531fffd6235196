"""bench.py on the GPU at a reduced shape: the JSON contract of the B200 arm,
for the headline operator and for XOR (each verified against the C oracle over
every unknown x every known inside bench.py)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import gpu_available

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


@pytest.mark.parametrize("op", ["andnot", "xor"])
def test_bench_line_small_shape(op):
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3", "--n-known", "400000",
         "--n-unknown", "512", "--no-cpu-baseline", "--op", op],
        capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    for key in ("metric", "value", "unit", "n_gpus", "ms_per_step", "roofline", "e2e", "clocks", "gpu_launches",
                "verified_vs_oracle"):
        assert key in d, key
    assert d["verified_vs_oracle"]["ok"] is True and d["verified_vs_oracle"]["unknowns"] == 512
    assert d["config"]["operator"] == op
    assert d["gpu_launches"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert 0 < d["roofline"]["frac"] < 1.2
