"""bench.py's JSON contract for the reference arm (CPU-only, tiny sample)."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2", "--warmup", "1",
         "--cpu-sample-known", "3000", "--n-unknown", "256"],
        capture_output=True, text=True, timeout=300, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference"
    assert d["unit"] == "comparisons/s" and d["value"] > 0
    # the pip-installed reference (baseline/_ref) when importable, else the C port
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert "physical_cores" in d["cpu_baseline"] and "cpu_model" in d["cpu_baseline"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_reference_arm_non_zero_rank_is_silent():
    env = {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}
    import os

    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1"],
                         capture_output=True, text=True, timeout=120, cwd=str(ROOT), env={**os.environ, **env})
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_bench_spawns_its_own_ranks_for_the_reference_arm():
    """`--gpus N` without a launcher: the reference arm reports n_gpus = N and
    prints one line (only rank 0 works)."""
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
         "--warmup", "0", "--cpu-sample-known", "2000", "--n-unknown", "64"],
        capture_output=True, text=True, timeout=300, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["n_gpus"] == 2


def test_spawn_ranks_sets_the_launcher_environment(tmp_path):
    """bench.spawn_ranks gives every child the torchrun variables on 127.0.0.1."""
    sys.path.insert(0, str(ROOT))
    import bench

    script = tmp_path / "probe.py"
    script.write_text("import os,sys\n"
                      "print(os.environ['RANK'], os.environ['WORLD_SIZE'], os.environ['LOCAL_RANK'],"
                      " os.environ['MASTER_ADDR'], sys.argv[1:], flush=True)\n")
    old = bench.__file__
    try:
        bench.__file__ = str(script)
        rc = bench.spawn_ranks(3, ["--x"])
    finally:
        bench.__file__ = old
    assert rc == 0


def test_reference_arm_has_no_xor():
    """`--op xor` is a library extension: the reference arm says it is unavailable."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--op", "xor",
                          "--steps", "1"], capture_output=True, text=True, timeout=120, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][0])
    assert d["impl"] == "reference" and "AND-NOT" in d["unavailable"]
