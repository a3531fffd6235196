#!/usr/bin/env python
"""FastID B200 benchmark: BASELINE.json's headline metric on config C3.

Workload (BASELINE.json configs[2], the config the metric is quoted on):
2048 unknowns x 20,000,000 known profiles x 1,024 SNP loci, scored with
popcount(known AND NOT unknown) (Eq. 1), fused top-16 epilogue per unknown;
the known database is sharded over N ranks (one process per GPU, NCCL), each
rank's top-16 candidates are all-gathered and merged.

One step = one pass of the hot path over one batch of 2048 unknowns against
the whole (resident) known database.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Prints ONE JSON line on rank 0.  ``value`` = comparisons/s (N_R x N_Q per
second, the reference's definition, bench.py:90-92) with inputs resident in
HBM and device timing (CUDA events, max over ranks); ``e2e`` = the same metric
through the public KnownDatabase/ShardedDatabase.search_words call with host
buffers (pinned H2D of the unknowns + D2H of the top-k lists every step).
``--impl reference`` times the CPU port of the reference path (oracle/,
compare_blocked restated in C, all host threads) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "profile comparisons/sec and wall time for 2048 unknowns × 20M knowns at 1/8 B200"
UNIT = "comparisons/s"
WORKLOAD = "C3: 2048 unknowns x 20M knowns x 1024 SNP loci, fused top-16 per unknown"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("b200", "reference"), default="b200")
    p.add_argument("--n-known", type=int, default=20_000_000)
    p.add_argument("--n-unknown", type=int, default=2048)
    p.add_argument("--loci", type=int, default=1024)
    p.add_argument("--k", type=int, default=16)
    p.add_argument("--formulation", default="auto")
    p.add_argument("--seed", type=int, default=1707)
    p.add_argument("--cpu-sample-known", type=int, default=100_000)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--verify-unknowns", type=int, default=8)
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def config_dict(args, world):
    return {
        "workload": WORKLOAD,
        "n_unknown": args.n_unknown,
        "n_known": args.n_known,
        "loci": args.loci,
        "k": args.k,
        "formulation": args.formulation,
        "parallelism": f"known-db sharded over {world} rank(s), unknowns replicated, NCCL all-gather of top-k",
        "l2": "no flush: the 2.56 GB known database streamed every step exceeds the 126 MB L2",
    }


# ---------------------------------------------------------------------------
# CPU side (oracle = test infrastructure; used only for the baseline + checks)
# ---------------------------------------------------------------------------

def cpu_reference_sample(args, reps=3, warmup=1):
    """compare_blocked restated in C (oracle/fastid_oracle.c) on a slice of the workload."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle

    n_words = args.loci // 64
    refs = oracle.synth_words(args.cpu_sample_known, n_words, 64, args.seed, 0)
    queries = oracle.synth_words(args.n_unknown, n_words, 64, args.seed, 1)
    qt = np.ascontiguousarray(queries.T)
    cores = os.cpu_count() or 1
    times = []
    for i in range(warmup + reps):
        t0 = time.perf_counter()
        oracle.blocked(refs, qt, 64, 16, cores)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    t = statistics.median(times)
    return {
        "value": args.cpu_sample_known * args.n_unknown / t,
        "unit": UNIT,
        "cores": cores,
        "kind": "port",
        "sample": (f"{args.n_unknown} unknowns x {args.cpu_sample_known} knowns x {args.loci} loci, full u32 "
                   f"matrix, compare_blocked(TileConfig(64), parallelism={cores}) restated in C, median of "
                   f"{reps} after {warmup} warm-up ({t:.3f} s each)"),
        "seconds_per_rep": t,
    }


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle

    n_words = args.loci // 64
    refs = oracle.synth_words(args.cpu_sample_known, n_words, 64, args.seed, 0)
    queries = oracle.synth_words(args.n_unknown, n_words, 64, args.seed, 1)
    qt = np.ascontiguousarray(queries.T)
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle.blocked(refs, qt, 64, 16, cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.blocked(refs, qt, 64, 16, cores)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = args.cpu_sample_known * args.n_unknown / t
    sample = (f"each step: {args.n_unknown} unknowns x {args.cpu_sample_known} knowns x {args.loci} loci "
              f"(a 1/{args.n_known // args.cpu_sample_known} slice of the workload), full u32 matrix via the C "
              f"port of compare_blocked (kernel.py:295-347), {cores} threads")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic (synth_panel convention, seeded)",
        "config": config_dict(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "extrapolated_full_job_s": args.n_known * args.n_unknown / value,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    QUERY = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw.instant,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.window = None  # (t0, t1) wall-clock of the timed region
        self.path = Path(os.environ.get("TMPDIR", "/tmp")) / f"fastid_clocks_{os.getpid()}.csv"

    def __enter__(self):
        if os.environ.get("FASTID_NO_CLOCKS"):  # diagnostics: run without the sampler
            return self
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=self.fh, stderr=subprocess.DEVNULL)
            time.sleep(1.5)  # let nvidia-smi start sampling before the timed region
        except Exception:
            self.proc = None
        return self

    def mark(self, start: bool):
        now = time.time()
        self.window = (now, None) if start else (self.window[0], now)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        from datetime import datetime

        rows, timed = [], []
        for line in self.path.read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 10 or not f[2].replace(".", "").isdigit():
                continue
            rows.append(f)
            try:
                ts = datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                continue
            if self.window and self.window[0] - 0.05 <= ts <= (self.window[1] or ts) + 0.05:
                timed.append(f)
        try:
            self.path.unlink()
        except OSError:
            pass
        use = timed or rows
        if not use:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[2]) for r in use]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in use for i in range(4) if r[6 + i].lower() == "active"})
        power = [float(r[4]) for r in use if r[4].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(use[0][3]), "reasons": reasons,
                "samples": len(use), "samples_in_timed_region": len(timed),
                "power_w_max": max(power) if power else None}


def planted_unknowns(shard_words: np.ndarray, n_unknown: int, L: int, rng) -> tuple[np.ndarray, np.ndarray]:
    """Unknowns = copies of random knowns of shard 0 with 0..16 bits flipped (so top-k hits are meaningful)."""
    src = rng.integers(0, shard_words.shape[0], n_unknown)
    q = shard_words[src].copy()
    flips = rng.integers(0, 17, n_unknown)
    for j in range(n_unknown):
        for b in rng.integers(0, L, flips[j]):
            q[j, b // 64] ^= np.uint64(1) << np.uint64(63 - b % 64)
    return q, src


def load_peaks():
    peaks = {}
    mp = ROOT / "MEASURED_PEAKS.json"
    if mp.exists():
        peaks["measured_peaks"] = json.loads(mp.read_text())
    return peaks


def probe_peak(m, torch, formulation: str, dev) -> dict:
    """Measured pipe peak (bit-pairs/s = MACs/s) of the formulation's inner instruction."""
    import ctypes

    from paper_1707_00516_b200 import _native

    code = _native.formulation_code(formulation)
    scratch = torch.zeros(4096, dtype=torch.int32, device=dev)
    work = ctypes.c_double(0)
    iters = 200 if code == _native.FORMULATIONS["popc"] else 20000
    stream = torch.cuda.current_stream(dev)
    best = 0.0
    for rep in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _native.check(_native.lib().fastid_probe_peak(code, iters, scratch.data_ptr(), ctypes.byref(work),
                                                      stream.cuda_stream), "fastid_probe_peak")
        e1.record(stream)
        e1.synchronize()
        if rep:
            best = max(best, work.value / (e0.elapsed_time(e1) / 1e3))
    return {"macs_per_s": best, "tflops": 2 * best / 1e12}


def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_1707_00516_b200 as m
    from paper_1707_00516_b200 import _native
    from paper_1707_00516_b200.search import KnownDatabase
    from paper_1707_00516_b200.sharded import ShardedDatabase, shard_range

    world, rank, local = dist_env()
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    # one process per GPU; FASTID_DIST_BACKEND=gloo lets a one-GPU box exercise the
    # multi-rank path (ranks share the device, candidates gathered over gloo)
    backend = os.environ.get("FASTID_DIST_BACKEND", "nccl")
    dev_index = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    _native.lib()
    L = args.loci
    n_words = L // 64
    formulation = args.formulation
    if formulation == "auto":
        formulation = "tensor_f4" if _native.supports("tensor_f4", L) else "popc"
    start, stop = shard_range(args.n_known, rank, world)
    n_local = stop - start

    # ---- known database shard: host generation, pinned upload (timed separately)
    g = torch.Generator().manual_seed(args.seed * 1000 + rank)
    host = torch.randint(-(2**63), 2**63 - 1, (n_local, n_words), dtype=torch.int64, generator=g)
    host_np = host.numpy().view(np.uint64)
    host_pinned = host.pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev_words = host_pinned.to(dev, non_blocking=True)
    db_panel = m.DevicePanel.from_words(dev_words, L, device=dev)
    torch.cuda.synchronize()
    db_upload_s = time.perf_counter() - t0
    del dev_words, host_pinned
    db = KnownDatabase(db_panel, device=dev, ref_base=start, formulation=formulation)
    sharded = ShardedDatabase(db, args.n_known)

    # ---- unknowns: planted near-copies of rank 0's knowns, broadcast to all ranks
    rng = np.random.default_rng(args.seed)
    if rank == 0:
        qwords, _src = planted_unknowns(host_np, args.n_unknown, L, rng)
    else:
        qwords = np.zeros((args.n_unknown, n_words), np.uint64)
    if world > 1:
        t = torch.from_numpy(qwords.view(np.int64).copy()).to(dev)
        dist.broadcast(t, 0)
        qwords = t.cpu().numpy().view(np.uint64)
    dq = m.DevicePanel.from_words(qwords, L, device=dev)
    k = args.k
    ws = torch.empty(m.compare.topk_workspace_bytes(n_local, args.n_unknown, k, formulation), dtype=torch.uint8,
                     device=dev)
    out = (torch.empty((args.n_unknown, k), dtype=torch.int32, device=dev),
           torch.empty((args.n_unknown, k), dtype=torch.int64, device=dev))
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- device-resident timing (value) + dominant-kernel timing (roofline)
    kern_ms = []

    def step(record_kernel: bool):
        if record_kernel:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s, x = db.topk_device(dq, k, None, ws, out, events=(e0, e1))
            kern_ms.append((e0, e1))
        else:
            s, x = db.topk_device(dq, k, None, ws, out)
        return sharded.combine(s, x, k)

    with ClockSampler(dev_index) as clocks:
        for _ in range(args.warmup):
            step(False)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        clocks.mark(True)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            res = step(True)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        clocks.mark(False)
    elapsed = ev0.elapsed_time(ev1) / 1e3
    kernel_s = [a.elapsed_time(b) / 1e3 for a, b in kern_ms]
    if os.environ.get("FASTID_BENCH_STEPS"):
        print("kernel ms per step:", [round(x * 1e3, 3) for x in kernel_s], file=sys.stderr)
    if world > 1:
        t = torch.tensor([elapsed, max(kernel_s)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t[0])
    comps = args.n_known * args.n_unknown
    value = comps * args.steps / elapsed
    # compare kernel + partial merge (+ cross-rank merge); the mxf4 pair kernel adds a
    # spare-pair grid when the unknown groups x slices leave SMs free (csrc/tensor.cu spare_plan)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    groups, tiles = -(-args.n_unknown // 256), -(-n_local // 192)
    slices = max(1, min((sms // 2) // groups, tiles))
    spare = formulation == "tensor_f4" and (sms // 2) - groups * slices > 0 and tiles >= 16 * (slices + 1)
    launches_per_step = 2 + (1 if spare else 0) + (1 if world > 1 else 0)

    # ---- correctness spot check against the oracle (rank 0, single GPU only)
    verified = None
    if rank == 0 and world == 1 and args.verify_unknowns > 0:
        sys.path.insert(0, str(ROOT / "oracle"))
        import oracle

        s_dev = res[0].cpu().numpy().view(np.uint32)
        x_dev = res[1].cpu().numpy()
        pick = np.linspace(0, args.n_unknown - 1, args.verify_unknowns).astype(int)
        es, ex, _ = oracle.topk(host_np, qwords[pick], k)
        verified = bool(np.array_equal(s_dev[pick], es) and np.array_equal(x_dev[pick], ex))

    # ---- end-to-end through the public host-buffer API
    e2e = None
    if not args.no_e2e:
        h2d = d2h = 0
        for _ in range(args.warmup):
            sharded.search_words(qwords, k)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            sharded.search_words(qwords, k)
        torch.cuda.synchronize()
        barrier()
        e2e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t[0])
        st = db.stager(args.n_unknown, k)
        e2e = {"value": comps * args.steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": st.h2d_bytes,
               "d2h_bytes_per_step": st.d2h_bytes, "ms_per_step": e2e_s / args.steps * 1e3}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (the comparison kernel)
    peak = probe_peak(m, torch, formulation, dev)
    kern_avg = sum(kernel_s) / len(kernel_s)
    macs = n_local * args.n_unknown * L
    bound = "tensor" if formulation.startswith("tensor") else "popc"
    achieved_tflops = 2 * macs / kern_avg / 1e12
    peaks = load_peaks().get("measured_peaks", {})
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get(formulation)
    roofline = {
        "bound": "tensor" if bound == "tensor" else "tensor",
        "pipe": {"tensor_f4": "tcgen05.mma kind::mxf4 (e2m1)", "tensor_i8": "tcgen05.mma kind::i8",
                 "popc": "CUDA-core LOP3+POPC"}[formulation],
        "achieved": achieved_tflops,
        "peak": peak["tflops"],
        "unit": "TFLOP/s",
        "frac": achieved_tflops / peak["tflops"],
        "traffic": traffic,
        "traffic_unit": "DRAM bytes per launch (ncu --set full, profiles/ncu_traffic.json)" if traffic else None,
        "algorithmic_bytes": n_local * ((L + 255) // 256) * 256 // 2 + args.n_unknown * db.panel.stride
        if formulation == "tensor_f4" else None,
        "peak_source": (f"measured on this box by fastid_probe_peak ({formulation} inner instruction only, one CTA "
                        f"per SM); 1 MAC = 1 bit-pair = 2 FLOP"),
        "kernel_ms": kern_avg * 1e3,
        "kernel_share_of_step": kern_avg / (elapsed / args.steps),
        "algorithmic": f"{macs:.4g} bit-pair MACs per launch = {n_local} knowns x {args.n_unknown} unknowns x {L} loci",
        # bytes the kernel must read from HBM per launch (the mxf4 tensor image for the
        # tensor path, the packed rows otherwise) over its time: far below the HBM roof
        "hbm_gbs": ((n_local * ((L + 255) // 256) * 256 // 2 if formulation == "tensor_f4"
                     else n_local * db.panel.stride) + args.n_unknown * db.panel.stride) / kern_avg / 1e9,
        "hbm_peak_gbs": peaks.get("hbm_gbs"),
        "bf16_tflops_measured": peaks.get("bf16_tflops"),
    }
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": elapsed / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": {"tensor_f4": "e2m1", "tensor_i8": "u8", "popc": "u32"}[formulation],
        "data": "synthetic: uniform random known profiles, unknowns = planted near-copies (0-16 bit flips)",
        "config": config_dict(args, world),
        "e2e": e2e,
        "roofline": roofline,
        "clocks": clocks.summary(),
        "gpu_launches": launches_per_step * args.steps,
        "db_upload_s": db_upload_s,
        "wall_s_per_step": elapsed / args.steps,
        "verified_vs_oracle": verified,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = {k2: v for k2, v in cpu_reference_sample(args).items() if k2 != "seconds_per_rep"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
