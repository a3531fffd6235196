#!/usr/bin/env python
"""FastID B200 benchmark: BASELINE.json's headline metric.

Workloads (BASELINE.json configs):

* ``C3`` (default; configs[2], the config the metric is quoted on): 2048
  unknowns x 20,000,000 known profiles x 1,024 SNP loci, scored with
  popcount(known AND NOT unknown) (Eq. 1), fused top-16 epilogue per unknown.
* ``C4`` (configs[3]): 512 synthetic 2-5-contributor mixtures x 20M knowns x
  5,000 loci, AND-NOT exclusion counts, fused top-16 per mixture.

The known database is sharded over N ranks (one process per GPU, NCCL); each
rank's top-k candidates are all-gathered and merged.  One step = one pass of
the hot path over one batch of unknowns against the whole (resident) known
database.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload C3|C4] [--verify full|sample|none]

``--gpus N`` without a torchrun environment spawns the N ranks itself
(RANK / WORLD_SIZE / MASTER_* set per child, 127.0.0.1).  Prints ONE JSON line
on rank 0.  ``value`` = comparisons/s (N_R x N_Q per second, the reference's
definition, bench.py:90-92) with inputs resident in HBM and device timing (CUDA
events, max over ranks); ``e2e`` = the same metric through the public
ShardedDatabase.search_words call with host buffers (pinned H2D of the
unknowns + D2H of the top-k lists every step).  After timing, rank 0 checks
the last step's global top-k against the CPU oracle (``--verify full``: every
unknown against every known).  ``--impl reference`` times the reference's own
CPU implementation (the pip-installed reference in baseline/_ref when
importable, else the C port of compare_blocked in oracle/) on a bounded slice.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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

WORKLOADS = {
    "C3": dict(n_known=20_000_000, n_unknown=2048, loci=1024, k=16,
               desc="C3: 2048 unknowns x 20M knowns x 1024 SNP loci, fused top-16 per unknown",
               data="synthetic: uniform random known profiles, unknowns = planted near-copies (0-16 bit flips)"),
    "C4": dict(n_known=20_000_000, n_unknown=512, loci=5000, k=16,
               desc=("C4: 512 mixtures (2-5 contributors) x 20M knowns x 5000 SNP loci, AND-NOT exclusion "
                     "counts, fused top-16 per mixture"),
               data=("synthetic: known profiles with per-locus minor-allele presence p ~ U(0.1, 0.5); "
                     "unknowns = bitwise OR of 2-5 known contributors")),
}


def parse_args(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("b200", "reference"), default="b200")
    p.add_argument("--workload", choices=tuple(WORKLOADS), default="C3")
    p.add_argument("--n-known", type=int, default=None)
    p.add_argument("--n-unknown", type=int, default=None)
    p.add_argument("--loci", type=int, default=None)
    p.add_argument("--k", type=int, default=None)
    p.add_argument("--formulation", default="auto")
    # the bitwise operator before the popcount: "andnot" is the reference's Eq. 1 (the
    # headline); "and" / "xor" are the library's operator extensions (no reference arm)
    p.add_argument("--op", choices=("andnot", "and", "xor"), default="andnot")
    p.add_argument("--seed", type=int, default=1707)
    p.add_argument("--cpu-sample-known", type=int, default=100_000)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--verify", choices=("full", "sample", "none"), default="full")
    p.add_argument("--no-e2e", action="store_true")
    args = p.parse_args(argv)
    w = WORKLOADS[args.workload]
    for key in ("n_known", "n_unknown", "loci", "k"):
        if getattr(args, key) is None:
            setattr(args, key, w[key])
    return args


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def config_dict(args, world):
    full = (args.n_known, args.n_unknown, args.loci, args.k) == tuple(
        WORKLOADS[args.workload][x] for x in ("n_known", "n_unknown", "loci", "k"))
    return {
        "workload": WORKLOADS[args.workload]["desc"] if full else
        f"{args.workload} shape override: {args.n_unknown} unknowns x {args.n_known} knowns x {args.loci} loci, "
        f"top-{args.k}",
        "n_unknown": args.n_unknown,
        "n_known": args.n_known,
        "loci": args.loci,
        "k": args.k,
        "formulation": args.formulation,
        "operator": args.op,
        "parallelism": f"known-db sharded over {world} rank(s), unknowns replicated, NCCL all-gather of top-k",
        "l2": (f"no flush: the {args.n_known * -(-args.loci // 128) * 16 / 1e9:.2f} GB packed known database "
               "(and its larger tensor image) streamed every step exceeds the 126 MB L2"),
    }


def host_cpu():
    """CPU model, logical threads and physical cores of this host (lscpu)."""
    info = {"logical_cpus": os.cpu_count() or 1, "model": None, "physical_cores": None}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                a, b = line.split(":", 1)
                kv[a.strip()] = b.strip()
        info["model"] = kv.get("Model name")
        cps, sockets = kv.get("Core(s) per socket"), kv.get("Socket(s)")
        if cps and sockets and cps.isdigit() and sockets.isdigit():
            info["physical_cores"] = int(cps) * int(sockets)
    except Exception:
        pass
    return info


# ---------------------------------------------------------------------------
# CPU side (oracle/ and the reference = test infrastructure: baseline + checks)
# ---------------------------------------------------------------------------

def _oracle():
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle

    return oracle


def _reference_module():
    """The unmodified reference package, pip-installed into baseline/_ref
    (DESIGN.md "Reference arm"), or None when it is not importable here."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "fastid" / "kernel.py").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", str(Path(os.environ.get("TMPDIR", "/tmp")) / "fastid_numba_cache"))
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import fastid.kernel as K

        return K
    except Exception as e:  # numba missing, etc.
        print(f"reference package not importable: {e}", file=sys.stderr)
        return None


def _cpu_sample(args):
    """The bounded CPU sample: args.cpu_sample_known knowns x all unknowns at the
    workload's loci, synth_panel inputs (reference bench.py:41-54), padding masked."""
    oracle = _oracle()
    n_words = -(-args.loci // 64)
    refs = oracle.mask_padding(oracle.synth_words(args.cpu_sample_known, n_words, 64, args.seed, 0), args.loci)
    queries = oracle.mask_padding(oracle.synth_words(args.n_unknown, n_words, 64, args.seed, 1), args.loci)
    return refs, queries


def _time_reps(fn, reps, warmup):
    for _ in range(warmup):
        fn()
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    return statistics.median(times), times


def cpu_reference_sample(args, reps=3, warmup=1, prefer_reference=True):
    """compare_blocked(refs, relayout_queries(q), TileConfig(64), parallelism=cores) -- the
    reference's CLI default (cli.py:202-203) -- on the bounded slice: the reference
    package itself when importable (kind "reference"), else its C restatement
    (kind "port").  Median of `reps` after `warmup` (reference bench.py:129-154)."""
    oracle = _oracle()
    refs, queries = _cpu_sample(args)
    cores = os.cpu_count() or 1
    K = _reference_module() if prefer_reference else None
    qt = np.ascontiguousarray(queries.T)
    port_t, _ = _time_reps(lambda: oracle.blocked(refs, qt, 64, 16, cores), reps, warmup)
    kind, t = "port", port_t
    what = "compare_blocked restated in C (oracle/fastid_oracle.c)"
    ref_t = None
    if K is not None:
        rp = K.Panel(tuple(f"r{i}" for i in range(refs.shape[0])), refs, args.loci)
        qp = K.relayout_queries(K.Panel(tuple(f"q{j}" for j in range(queries.shape[0])), queries, args.loci))
        ref_t, _ = _time_reps(lambda: K.compare_blocked(rp, qp, K.TileConfig(64), cores), reps, warmup)
        kind, t = "reference", ref_t
        what = "the reference package (baseline/_ref, numba) compare_blocked"
    cpu = host_cpu()
    out = {
        "value": args.cpu_sample_known * args.n_unknown / t,
        "unit": UNIT,
        "cores": cores,
        "kind": kind,
        "sample": (f"{args.n_unknown} unknowns x {args.cpu_sample_known} knowns x {args.loci} loci, full u32 matrix, "
                   f"{what}(TileConfig(64), parallelism={cores}), median of {reps} after {warmup} warm-up "
                   f"({t:.3f} s each); host {cpu['model']}, {cpu['physical_cores']} physical cores / "
                   f"{cpu['logical_cpus']} threads"),
        "cpu_model": cpu["model"],
        "physical_cores": cpu["physical_cores"],
        "port_value": args.cpu_sample_known * args.n_unknown / port_t,
        "seconds_per_rep": t,
    }
    if ref_t is not None:
        out["reference_value"] = args.cpu_sample_known * args.n_unknown / ref_t
    return out


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    if args.op != "andnot":
        print(json.dumps({"impl": "reference", "unavailable": f"the reference computes AND-NOT only (kernel.py:33-35), "
                          f"not {args.op}"}))
        return 0
    world = max(world, args.gpus)
    oracle = _oracle()
    refs, queries = _cpu_sample(args)
    cores = os.cpu_count() or 1
    K = _reference_module()
    if K is not None:
        rp = K.Panel(tuple(f"r{i}" for i in range(refs.shape[0])), refs, args.loci)
        qp = K.relayout_queries(K.Panel(tuple(f"q{j}" for j in range(queries.shape[0])), queries, args.loci))
        t, _ = _time_reps(lambda: K.compare_blocked(rp, qp, K.TileConfig(64), cores), args.steps, args.warmup)
        kind = "reference"
        what = "the unmodified reference package (baseline/_ref, numba) compare_blocked(TileConfig(64))"
    else:
        qt = np.ascontiguousarray(queries.T)
        t, _ = _time_reps(lambda: oracle.blocked(refs, qt, 64, 16, cores), args.steps, args.warmup)
        kind = "port"
        what = "the C port of compare_blocked (kernel.py:295-347, oracle/fastid_oracle.c)"
    value = args.cpu_sample_known * args.n_unknown / t
    cpu = host_cpu()
    sample = (f"each step: {args.n_unknown} unknowns x {args.cpu_sample_known} knowns x {args.loci} loci "
              f"(a 1/{args.n_known // args.cpu_sample_known} slice of the workload), full u32 matrix via {what}, "
              f"parallelism={cores}; median of {args.steps} steps after {args.warmup} warm-up; host {cpu['model']}, "
              f"{cpu['physical_cores']} physical cores / {cpu['logical_cpus']} threads")
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
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample,
                         "cpu_model": cpu["model"], "physical_cores": cpu["physical_cores"]},
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


# ---- synthetic inputs --------------------------------------------------------

def c3_shard_words(seed: int, rank: int, n_local: int, n_words: int) -> np.ndarray:
    """Rank `rank`'s C3 shard: uniform random words (torch CPU generator, seed*1000+rank)."""
    import torch

    g = torch.Generator().manual_seed(seed * 1000 + rank)
    host = torch.randint(-(2**63), 2**63 - 1, (n_local, n_words), dtype=torch.int64, generator=g)
    return host.numpy().view(np.uint64)


def c4_locus_presence(seed: int, loci: int) -> np.ndarray:
    """Per-locus minor-allele presence p ~ U(0.1, 0.5)."""
    return np.random.default_rng([seed, 4, loci]).uniform(0.1, 0.5, loci).astype(np.float32)


def c4_shard_panel(m, seed: int, rank: int, n_local: int, loci: int, dev, chunk: int = 1 << 18):
    """Rank `rank`'s C4 shard, generated on the device: bit (i, l) = [u < p_l] with u
    from a CUDA Philox generator seeded seed*1000+rank (the same stream on any
    device), packed MSB-first by the library's encoder (fastid_pack_bits)."""
    import torch

    from paper_1707_00516_b200 import _native

    p = torch.from_numpy(c4_locus_presence(seed, loci)).to(dev)
    g = torch.Generator(device=dev).manual_seed(seed * 1000 + rank)
    panel = m.DevicePanel.empty(n_local, loci, 64, dev)
    stream = torch.cuda.current_stream(dev)
    for r0 in range(0, n_local, chunk):
        rows = min(chunk, n_local - r0)
        bits = (torch.rand((rows, loci), generator=g, device=dev) < p).to(torch.uint8)
        _native.check(_native.lib().fastid_pack_bits(
            bits.data_ptr(), rows, loci, 64, panel.rows[r0:].data_ptr(), panel.stride, stream.cuda_stream),
            "fastid_pack_bits")
        del bits
    torch.cuda.synchronize(dev)
    return panel


def planted_unknowns(shard_words: np.ndarray, n_unknown: int, L: int, rng) -> np.ndarray:
    """C3 unknowns = copies of random knowns of shard 0 with 0..16 bits flipped (meaningful top-k)."""
    src = rng.integers(0, shard_words.shape[0], n_unknown)
    q = shard_words[src].copy()
    flips = rng.integers(0, 17, n_unknown)
    for j in range(n_unknown):
        for b in rng.integers(0, L, flips[j]):
            q[j, b // 64] ^= np.uint64(1) << np.uint64(63 - b % 64)
    return q


def mixture_unknowns(panel, n_unknown: int, rng) -> np.ndarray:
    """C4 unknowns = bitwise OR of 2-5 known contributors of shard 0 (contributors score 0)."""
    import torch

    out = np.zeros((n_unknown, panel.n_words), np.uint64)
    for j in range(n_unknown):
        idx = rng.choice(panel.n_profiles, int(rng.integers(2, 6)), replace=False)
        rows = panel.rows[torch.from_numpy(np.sort(idx)).to(panel.device)]
        words = rows[:, : panel.n_words * 8].contiguous().cpu().numpy().view(np.uint64)
        out[j] = np.bitwise_or.reduce(words, axis=0)
    return out


def load_peaks():
    mp = ROOT / "MEASURED_PEAKS.json"
    return json.loads(mp.read_text()) if mp.exists() else {}


def probe_peak(torch, formulation: str, dev) -> dict:
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
    lib = _native.lib()
    L = args.loci
    n_words = -(-L // 64)
    formulation = args.formulation
    if formulation == "auto":
        formulation = "tensor_f4" if _native.supports("tensor_f4", L) else "popc"
    start, stop = shard_range(args.n_known, rank, world)
    n_local = stop - start
    k = args.k

    # ---- known database shard (built once; timed separately)
    host_np = None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if args.workload == "C4":
        db_panel = c4_shard_panel(m, args.seed, rank, n_local, L, dev)
        db_build = "generated on the device (Philox uniforms vs per-locus p, packed by fastid_pack_bits)"
    else:
        host_np = c3_shard_words(args.seed, rank, n_local, n_words)
        t0 = time.perf_counter()  # the upload alone
        host_pinned = torch.from_numpy(host_np.view(np.int64)).pin_memory()
        dev_words = host_pinned.to(dev, non_blocking=True)
        db_panel = m.DevicePanel.from_words(dev_words, L, device=dev)
        del dev_words, host_pinned
        db_build = "pinned H2D upload of the host-generated shard + fastid_load_words"
    torch.cuda.synchronize()
    db_upload_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    db = KnownDatabase(db_panel, device=dev, ref_base=start, formulation=formulation, op=args.op)
    torch.cuda.synchronize()
    db_prepare_s = time.perf_counter() - t0
    sharded = ShardedDatabase(db, args.n_known)

    # ---- unknowns: built on rank 0 from its shard, broadcast to all ranks
    rng = np.random.default_rng(args.seed)
    if rank == 0:
        if args.workload == "C4":
            qwords = mixture_unknowns(db_panel, args.n_unknown, rng)
        else:
            qwords = planted_unknowns(host_np, args.n_unknown, L, rng)
    else:
        qwords = np.zeros((args.n_unknown, n_words), np.uint64)
    if world > 1:
        t = torch.from_numpy(qwords.view(np.int64).copy())
        t = t.to(dev) if backend == "nccl" else t
        dist.broadcast(t, 0)
        qwords = t.cpu().numpy().view(np.uint64)
    dq = m.DevicePanel.from_words(qwords, L, device=dev)
    ws = torch.empty(m.compare.topk_workspace_bytes(n_local, args.n_unknown, k, formulation), dtype=torch.uint8,
                     device=dev)
    out = (torch.empty((args.n_unknown, k), dtype=torch.int32, device=dev),
           torch.empty((args.n_unknown, k), dtype=torch.int64, device=dev))
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(values):
        if world == 1:
            return values
        t = torch.tensor(values, dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def sum_over_ranks(value):
        if world == 1:
            return value
        t = torch.tensor([value], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.item()

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
        launches0 = lib.fastid_launch_count()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            res = step(True)
        ev1.record(stream)
        torch.cuda.synchronize()
        launches = lib.fastid_launch_count() - launches0
        barrier()
        torch.cuda.synchronize()
        clocks.mark(False)
    elapsed = ev0.elapsed_time(ev1) / 1e3
    kernel_s = [a.elapsed_time(b) / 1e3 for a, b in kern_ms]
    if os.environ.get("FASTID_BENCH_STEPS"):
        print("kernel ms per step:", [round(x * 1e3, 3) for x in kernel_s], file=sys.stderr)
    elapsed, kern_max = max_over_ranks([elapsed, sum(kernel_s) / len(kernel_s)])
    launches_total = int(sum_over_ranks(launches))
    comps = args.n_known * args.n_unknown
    value = comps * args.steps / elapsed
    s_dev = res[0].cpu().numpy().view(np.uint32).copy()
    x_dev = res[1].cpu().numpy().copy()

    # ---- end-to-end through the public host-buffer API
    e2e = None
    if not args.no_e2e:
        # the serving loop: every step copies its unknowns host->device and reads its
        # top-k lists back; step i+1 is staged and enqueued before step i's lists are
        # read back (ShardedDatabase.search_many), so host work overlaps device work
        for _ in sharded.search_many((qwords for _ in range(args.warmup)), k):
            pass
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for e2e_s_host, e2e_x_host in sharded.search_many((qwords for _ in range(args.steps)), k):
            pass
        torch.cuda.synchronize()
        barrier()
        e2e_s = max_over_ranks([time.perf_counter() - t0])[0]
        st = db.stager(args.n_unknown, k)
        e2e = {"value": comps * args.steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": st.h2d_bytes,
               "d2h_bytes_per_step": st.d2h_bytes, "ms_per_step": e2e_s / args.steps * 1e3,
               "call": "ShardedDatabase.search_many (pipelined: step i+1 staged before step i is read back)",
               "same_result_as_device_path": bool(np.array_equal(e2e_s_host, s_dev)
                                                  and np.array_equal(e2e_x_host, x_dev))}

    # ---- correctness against the CPU oracle (rank 0, outside every timed region):
    # rank 0 rebuilds every rank's shard from its seed and scans the whole database
    verified = None
    if args.verify != "none":
        if rank == 0:
            oracle = _oracle()
            t0 = time.perf_counter()
            shards = []
            for r in range(world):
                r0, r1 = shard_range(args.n_known, r, world)
                if r == rank and host_np is not None:
                    shards.append(host_np)
                elif args.workload == "C4":
                    p = db_panel if r == rank else c4_shard_panel(m, args.seed, r, r1 - r0, L, dev)
                    shards.append(p.to_words())
                    if r != rank:
                        del p
                        torch.cuda.empty_cache()
                else:
                    shards.append(c3_shard_words(args.seed, r, r1 - r0, n_words))
            refs_all = shards[0] if world == 1 else np.concatenate(shards)
            del shards
            gen_s = time.perf_counter() - t0
            pick = (np.arange(args.n_unknown) if args.verify == "full"
                    else np.unique(np.linspace(0, args.n_unknown - 1, 64).astype(int)))
            t0 = time.perf_counter()
            (es, ex, _), _ = oracle.scan(refs_all, qwords[pick], k, op=args.op)
            verify_s = time.perf_counter() - t0
            ok = bool(np.array_equal(s_dev[pick], es) and np.array_equal(x_dev[pick], ex))
            verified = {"ok": ok, "unknowns": int(len(pick)), "knowns": int(refs_all.shape[0]),
                        "oracle": "oracle.scan (oracle/fastid_oracle.c), all host threads",
                        "oracle_s": verify_s, "rebuild_s": gen_s}
            del refs_all
        barrier()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (the comparison kernel)
    peak = probe_peak(torch, formulation, dev)
    kern_avg = kern_max
    macs = n_local * args.n_unknown * L
    achieved_tflops = 2 * macs / kern_avg / 1e12
    peaks = load_peaks()
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        tr = json.loads(tfile.read_text())
        traffic = tr.get(f"{args.workload}:{formulation}", tr.get(formulation) if args.workload == "C3" else None)
    image_bytes = n_local * (-(-L // 256) * 256) // 2 if formulation == "tensor_f4" else n_local * db.panel.stride
    algo_bytes = image_bytes + args.n_unknown * db.panel.stride
    roofline = {
        "bound": "tensor" if formulation.startswith("tensor") else "alu",
        "pipe": {"tensor_f4": "tcgen05.mma kind::mxf4 (e2m1)", "tensor_i8": "tcgen05.mma kind::i8",
                 "popc": "CUDA-core LOP3+POPC"}[formulation],
        "achieved": achieved_tflops,
        "peak": peak["tflops"],
        "unit": "TFLOP/s",
        "frac": achieved_tflops / peak["tflops"],
        "traffic": traffic,
        "traffic_unit": "DRAM bytes per launch (ncu --set full, profiles/ncu_traffic.json)" if traffic else None,
        "algorithmic_bytes": algo_bytes,
        "peak_source": (f"measured on this box by fastid_probe_peak ({formulation} inner instruction only, one CTA "
                        f"per SM); 1 MAC = 1 bit-pair = 2 FLOP"),
        "kernel_ms": kern_avg * 1e3,
        "kernel_share_of_step": kern_avg / (elapsed / args.steps),
        "algorithmic": f"{macs:.4g} bit-pair MACs per launch = {n_local} knowns x {args.n_unknown} unknowns x {L} loci",
        # bytes the kernel must read from HBM per launch (the mxf4 tensor image for the
        # tensor path, the packed rows otherwise) over its time: far below the HBM roof
        "hbm_gbs": algo_bytes / kern_avg / 1e9,
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
        "data": WORKLOADS[args.workload]["data"],
        "config": config_dict(args, world),
        "e2e": e2e,
        "roofline": roofline,
        "clocks": clocks.summary(),
        "gpu_launches": launches_total,
        "gpu_launches_per_rank_step": launches / args.steps,
        "db_upload_s": db_upload_s,
        "db_build": db_build,
        "db_prepare_s": db_prepare_s,
        "wall_s_per_step": elapsed / args.steps,
        "verified_vs_oracle": verified,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = {k2: v for k2, v in cpu_reference_sample(args).items() if k2 != "seconds_per_rep"}
        if args.op != "andnot":  # the reference path has one operator; same words, same byte work
            line["cpu_baseline"]["note"] = f"the reference computes AND-NOT only; timed on AND-NOT, not {args.op}"
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(n: int, argv) -> int:
    """`--gpus N` without a launcher: start N ranks of this script (one process per
    GPU), the environment torchrun would give them, rendezvous on 127.0.0.1."""
    port = _free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   GROUP_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve()), *argv], env=env))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse_args(argv)
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus, argv)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
