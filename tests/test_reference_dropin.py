"""The drop-in claim, checked against the reference package itself.

The unmodified reference (pip-installed into baseline/_ref, which travels to
the GPU box; or /root/reference/pkg/src where it exists) supplies the panels,
the scheduler, the CLI and the oracle (compare_naive).  The B200 path enters
only through the reference's own seams:

* ``run_pipeline(..., executor=B200Executor())`` (scheduler.py:270-285), for the
  shapes of the reference's pipeline tests (test_scheduler.py:161-193, 290-303);
* ``PipelineConfig(kernel="b200")`` / ``fastid compare|bench --kernel b200``
  after ``reference_plugin.install()`` (scheduler.py:28, 243-246; cli.py:108-180),
  compared with the reference's own kernels (test_cli.py:99-119);
* ``compare_b200`` / ``compare_blocked_b200`` on reference ``Panel`` /
  ``QueryLayout`` objects, returning the reference's ``ScoreMatrix``
  (test_kernel.py:190-220).

Everything is skipped when the reference package is not importable.
"""

import ctypes
import os
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import gpu_available

ROOT = Path(__file__).resolve().parents[1]


def _reference():
    for cand in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (cand / "fastid" / "kernel.py").exists():
            os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/fastid_numba_cache")
            if str(cand) not in sys.path:
                sys.path.append(str(cand))
            try:
                import fastid  # noqa: F401

                return True
            except Exception:
                return False
    return False


HAVE_REF = _reference()
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="reference package not importable")
needs_gpu = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def rand_panel(rng, n_rows, n_words, word_width=64, bit_length=None, prefix="p"):
    """A reference Panel of random words with zero padding (the reference conftest's rule)."""
    from fastid.kernel import Panel

    bit_length = bit_length or n_words * word_width
    dtype = np.uint32 if word_width == 32 else np.uint64
    words = rng.integers(0, 2**word_width, size=(n_rows, n_words), dtype=dtype)
    tail = bit_length % word_width
    if tail and n_words:
        words[:, -1] &= dtype((2**word_width - 1) ^ ((1 << (word_width - tail)) - 1))
    return Panel(tuple(f"{prefix}{i}" for i in range(n_rows)), words, bit_length)


@pytest.fixture
def plugin():
    from paper_1707_00516_b200 import reference_plugin

    reference_plugin.install()
    yield reference_plugin
    reference_plugin.uninstall()


# ---- CPU: the plugin edits exactly the reference's kernel table / parser ----------

@needs_ref
def test_plugin_registers_b200_kernel(plugin):
    import fastid.cli as cli
    import fastid.scheduler as S

    from paper_1707_00516_b200 import B200Executor

    assert S.KERNELS == ("blocked", "naive", "b200")
    assert isinstance(S.make_executor(S.PipelineConfig(kernel="b200")), B200Executor)
    assert type(S.make_executor(S.PipelineConfig(kernel="naive"))).__name__ == "NaiveExecutor"
    args = cli.build_parser().parse_args(["compare", "--refs", "r", "--queries", "q", "--out", "o",
                                          "--kernel", "b200"])
    assert args.kernel == "b200"
    args = cli.build_parser().parse_args(["bench", "--sizes", "10x10x1", "--kernel", "b200"])
    assert args.kernel == "b200"
    plugin.uninstall()
    assert S.KERNELS == ("blocked", "naive")
    with pytest.raises(ValueError):
        S.PipelineConfig(kernel="b200")


# ---- GPU: the reference's own pipeline, CLI and bench over the B200 kernel ---------

@needs_ref
@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("buffers", ["reusable", "fresh"])
def test_multi_batch_composition_through_b200_executor(rng, overlap, buffers):
    """test_scheduler.py:161-173 with executor=B200Executor(): 4 batches of
    260/260/260/220 rows, scores byte-equal to compare_naive."""
    from fastid.kernel import compare_naive
    from fastid.scheduler import SCORE_CELL_BYTES, MemoryBudget, PipelineConfig, plan_batches, run_pipeline

    from paper_1707_00516_b200 import B200Executor

    refs = rand_panel(rng, 1000, 4, prefix="r")
    queries = rand_panel(rng, 256, 4, prefix="q")
    row_bytes = 4 * 8 + 256 * SCORE_CELL_BYTES
    plan = plan_batches(1000, 256, 4, 64, MemoryBudget(256 * 4 * 8 + 260 * row_bytes))
    assert plan.n_batches == 4
    ex = B200Executor()
    matrix, ledger = run_pipeline(plan, refs, queries, PipelineConfig(workers=2, overlap=overlap, buffers=buffers),
                                  executor=ex)
    assert np.array_equal(matrix.scores, compare_naive(refs, queries).scores)
    assert [b.rows for b in ledger.batches] == [260, 260, 260, 220]
    assert ex.calls == 4
    assert matrix.ref_ids == refs.ids and matrix.query_ids == queries.ids


@needs_ref
@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_custom_executor_seam_counts_batches(rng):
    """test_scheduler.py:290-303 with a counting subclass of B200Executor."""
    from fastid.kernel import compare_naive
    from fastid.scheduler import BatchPlan, run_pipeline

    from paper_1707_00516_b200 import B200Executor

    class CountingExecutor(B200Executor):
        calls_seen = 0

        def run(self, ref_words, query_words, out):
            CountingExecutor.calls_seen += 1
            super().run(ref_words, query_words, out)

    refs = rand_panel(rng, 12, 2, prefix="r")
    queries = rand_panel(rng, 5, 2, prefix="q")
    plan = BatchPlan(12, 5, 2, 64, ((0, 4), (4, 8), (8, 12)))
    matrix, _ = run_pipeline(plan, refs, queries, executor=CountingExecutor())
    assert CountingExecutor.calls_seen == 3
    assert np.array_equal(matrix.scores, compare_naive(refs, queries).scores)


@needs_ref
@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_pipeline_sink_and_one_row_batches(rng, plugin):
    """PipelineConfig(kernel="b200") through run_pipeline: one-row batches
    (test_scheduler.py:175-179) and a streaming sink fed in row order
    (test_scheduler.py:270-288), 32-bit words, overlap on."""
    from fastid.kernel import compare_naive
    from fastid.scheduler import ArraySink, BatchPlan, PipelineConfig, run_pipeline

    refs = rand_panel(rng, 7, 2, 32, prefix="r")
    queries = rand_panel(rng, 5, 2, 32, prefix="q")
    plan = BatchPlan(7, 5, 2, 32, tuple((i, i + 1) for i in range(7)))
    matrix, _ = run_pipeline(plan, refs, queries, PipelineConfig(kernel="b200", overlap=True))
    assert np.array_equal(matrix.scores, compare_naive(refs, queries).scores)

    class RecordingSink(ArraySink):
        def __init__(self, n_refs, n_queries):
            super().__init__(n_refs, n_queries)
            self.starts = []

        def put(self, start_row, chunk):
            self.starts.append(start_row)
            super().put(start_row, chunk)

    refs = rand_panel(rng, 30, 2, prefix="r")
    queries = rand_panel(rng, 4, 2, prefix="q")
    sink = RecordingSink(30, 4)
    matrix, _ = run_pipeline(BatchPlan(30, 4, 2, 64, ((0, 10), (10, 20), (20, 30))), refs, queries,
                             PipelineConfig(kernel="b200", overlap=True), sink=sink)
    assert matrix is None and sink.starts == [0, 10, 20]
    assert np.array_equal(sink.scores, compare_naive(refs, queries).scores)


@needs_ref
@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_compare_entries_on_reference_panels(rng):
    """compare_b200 / compare_blocked_b200 on the reference's own Panel and
    QueryLayout objects: the reference's ScoreMatrix type, byte-equal to
    compare_naive for the sweep of test_kernel.py:190-200 (blocks 16/32/64,
    workers 1/2/8, widths 32/64), the all-ones row of test_kernel.py:202-212,
    and identical bytes on repeated calls (test_kernel.py:214-221)."""
    from fastid.kernel import Panel, ScoreMatrix, TileConfig, compare_blocked, compare_naive, relayout_queries

    from paper_1707_00516_b200 import compare_b200, compare_blocked_b200

    for width in (32, 64):
        refs = rand_panel(rng, 100, 3, width, prefix="r")
        queries = rand_panel(rng, 100, 3, width, prefix="q")
        expected = compare_naive(refs, queries)
        got = compare_b200(refs, queries)
        assert isinstance(got, ScoreMatrix) and np.array_equal(got.scores, expected.scores)
        for block in (16, 32, 64):
            for workers in (1, 2, 8):
                got = compare_blocked_b200(refs, relayout_queries(queries), TileConfig(block), workers)
                assert isinstance(got, ScoreMatrix)
                assert np.array_equal(got.scores, expected.scores), (width, block, workers)
    words = np.zeros((2, 2), dtype=np.uint64)
    words[0] = [2**64 - 1, np.uint64(0xFFFFFFFF) << np.uint64(32)]
    refs = Panel(("ones", "zeros"), words, 96)
    queries = Panel(tuple(f"q{j}" for j in range(5)), np.zeros((5, 2), dtype=np.uint64), 96)
    got = compare_blocked_b200(refs, relayout_queries(queries), TileConfig(16), 2)
    assert got.scores[0].tolist() == [96] * 5 and got.scores[1].tolist() == [0] * 5
    refs = rand_panel(rng, 70, 5, prefix="r")
    queries = rand_panel(rng, 64, 5, prefix="q")
    layout = relayout_queries(queries)
    base = compare_blocked(refs, layout, TileConfig(32), 1).scores.tobytes()
    for _ in range(3):
        assert compare_blocked_b200(refs, layout, TileConfig(32), 8).scores.tobytes() == base
    with pytest.raises(ValueError):
        compare_blocked_b200(refs, layout, TileConfig(16), 0)


@needs_ref
@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_reference_cli_compare_with_b200_kernel(rng, tmp_path, plugin, capsys):
    """The reference CLI (fastid.cli.main) with --kernel b200: the CSV equals the
    naive kernel's file byte for byte (test_cli.py:110-119), matches
    compare_naive (test_cli.py:99-108), and a budgeted binary run equals the
    unlimited one (test_cli.py:121-133)."""
    from fastid.cli import EXIT_OK, main
    from fastid.io import read_scores_csv, save_panel
    from fastid.kernel import compare_naive
    from fastid.scheduler import SCORE_CELL_BYTES

    refs = rand_panel(rng, 50, 2, 64, prefix="ref")
    queries = rand_panel(rng, 20, 2, 64, prefix="qry")
    rp, qp = tmp_path / "refs.panel", tmp_path / "queries.panel"
    save_panel(refs, rp)
    save_panel(queries, qp)
    outs = {}
    for kernel in ("naive", "b200"):
        out = tmp_path / f"{kernel}.csv"
        assert main(["compare", "--refs", str(rp), "--queries", str(qp), "--out", str(out),
                     "--kernel", kernel]) == EXIT_OK
        outs[kernel] = out.read_bytes()
    assert outs["naive"] == outs["b200"]
    assert np.array_equal(read_scores_csv(tmp_path / "b200.csv").scores, compare_naive(refs, queries).scores)
    row_bytes = 2 * 8 + 20 * SCORE_CELL_BYTES
    budget = str(20 * 2 * 8 + 12 * row_bytes)
    a, b = tmp_path / "budget.bin", tmp_path / "unlimited.bin"
    capsys.readouterr()
    assert main(["compare", "--refs", str(rp), "--queries", str(qp), "--out", str(a), "--format", "binary",
                 "--budget", budget, "--kernel", "b200"]) == EXIT_OK
    assert "5 batch(es)" in capsys.readouterr().out
    assert main(["compare", "--refs", str(rp), "--queries", str(qp), "--out", str(b), "--format", "binary",
                 "--kernel", "b200"]) == EXIT_OK
    assert a.read_bytes() == b.read_bytes()


@needs_ref
@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_reference_cli_bench_schema_with_b200_kernel(tmp_path, plugin):
    """`fastid bench --kernel b200` writes the reference's bench CSV schema
    (cli.py:144-147) with the same score checksum as the blocked kernel on the
    same synthetic job (the reference's determinism guard)."""
    import csv

    from fastid.cli import EXIT_OK, main

    rows = {}
    for kernel in ("blocked", "b200"):
        out = tmp_path / f"{kernel}.csv"
        assert main(["bench", "--sizes", "3000x256x16,777x33x3", "--kernel", kernel, "--reps", "2",
                     "--out", str(out)]) == EXIT_OK
        with open(out) as fh:
            rows[kernel] = list(csv.DictReader(fh))
    header = ("n_refs,n_queries,n_words,kernel,tile,workers,stage_in_ms,compute_ms,stage_out_ms,"
              "comparisons_per_s,seed,checksum").split(",")
    assert list(rows["b200"][0].keys()) == header
    assert [r["checksum"] for r in rows["b200"]] == [r["checksum"] for r in rows["blocked"]]
    assert all(r["kernel"] == "b200" and float(r["comparisons_per_s"]) > 0 for r in rows["b200"])


# ---- the single-call top-k entry INTEGRATION.md points integrators to -------------

@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
@pytest.mark.parametrize("form", ["popc", "tensor_i8", "tensor_f4"])
def test_fastid_compare_topk_single_call(rng, form):
    """fastid_compare_topk (partials + merge in one C call) through ctypes, with
    a ref_base offset and a score cap, equals the oracle; empty known panels
    give empty slots."""
    import torch

    import oracle
    import paper_1707_00516_b200 as m
    from paper_1707_00516_b200 import _native
    from conftest import rand_words

    L, n_r, n_q, k = 1000, 5000, 130, 16
    r, _ = rand_words(rng, n_r, 16, 64, L)
    q, _ = rand_words(rng, n_q, 16, 64, L)
    q[:40] = r[rng.integers(0, n_r, 40)]
    dr, dq = m.DevicePanel.from_words(r, L), m.DevicePanel.from_words(q, L)
    lib = _native.lib()
    need = ctypes.c_size_t(0)
    code = _native.formulation_code(form)
    _native.check(lib.fastid_topk_workspace(n_r, n_q, k, code, ctypes.byref(need)), "workspace")
    ws = torch.empty(need.value, dtype=torch.uint8, device="cuda")
    s = torch.empty((n_q, k), dtype=torch.int32, device="cuda")
    x = torch.empty((n_q, k), dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    for cap in (0xFFFFFFFE, L // 5):
        _native.check(lib.fastid_compare_topk(dr.rows.data_ptr(), n_r, dq.rows.data_ptr(), n_q, dr.stride, L, k, cap,
                                              1_000_000, s.data_ptr(), x.data_ptr(), ws.data_ptr(), need.value,
                                              code, stream), "fastid_compare_topk")
        es, ex, _ = oracle.topk(r, q, k, cap)
        assert np.array_equal(s.cpu().numpy().view(np.uint32), es)
        assert np.array_equal(x.cpu().numpy(), np.where(ex >= 0, ex + 1_000_000, -1))
    _native.check(lib.fastid_compare_topk(0, 0, dq.rows.data_ptr(), n_q, dr.stride, L, k, 0xFFFFFFFE, 0,
                                          s.data_ptr(), x.data_ptr(), ws.data_ptr(), need.value, code, stream),
                  "fastid_compare_topk(empty)")
    assert (s.cpu().numpy().view(np.uint32) == 0xFFFFFFFF).all() and (x.cpu().numpy() == -1).all()
    # a workspace one byte short is refused before any launch
    assert lib.fastid_compare_topk(dr.rows.data_ptr(), n_r, dq.rows.data_ptr(), n_q, dr.stride, L, k, 0xFFFFFFFE, 0,
                                   s.data_ptr(), x.data_ptr(), ws.data_ptr(), need.value - 1, code,
                                   stream) == _native.E_CAPACITY
