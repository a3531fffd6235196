"""Small cases over every kernel path, for compute-sanitizer (memcheck / initcheck /
racecheck / synccheck) on a B200:

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py

Each case is checked against the oracle as well, so a run under the sanitizer
is also a parity run. Sizes are tiny: the sanitizer slows kernels by 100x+.
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np
import torch

import oracle
import paper_1707_00516_b200 as fb
from paper_1707_00516_b200.search import KnownDatabase


def panel(rng, n, L, tag):
    words = rng.integers(0, 2**64, (n, -(-L // 64)), dtype=np.uint64)
    if L % 64:
        words[:, -1] &= ~np.uint64(0) << np.uint64(64 - L % 64)
    return fb.Panel(tuple(f"{tag}{i}" for i in range(n)), words, L)


def main():
    rng = np.random.default_rng(7)
    n_cases = 0
    for L, n_r, n_q in ((1024, 600, 96), (127, 300, 33), (5000, 400, 40)):
        refs, queries = panel(rng, n_r, L, "r"), panel(rng, n_q, L, "q")
        expected = oracle.naive(refs.words, queries.words)
        for form in ("popc", "tensor_i8", "tensor_f4"):
            got = fb.compare_b200(refs, queries, formulation=form).scores
            assert np.array_equal(got, expected), (L, form, "full")
            res = fb.topk(refs, queries, 5, formulation=form)
            s, x, _ = oracle.topk_from_matrix(expected, 5)
            assert np.array_equal(res.scores, s) and np.array_equal(res.index, x), (L, form, "topk")
            n_cases += 2
        db = KnownDatabase(refs)
        s, x = db.search_words(queries.words, 16)
        es, ex, _ = oracle.topk_from_matrix(expected, 16)
        assert np.array_equal(s, es) and np.array_equal(x, ex), (L, "image topk")
        # poisoned output: bulk-tensor (TMA) stores are invisible to initcheck, so
        # a value check against the oracle is what proves every cell is written
        out = torch.full((n_r, n_q), -1, dtype=torch.int32, device="cuda")
        full = db.full_device(fb.DevicePanel.from_panel(queries), out).cpu().numpy().view(np.uint32)
        assert np.array_equal(full, expected), (L, "image full")
        thr = int(np.percentile(expected, 1))
        hits = db.threshold(queries, thr)
        jj, ii = np.nonzero(expected.T <= thr)
        assert np.array_equal(hits.query, jj) and np.array_equal(hits.ref, ii), (L, "threshold hits")
        assert np.array_equal(hits.score, expected.T[jj, ii]), (L, "threshold scores")
        n_cases += 3
    # dual-tile CTA pairs (streamed unknowns, >= 2 tiles per slice, odd remainder)
    refs, queries = panel(rng, 192 * 74 * 2 + 193, 5000, "r"), panel(rng, 40, 5000, "q")
    expected = oracle.naive(refs.words, queries.words)
    db = KnownDatabase(refs)
    s, x = db.search_words(queries.words, 16)
    es, ex, _ = oracle.topk_from_matrix(expected, 16)
    assert np.array_equal(s, es) and np.array_equal(x, ex), "dual-tile topk"
    out = torch.full((refs.words.shape[0], 40), -1, dtype=torch.int32, device="cuda")
    full = db.full_device(fb.DevicePanel.from_panel(queries), out).cpu().numpy().view(np.uint32)
    assert np.array_equal(full, expected), "dual-tile full"
    thr = int(np.percentile(expected, 1))
    hits = db.threshold(queries, thr)
    jj, ii = np.nonzero(expected.T <= thr)
    assert np.array_equal(hits.query, jj) and np.array_equal(hits.ref, ii), "dual-tile threshold"
    n_cases += 3
    # out-of-core top-k: host panel streamed in chunks (copy stream + device merge)
    refs, queries = panel(rng, 5000, 1024, "r"), panel(rng, 70, 1024, "q")
    expected = oracle.naive(refs.words, queries.words)
    res = fb.topk_streamed(refs, queries, 8, chunk_rows=1500)
    es, ex, _ = oracle.topk_from_matrix(expected, 8)
    assert np.array_equal(res.scores, es) and np.array_equal(res.index, ex), "streamed topk"
    n_cases += 1
    # chunked tensor image (one reusable buffer, fastid_db_create_in) and a graphed search
    refs, queries = panel(rng, 3000, 1024, "r"), panel(rng, 90, 1024, "q")
    expected = oracle.naive(refs.words, queries.words)
    db = KnownDatabase(refs, image_chunk_rows=192 * 5)
    db.chunked_min_queries = 1
    s, x = db.search_words(queries.words, 8)
    es, ex, _ = oracle.topk_from_matrix(expected, 8)
    assert np.array_equal(s, es) and np.array_equal(x, ex), "chunked topk"
    full = db.full_device(fb.DevicePanel.from_panel(queries)).cpu().numpy().view(np.uint32)
    assert np.array_equal(full, expected), "chunked full"
    db = KnownDatabase(refs)
    g = db.graphed_search(90, 8)
    s, x = g.run(queries.words)
    assert np.array_equal(s, es) and np.array_equal(x, ex), "graphed topk"
    n_cases += 3
    # the CUDA-core scan (<= 16 unknowns): top-k and threshold
    refs, queries = panel(rng, 5000, 777, "r"), panel(rng, 3, 777, "q")
    expected = oracle.naive(refs.words, queries.words)
    res = fb.topk(refs, queries, 8, formulation="popc")
    es, ex, _ = oracle.topk_from_matrix(expected, 8)
    assert np.array_equal(res.scores, es) and np.array_equal(res.index, ex), "scan topk"
    thr = int(np.percentile(expected, 1))
    hits = fb.threshold_hits(refs, queries, thr, formulation="popc")
    jj, ii = np.nonzero(expected.T <= thr)
    assert np.array_equal(hits.query, jj) and np.array_equal(hits.ref, ii), "scan threshold"
    n_cases += 2
    # one and two unknowns: the scan's bulk (sort + merge) list updates
    for nq in (1, 2):
        res = fb.topk(refs, fb.Panel(queries.ids[:nq], queries.words[:nq], 777), 16, formulation="popc")
        es, ex, _ = oracle.topk_from_matrix(expected[:, :nq], 16)
        assert np.array_equal(res.scores, es) and np.array_equal(res.index, ex), ("scan bulk", nq)
        n_cases += 1
    # AND / XOR operators: tiled kernel, scan, tensor kernels (packed rows and the image,
    # XOR's signed mxf4 operand and the i8 popcount epilogue)
    for L, n_r, n_q in ((1024, 700, 40), (5000, 400, 3)):
        refs, queries = panel(rng, n_r, L, "r"), panel(rng, n_q, L, "q")
        for op in ("and", "xor"):
            expected = oracle.np_scores_op(refs.words, queries.words, op)
            es, ex, _ = oracle.topk_from_matrix(expected, 8)
            for form in ("popc", "tensor_i8", "tensor_f4"):
                if not fb._native.supports(form, L):
                    continue
                got = fb.compare_b200(refs, queries, formulation=form, op=op).scores
                assert np.array_equal(got, expected), (L, op, form, "full")
                res = fb.topk(refs, queries, 8, formulation=form, op=op)
                assert np.array_equal(res.scores, es) and np.array_equal(res.index, ex), (L, op, form, "topk")
                n_cases += 2
            db = KnownDatabase(refs, op=op)
            s, x = db.search_words(queries.words, 8)
            assert np.array_equal(s, es) and np.array_equal(x, ex), (L, op, "image topk")
            thr = int(np.percentile(expected, 2))
            hits = db.threshold(queries, thr)
            jj, ii = np.nonzero(expected.T <= thr)
            assert np.array_equal(hits.query, jj) and np.array_equal(hits.ref, ii), (L, op, "image threshold")
            n_cases += 2
    torch.cuda.synchronize()
    print(f"sanitize cases ok ({n_cases})")


if __name__ == "__main__":
    main()
