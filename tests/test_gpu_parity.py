"""Parity of the sm_100a kernels with the oracle and the reference goldens.

Every test here calls through the C ABI (include/fastid_b200.h) via the
package; the oracle (oracle/) is only the checker.  Bar: bit-exact.
"""

import json
import os

import numpy as np
import pytest
import torch

import oracle

from conftest import GOLDEN, gpu_available, rand_words

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

FORMS = ["popc", "tensor_i8", "tensor_f4", "auto"]


def fb():
    import paper_1707_00516_b200 as m

    return m


def _supported(form, L):
    from paper_1707_00516_b200 import _native

    return _native.supports(form, L)


def panels(c):
    m = fb()
    L = c["bits"]
    r = m.Panel(tuple(f"r{i}" for i in range(c["refs"].shape[0])), c["refs"], L)
    q = m.Panel(tuple(f"q{j}" for j in range(c["queries"].shape[0])), c["queries"], L)
    return r, q


@pytest.mark.parametrize("form", FORMS)
def test_full_matrix_goldens(kernel_cases, form):
    for c in kernel_cases:
        if not _supported(form, c["bits"]):
            continue
        r, q = panels(c)
        got = fb().compare_b200(r, q, formulation=form)
        assert got.scores.dtype == np.uint32
        assert np.array_equal(got.scores, c["scores"]), (form, c["name"])


@pytest.mark.parametrize("form", FORMS)
def test_topk_goldens(topk_cases, form):
    for c in topk_cases:
        if not _supported(form, c["bits"]):
            continue
        r, q = panels(c)
        k = int(c["k"])
        res = fb().topk(r, q, k, formulation=form)
        assert np.array_equal(res.scores, c["top_scores"]), (form, c["name"])
        assert np.array_equal(res.index, c["top_index"]), (form, c["name"])


@pytest.mark.parametrize("form", FORMS)
def test_threshold_goldens(topk_cases, form):
    for c in topk_cases:
        if not _supported(form, c["bits"]):
            continue
        r, q = panels(c)
        hits = fb().threshold_hits(r, q, int(c["threshold"]), formulation=form)
        assert np.array_equal(hits.query, c["hit_query"]), (form, c["name"])
        assert np.array_equal(hits.ref, c["hit_ref"]), (form, c["name"])
        assert np.array_equal(hits.score, c["hit_score"]), (form, c["name"])


@pytest.mark.parametrize("form", FORMS)
@pytest.mark.parametrize("k", [1, 5, 16, 32])
def test_topk_vs_oracle_random(rng, form, k):
    for n_r, n_q, L, width in ((3000, 200, 1024, 64), (999, 129, 777, 32), (5, 300, 5000, 64)):
        if not _supported(form, L):
            continue
        nw = -(-L // width)
        r, _ = rand_words(rng, n_r, nw, width, L)
        q, _ = rand_words(rng, n_q, nw, width, L)
        # plant exact copies and duplicates so ties and zeros occur
        q[: min(20, n_q)] = r[rng.integers(0, n_r, min(20, n_q))]
        r[n_r // 2 : n_r // 2 + 3] = r[:3]
        m = fb()
        R, Q = m.Panel(tuple(range(n_r)), r, L), m.Panel(tuple(range(n_q)), q, L)
        full = oracle.naive(r, q)
        for ms in (None, int(np.percentile(full, 2))):
            res = m.topk(R, Q, k, max_score=ms, formulation=form)
            es, ex, _ = oracle.topk_from_matrix(full, k, 0xFFFFFFFE if ms is None else ms)
            assert np.array_equal(res.scores, es), (form, n_r, n_q, L, ms)
            assert np.array_equal(res.index, ex), (form, n_r, n_q, L, ms)


@pytest.mark.parametrize("form", FORMS)
def test_checksums_vs_reference(checksum_rows, form):
    m = fb()
    import torch

    for row in checksum_rows:
        refs = oracle.synth_words(row["n_refs"], row["n_words"], row["word_width"], row["seed"], 0)
        queries = oracle.synth_words(row["n_queries"], row["n_words"], row["word_width"], row["seed"], 1)
        L = row["n_words"] * row["word_width"]
        if not _supported(form, L):
            continue
        dr = m.DevicePanel.from_words(refs, L)
        dq = m.DevicePanel.from_words(queries, L)
        out = m.compare_device(dr, dq, formulation=form)
        scores = out.cpu().numpy().view(np.uint32)
        assert oracle.score_checksum(scores) == row["checksum"], (form, row["label"])
        del out
        torch.cuda.empty_cache()


def test_empty_panels():
    m = fb()
    r = m.Panel((), np.zeros((0, 2), np.uint64), 128)
    q = m.Panel(("a", "b", "c"), np.zeros((3, 2), np.uint64), 128)
    assert m.compare_b200(r, q).shape == (0, 3)
    assert m.compare_b200(q, r).shape == (3, 0)
    res = m.topk(r, q, 4)
    assert (res.index == -1).all() and (res.scores == 0xFFFFFFFF).all()


def test_mismatch_errors():
    m = fb()
    a = m.Panel(("a",), np.zeros((1, 2), np.uint32), 64)
    b = m.Panel(("b",), np.zeros((1, 2), np.uint32), 40)
    with pytest.raises(m.PanelMismatchError):
        m.compare_b200(a, b)
    c = m.Panel(("c",), np.zeros((1, 1), np.uint64), 64)
    with pytest.raises(m.PanelMismatchError):
        m.compare_b200(a, c)
    with pytest.raises(ValueError):
        m.compare_blocked_b200(a, m.relayout_queries(a), m.TileConfig(16), 0)


@pytest.mark.parametrize("form", FORMS)
def test_run_kernel_host_path(rng, form):
    m = fb()
    for width, transposed in ((64, False), (32, True)):
        r, _ = rand_words(rng, 333, 1024 // width, width)
        q, _ = rand_words(rng, 77, 1024 // width, width)
        out = np.empty((333, 77), np.uint32)
        qa = np.ascontiguousarray(q.T) if transposed else q
        m.run_b200_kernel(r, qa, out, queries_transposed=transposed, formulation=form)
        assert np.array_equal(out, oracle.naive(r, q))


@pytest.mark.parametrize("width,transposed", [(64, False), (32, True)])
def test_run_kernel_chunked_pipeline(rng, width, transposed):
    """Outputs above 64 MB stream through the chunked pinned pipeline of
    fastid_run_kernel (two chunks, the second ragged): every cell written."""
    m = fb()
    n_r, n_q, L = 45_000, 520, 512
    r, _ = rand_words(rng, n_r, L // width, width)
    q, _ = rand_words(rng, n_q, L // width, width)
    out = np.empty((n_r, n_q), np.uint32)
    qa = np.ascontiguousarray(q.T) if transposed else q
    m.run_b200_kernel(r, qa, out, queries_transposed=transposed)
    assert out.nbytes > 64 << 20
    assert np.array_equal(out, oracle.naive(r, q))


def test_compare_b200_large_result(rng):
    """compare_b200 (the compare_naive drop-in) with a > 64 MB ScoreMatrix takes
    the chunked host pipeline; u32 panels, partial last word."""
    m = fb()
    n_r, n_q, L = 33_000, 600, 1000
    r, _ = rand_words(rng, n_r, -(-L // 32), 32, L)
    q, _ = rand_words(rng, n_q, -(-L // 32), 32, L)
    R, Q = m.Panel(tuple(range(n_r)), r, L), m.Panel(tuple(range(n_q)), q, L)
    got = m.compare_b200(R, Q)
    assert got.scores.nbytes > 64 << 20
    assert np.array_equal(got.scores, oracle.naive(r, q))


def test_compare_to_fidm_matches_reference_files(tmp_path, rng):
    """compare_to_fidm writes the reference's packed-binary score file byte for
    byte (reference-written goldens), small and through several pipeline chunks."""
    m = fb()
    d = np.load(GOLDEN / "fidm_cases.npz")
    for name in ("golden_4x4", "rand_37x23_L100"):
        r, q, L = d[f"{name}__refs"], d[f"{name}__queries"], int(d[f"{name}__bits"])
        path = tmp_path / f"{name}.fidm"
        m.compare_to_fidm(m.Panel(tuple(range(len(r))), r, L), m.Panel(tuple(range(len(q))), q, L), path)
        assert path.read_bytes() == d[f"{name}__fidm"].tobytes(), name
    n_r, n_q, L = 70_000, 300, 256
    r, _ = rand_words(rng, n_r, L // 64, 64, L)
    q, _ = rand_words(rng, n_q, L // 64, 64, L)
    path = tmp_path / "big.fidm"
    assert m.compare_to_fidm(m.Panel(tuple(range(n_r)), r, L), m.Panel(tuple(range(n_q)), q, L), path) == (n_r, n_q)
    blob = path.read_bytes()
    assert blob[:21] == __import__("struct").pack("<4sBQQ", b"FIDM", 1, n_r, n_q)
    assert np.array_equal(np.frombuffer(blob[21:], "<u4").reshape(n_r, n_q), oracle.naive(r, q))


def test_executor_seam(rng):
    m = fb()
    r, _ = rand_words(rng, 100, 4, 64)
    q, _ = rand_words(rng, 9, 4, 64)
    ex = m.B200Executor()
    out = np.empty((100, 9), np.uint32)
    ex.run(r, q, out)
    assert ex.calls == 1 and np.array_equal(out, oracle.naive(r, q))


def test_encoder_matches_reference_pack(pack_cases):
    m = fb()
    for L in pack_cases["lengths"]:
        bits = pack_cases[f"L{L}_bits"]
        for width in (32, 64):
            d = m.DevicePanel.from_bits(bits, width)
            assert np.array_equal(d.to_words(), pack_cases[f"L{L}_w{width}"]), (L, width)
            # padding of the device row is zero past the packed words
            nb = d.n_words * width // 8
            assert int(d.rows[:, nb:].sum()) == 0


def test_genotype_encoder(genotype_rows):
    m = fb()
    codes_of = {"MM": 0, "Mm": 1, "mM": 2, "mm": 3}
    for row in genotype_rows:
        codes = np.array([[codes_of[c] for c in row["codes"]]], np.uint8)
        d = m.DevicePanel.from_genotypes(codes, 32)
        assert d.bit_length == len(row["bits"])
        assert d.to_words().tolist() == [row["w32"]]
    with pytest.raises(m.CodecError):
        m.DevicePanel.from_genotypes(np.array([[0, 4]], np.uint8))


def test_load_words_roundtrip(rng):
    m = fb()
    for width, L in ((32, 50), (64, 5000), (64, 1)):
        w, _ = rand_words(rng, 17, -(-L // width), width, L)
        d = m.DevicePanel.from_words(w, L)
        assert d.stride % 16 == 0 and d.stride == m.row_stride(L)
        assert np.array_equal(d.to_words(), w)


@pytest.mark.parametrize("form", FORMS)
@pytest.mark.parametrize("L", [2048, 2049, 5000, 40000])
def test_long_profiles_exact(rng, form, L):
    """Large accumulations stay exact (scores up to L), incl. the streamed-A path."""
    m = fb()
    nw = -(-L // 64)
    r, _ = rand_words(rng, 300, nw, 64, L)
    q, _ = rand_words(rng, 140, nw, 64, L)
    # extremes: an all-ones known (score L vs the all-zero unknown), dense/sparse rows
    r[0] = np.uint64(2**64 - 1)
    r = oracle.mask_padding(r, L)
    q[0] = 0
    r[1] &= r[2]
    q[1] |= q[2]
    R, Q = m.Panel(tuple(range(300)), r, L), m.Panel(tuple(range(140)), q, L)
    exp = oracle.naive(r, q)
    assert exp[0, 0] == L
    got = m.compare_b200(R, Q, formulation=form).scores
    assert np.array_equal(got, exp), (form, L)
    res = m.topk(R, Q, 8, formulation=form)
    es, ex, _ = oracle.topk_from_matrix(exp, 8)
    assert np.array_equal(res.scores, es) and np.array_equal(res.index, ex)


@pytest.mark.parametrize("form", ["tensor_f4", "tensor_i8", "popc"])
@pytest.mark.parametrize("L", [300, 1024, 5000])
def test_prepared_database_image(rng, form, L):
    """KnownDatabase (fastid_db handle, tensor image) == oracle for top-k, full matrix and threshold."""
    m = fb()
    from paper_1707_00516_b200.search import KnownDatabase

    nw = -(-L // 64)
    r, _ = rand_words(rng, 2500, nw, 64, L)
    q, _ = rand_words(rng, 150, nw, 64, L)
    q[:30] = r[rng.integers(0, 2500, 30)]
    r[1000:1003] = r[:3]
    db = KnownDatabase(r, L, formulation=form, ref_base=1000)
    if form != "popc":
        assert db.image.image_bytes > 0
    dq = m.DevicePanel.from_words(q, L)
    full = db.full_device(dq).cpu().numpy().view(np.uint32)
    exp = oracle.naive(r, q)
    assert np.array_equal(full, exp)
    # every cell is written (the output is poisoned first, so stale allocator
    # contents cannot pass for results), including a row pitch wider than N_Q
    poisoned = torch.full((2500, 160), -1, dtype=torch.int32, device=dq.rows.device)
    db.full_device(dq, poisoned)
    got = poisoned.cpu().numpy().view(np.uint32)
    assert np.array_equal(got[:, :150], exp) and (got[:, 150:] == 0xFFFFFFFF).all()
    s, x = db.search_words(q, 16)
    es, ex, _ = oracle.topk_from_matrix(exp, 16)
    assert np.array_equal(s, es)
    assert np.array_equal(x, np.where(ex >= 0, ex + 1000, -1))
    thr = int(np.percentile(exp, 1))
    hits = db.threshold(m.Panel(tuple(range(150)), q, L), thr)
    hq, hr, hs = oracle.threshold_from_matrix(exp, thr)
    assert np.array_equal(hits.query, hq) and np.array_equal(hits.ref, hr + 1000) and np.array_equal(hits.score, hs)


@pytest.mark.parametrize("pairs", [True, False])
@pytest.mark.parametrize("L", [10_000, 40_000])
def test_prepared_image_streamed_unknowns_long_profiles(rng, pairs, L):
    """The C5 long-profile path: prepared mxf4 image with the unknowns streamed per
    stage (L > 2048), on the CTA-pair kernel and on the single-CTA split-B
    kernel: top-k (k = 1, 16, 32), threshold and full matrix equal the oracle,
    with a ragged second pair group (300 unknowns), planted copies, duplicate
    knowns (ties) and an all-ones known (score L against an all-zero unknown)."""
    m = fb()
    from paper_1707_00516_b200.search import KnownDatabase

    n_r, n_q = 2311, 300
    nw = -(-L // 64)
    r, _ = rand_words(rng, n_r, nw, 64, L)
    q, _ = rand_words(rng, n_q, nw, 64, L)
    r[5] = np.uint64(2**64 - 1)
    r = oracle.mask_padding(r, L)
    q[0] = 0
    q[1:60] = r[rng.integers(0, n_r, 59)]
    r[n_r - 7 : n_r - 4] = r[10:13]
    db = KnownDatabase(r, L, formulation="tensor_f4", ref_base=3)
    db.set_option("no_cta_pairs", not pairs)
    exp = oracle.naive(r, q)
    assert exp[5, 0] == L
    for k in (1, 16, 32):
        s, x = db.search_words(q, k)
        es, ex, _ = oracle.topk_from_matrix(exp, k)
        assert np.array_equal(s, es), k
        assert np.array_equal(x, np.where(ex >= 0, ex + 3, -1)), k
    thr = int(np.percentile(exp, 3))
    hits = db.threshold(m.Panel(tuple(range(n_q)), q, L), thr)
    hq, hr, hs = oracle.threshold_from_matrix(exp, thr)
    assert np.array_equal(hits.query, hq) and np.array_equal(hits.ref, hr + 3) and np.array_equal(hits.score, hs)
    full = db.full_device(m.DevicePanel.from_words(q, L)).cpu().numpy().view(np.uint32)
    assert np.array_equal(full, exp)


@pytest.mark.parametrize("form", ["tensor_f4", "tensor_i8", "popc"])
def test_longest_profiles_all_ones_exact(rng, form):
    """L = 2^20 loci, the reference's upper bound: an all-ones known
    scores 1,048,576 against an all-zero unknown.  The accumulators stay exact
    (fp32 < 2^24 for mxf4, s32 for i8, u32 for POPC) on the packed-operand
    kernels and on the prepared-image kernels (CTA pairs for mxf4), for the
    full matrix, top-k and threshold."""
    m = fb()
    from paper_1707_00516_b200.search import KnownDatabase

    L = 1 << 20
    nw = L // 64
    r, _ = rand_words(rng, 40, nw, 64, L)
    q, _ = rand_words(rng, 6, nw, 64, L)
    r[0] = np.uint64(2**64 - 1)
    r[1] = 0
    r[2, : nw // 2] = np.uint64(2**64 - 1)
    r[2, nw // 2 :] = 0
    q[0] = 0
    q[1] = np.uint64(2**64 - 1)
    q[2] = r[3]
    exp = oracle.naive(r, q)
    assert exp[0, 0] == L and exp[2, 0] == L // 2 and exp[0, 1] == 0 and exp[3, 2] == 0
    R, Q = m.Panel(tuple(range(40)), r, L), m.Panel(tuple(range(6)), q, L)
    assert np.array_equal(m.compare_b200(R, Q, formulation=form).scores, exp), "packed full"
    res = m.topk(R, Q, 4, formulation=form)
    es, ex, _ = oracle.topk_from_matrix(exp, 4)
    assert np.array_equal(res.scores, es) and np.array_equal(res.index, ex), "packed top-k"
    db = KnownDatabase(r, L, formulation=form)
    full = db.full_device(m.DevicePanel.from_words(q, L)).cpu().numpy().view(np.uint32)
    assert np.array_equal(full, exp), "image full"
    s, x = db.search_words(q, 4)
    assert np.array_equal(s, es) and np.array_equal(x, ex), "image top-k"
    hits = db.threshold(Q, L // 2)
    hq, hr, hs = oracle.threshold_from_matrix(exp, L // 2)
    assert np.array_equal(hits.query, hq) and np.array_equal(hits.ref, hr) and np.array_equal(hits.score, hs)


@pytest.mark.parametrize("pairs", [True, False])
@pytest.mark.parametrize("shape", [(1137, 129, 1024), (2500, 520, 2048), (700, 300, 1800), (224, 256, 64),
                                   (3001, 388, 1024), (5000, 260, 512), (1500, 300, 5000), (900, 520, 2304)])
def test_image_pairs_and_split(rng, pairs, shape):
    """Prepared mxf4 image: the CTA-pair kernel (cta_group::2, M=256) and the
    single-CTA split-B kernel (option no_cta_pairs) both equal the oracle, for every
    epilogue, with ragged unknown groups and known tiles.  Unknown counts that
    are multiples of 4 with L <= 1024 take the TMA-store full-matrix epilogue,
    the others its direct-store fallback."""
    m = fb()
    from paper_1707_00516_b200 import _native
    from paper_1707_00516_b200.search import KnownDatabase

    n_r, n_q, L = shape
    nw = -(-L // 64)
    r, _ = rand_words(rng, n_r, nw, 64, L)
    q, _ = rand_words(rng, n_q, nw, 64, L)
    q[: n_q // 4] = r[rng.integers(0, n_r, n_q // 4)]
    r[n_r // 2 : n_r // 2 + 3] = r[:3]
    db = KnownDatabase(r, L, formulation="tensor_f4", ref_base=7)
    db.set_option("no_cta_pairs", not pairs)
    dq = m.DevicePanel.from_words(q, L)
    exp = oracle.naive(r, q)
    full = db.full_device(dq).cpu().numpy().view(np.uint32)
    assert np.array_equal(full, exp)
    for k in (1, 16, 32):
        s, x = db.search_words(q, k)
        es, ex, _ = oracle.topk_from_matrix(exp, k)
        assert np.array_equal(s, es), k
        assert np.array_equal(x, np.where(ex >= 0, ex + 7, -1)), k
    thr = int(np.percentile(exp, 2))
    hits = db.threshold(m.Panel(tuple(range(n_q)), q, L), thr)
    hq, hr, hs = oracle.threshold_from_matrix(exp, thr)
    assert np.array_equal(hits.query, hq) and np.array_equal(hits.ref, hr + 7)
    assert np.array_equal(hits.score, hs)


@pytest.mark.parametrize("k,max_score", [(5, None), (16, 240), (1, 250), (32, None)])
def test_pairs_topk_caps_and_list_sizes(rng, k, max_score):
    """CTA-pair top-k with list sizes 8/16/32, a score cap, and shared
    admission bounds over many lists (25 slices x 3 splits per unknown)."""
    m = fb()
    from paper_1707_00516_b200.search import KnownDatabase

    L, n_r, n_q = 1024, 4800, 512
    r, _ = rand_words(rng, n_r, L // 64, 64, L)
    q, _ = rand_words(rng, n_q, L // 64, 64, L)
    q[::7] = r[rng.integers(0, n_r, len(q[::7]))]
    db = KnownDatabase(r, L, formulation="tensor_f4")
    s, x = db.search_words(q, k, max_score)
    es, ex, _ = oracle.topk(r, q, k, 0xFFFFFFFE if max_score is None else max_score)
    assert np.array_equal(s, es) and np.array_equal(x, ex)


def test_pairs_more_groups_than_sms(rng):
    """More unknown groups than co-resident CTA pairs (drift control off; the
    grid runs in waves): still exact."""
    m = fb()
    from paper_1707_00516_b200.search import KnownDatabase

    L, n_r, n_q = 256, 1500, 80 * 256 + 37
    r, _ = rand_words(rng, n_r, L // 64, 64, L)
    q, _ = rand_words(rng, n_q, L // 64, 64, L)
    db = KnownDatabase(r, L, formulation="tensor_f4")
    s, x = db.search_words(q, 4)
    pick = np.arange(0, n_q, 97)
    es, ex, _ = oracle.topk(r, q[pick], 4)
    assert np.array_equal(s[pick], es) and np.array_equal(x[pick], ex)
    full = db.full_device(m.DevicePanel.from_words(q[:300], L)).cpu().numpy().view(np.uint32)
    assert np.array_equal(full, oracle.naive(r, q[:300]))


def test_cli_compare_and_search(tmp_path):
    """python -m paper_1707_00516_b200 compare / search on panel files: the
    binary output is the reference-written FIDM file, the CSV the reference's
    golden scores_4x4.csv bytes, search the oracle's top-k."""
    m = fb()
    from paper_1707_00516_b200.__main__ import main
    from paper_1707_00516_b200.ingest import save_panel

    d = np.load(GOLDEN / "fidm_cases.npz")
    r, q = d["golden_4x4__refs"], d["golden_4x4__queries"]
    save_panel(m.Panel(tuple(f"r{i}" for i in range(4)), r, 8), tmp_path / "r.panel")
    save_panel(m.Panel(tuple(f"q{j}" for j in range(4)), q, 8), tmp_path / "q.panel")
    args = ["--refs", str(tmp_path / "r.panel"), "--queries", str(tmp_path / "q.panel"), "--word-width", "32"]
    assert main(["compare", *args, "--out", str(tmp_path / "s.fidm"), "--format", "binary"]) == 0
    assert (tmp_path / "s.fidm").read_bytes() == d["golden_4x4__fidm"].tobytes()
    assert main(["compare", *args, "--out", str(tmp_path / "s.csv")]) == 0
    assert (tmp_path / "s.csv").read_text() == "ref_id,q0,q1,q2,q3\nr0,0,4,2,2\nr1,4,0,4,2\nr2,4,4,6,4\nr3,0,0,0,0\n"
    assert main(["search", *args, "--out", str(tmp_path / "t.csv"), "-k", "2"]) == 0
    rows = (tmp_path / "t.csv").read_text().splitlines()
    assert rows[0] == "query_id,rank,ref_id,score" and rows[1:3] == ["q0,1,r0,0", "q0,2,r3,0"]
    assert main(["compare", "--refs", str(tmp_path / "missing"), "--queries", "x", "--out", "y"]) == 1


@pytest.mark.parametrize("shape", [(60_000, 2048, 1024), (80_000, 700, 512), (40_000, 1024, 2304)])
def test_pairs_large_panels(rng, shape):
    """Larger panels on the CTA-pair kernel (resident and streamed unknowns,
    drift control active, and -- where (unknown groups x slices) leaves SMs
    free -- the spare-pair grid over the tail tiles of several groups): top-k,
    threshold and full rows near both ends of the known range equal the oracle,
    and the top-k equals the launch without spare pairs (option no_spare_pairs)."""
    import torch

    m = fb()
    from paper_1707_00516_b200.search import KnownDatabase

    n_r, n_q, L = shape
    nw = L // 64
    r, _ = rand_words(rng, n_r, nw, 64, L)
    q, _ = rand_words(rng, n_q, nw, 64, L)
    q[::5] = r[rng.integers(n_r - n_r // 30, n_r, len(q[::5]))]  # copies near the end of the known range
    db = KnownDatabase(r, L, formulation="tensor_f4")
    s, x = db.search_words(q, 16)
    pick = np.arange(0, n_q, 7)
    es, ex, _ = oracle.topk(r, q[pick], 16)
    assert np.array_equal(s[pick], es) and np.array_equal(x[pick], ex)
    db.set_option("no_spare_pairs")
    s2, x2 = db.search_words(q, 16)
    db.set_option("no_spare_pairs", False)
    assert np.array_equal(s, s2) and np.array_equal(x, x2)
    dq = m.DevicePanel.from_words(q, L)
    full = db.full_device(dq)
    rows = np.concatenate([np.arange(0, 64), np.arange(n_r - 300, n_r)])
    got = full[torch.from_numpy(rows).cuda()].cpu().numpy().view(np.uint32)
    assert np.array_equal(got, oracle.naive(r[rows], q))
    thr = L // 8  # planted copies (0) only; random pairs sit near L/4
    hits = db.threshold(m.Panel(tuple(range(n_q)), q, L), thr)
    sub = oracle.naive(r[n_r - 300:], q)
    hq, hr, hs = oracle.threshold_from_matrix(sub, thr)
    sel = hits.ref >= n_r - 300
    assert np.array_equal(hits.query[sel], hq) and np.array_equal(hits.ref[sel], hr + n_r - 300)


@pytest.mark.parametrize("n_r,n_q,k,max_score", [(5, 1, 16, None), (3, 300, 8, 0), (200, 1, 32, 300),
                                                 (193, 257, 16, None), (1, 2, 1, None)])
def test_pairs_edge_shapes(rng, n_r, n_q, k, max_score):
    """Prepared-database (CTA-pair) top-k with fewer knowns than k, a single
    unknown, a zero or partial score cap, one-row tiles and a second pair group
    of one unknown: equal to the oracle, empty slots 0xFFFFFFFF / -1."""
    m = fb()
    from paper_1707_00516_b200.search import KnownDatabase

    L = 1024
    r, _ = rand_words(rng, n_r, 16, 64, L)
    q, _ = rand_words(rng, n_q, 16, 64, L)
    q[0] = r[0]  # one exact copy: score 0
    db = KnownDatabase(r, L, formulation="tensor_f4")
    s, x = db.search_words(q, k, max_score)
    es, ex, _ = oracle.topk(r, q, k, 0xFFFFFFFE if max_score is None else max_score)
    assert np.array_equal(s, es) and np.array_equal(x, ex)
    full = db.full_device(m.DevicePanel.from_words(q, L)).cpu().numpy().view(np.uint32)
    assert np.array_equal(full, oracle.naive(r, q))


def test_database_reuse_across_shapes(rng):
    """One resident database answering a sequence of batches of different sizes,
    list sizes and caps (launch scratch, shared bounds, progress counters and the
    spare-pair stream are reused between calls): every batch equals the oracle."""
    m = fb()
    from paper_1707_00516_b200.search import KnownDatabase

    L, n_r = 1024, 40_000
    r, _ = rand_words(rng, n_r, 16, 64, L)
    db = KnownDatabase(r, L, formulation="tensor_f4")
    for n_q, k, ms in ((2048, 16, None), (1, 1, None), (300, 32, 250), (2048, 5, None), (77, 16, 0)):
        q, _ = rand_words(rng, n_q, 16, 64, L)
        q[: max(1, n_q // 9)] = r[rng.integers(0, n_r, max(1, n_q // 9))]
        s, x = db.search_words(q, k, ms)
        pick = np.unique(np.linspace(0, n_q - 1, 12).astype(int))
        es, ex, _ = oracle.topk(r, q[pick], k, 0xFFFFFFFE if ms is None else ms)
        assert np.array_equal(s[pick], es) and np.array_equal(x[pick], ex), (n_q, k, ms)


@pytest.mark.parametrize("n_r,n_q", [(2500, 150), (2500, 152), (2431, 149)])
def test_full_matrix_writes_stay_in_view(rng, n_r, n_q):
    """The full matrix is written into a poisoned view [n_r, n_q] of a larger buffer
    (row pitch 160, 100 extra rows): every cell outside the view keeps the poison,
    for every formulation, with and without the prepared image and for each epilogue
    store variant (options no_tma_store / narrow_tma_store). Covers
    the TMA unit's 16-byte clipping of partial unknown granules."""
    m = fb()
    from paper_1707_00516_b200 import _native
    from paper_1707_00516_b200.search import KnownDatabase

    L = 1024
    r, _ = rand_words(rng, n_r, 16, 64, L)
    q, _ = rand_words(rng, n_q, 16, 64, L)
    exp = oracle.naive(r, q)
    dq = m.DevicePanel.from_words(q, L)
    dr = m.DevicePanel.from_words(r, L)
    for form in ("tensor_f4", "tensor_i8", "popc"):
        db = KnownDatabase(r, L, formulation=form)
        for flags in ((), ("no_tma_store",), ("narrow_tma_store",)):
            for name in ("no_tma_store", "narrow_tma_store"):
                db.set_option(name, name in flags)
            for use_db in (True, False):
                buf = torch.full((n_r + 100, 160), -1, dtype=torch.int32, device=dq.rows.device)
                view = buf[:n_r, :n_q]
                if use_db:
                    db.full_device(dq, view)
                else:
                    m.compare.compare_device(dr, dq, view, form)
                g = buf.cpu().numpy().view(np.uint32)
                assert np.array_equal(g[:n_r, :n_q], exp), (form, flags, use_db)
                g[:n_r, :n_q] = 0xFFFFFFFF
                assert (g == 0xFFFFFFFF).all(), (form, flags, use_db, "write outside the view")


@pytest.mark.parametrize("form", ["tensor_f4", "tensor_i8", "popc"])
def test_threshold_capacity_overflow(rng, form):
    """Threshold hits beyond `capacity` are counted but never written past the
    caller's buffers (poisoned tails stay intact), and threshold_hits' second pass
    with the exact count returns the oracle's hit list."""
    m = fb()
    from paper_1707_00516_b200 import _native
    from paper_1707_00516_b200.compare import threshold_hits
    from paper_1707_00516_b200.search import KnownDatabase

    L = 1024
    r, _ = rand_words(rng, 3000, 16, 64, L)
    q, _ = rand_words(rng, 70, 16, 64, L)
    exp = oracle.naive(r, q)
    thr = int(np.percentile(exp, 0.5))
    jj, ii = np.nonzero(exp.T <= thr)
    assert len(jj) > 200
    db = KnownDatabase(r, L, formulation=form)
    dq = m.DevicePanel.from_words(q, L)
    cap = 50
    dev = dq.rows.device
    for use_db in (True, False):
        hq = torch.full((cap + 64,), -7, dtype=torch.int32, device=dev)
        hr = torch.full((cap + 64,), -7, dtype=torch.int64, device=dev)
        hs = torch.full((cap + 64,), -7, dtype=torch.int32, device=dev)
        count = torch.zeros(1, dtype=torch.int64, device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        if use_db:
            rc = _native.lib().fastid_db_compare_threshold(
                db.image.handle, dq.rows.data_ptr(), dq.n_profiles, thr, 0,
                hq.data_ptr(), hr.data_ptr(), hs.data_ptr(), cap, count.data_ptr(), stream)
        else:
            dr = db.panel
            rc = _native.lib().fastid_compare_threshold(
                dr.rows.data_ptr(), dr.n_profiles, dq.rows.data_ptr(), dq.n_profiles, dr.stride, dr.bit_length, thr,
                0, hq.data_ptr(), hr.data_ptr(), hs.data_ptr(), cap, count.data_ptr(),
                _native.formulation_code(form), stream)
        assert rc == 0, _native.lib().fastid_last_error()
        torch.cuda.synchronize()
        assert int(count.item()) == len(jj)
        assert (hq[cap:] == -7).all() and (hr[cap:] == -7).all() and (hs[cap:] == -7).all()
        # the written prefix holds genuine hits
        got = set(zip(hq[:cap].cpu().tolist(), hr[:cap].cpu().tolist()))
        assert got <= set(zip(jj.tolist(), ii.tolist()))
    res = threshold_hits(db.panel, dq, thr, capacity=cap, formulation=form)
    assert np.array_equal(res.query, jj) and np.array_equal(res.ref, ii)
    assert np.array_equal(res.score, exp.T[jj, ii])


@pytest.mark.parametrize("form", ["tensor_f4", "tensor_i8", "popc"])
def test_topk_writes_stay_in_workspace(rng, form):
    """Top-k with exactly the advertised workspace (a view into a poisoned larger
    buffer) and output views: nothing past the workspace or outside the outputs is
    written. 600 unknowns = 3 pair groups, so the mxf4 path also runs the spare-pair
    grid (its list slot is part of the advertised size)."""
    m = fb()
    from paper_1707_00516_b200.compare import topk_workspace_bytes
    from paper_1707_00516_b200.search import KnownDatabase

    L, n_r, n_q, k = 1024, 100_000, 600, 16
    r, _ = rand_words(rng, n_r, 16, 64, L)
    q, _ = rand_words(rng, n_q, 16, 64, L)
    q[:40] = r[rng.integers(0, n_r, 40)]
    db = KnownDatabase(r, L, formulation=form)
    dq = m.DevicePanel.from_words(q, L)
    dev = dq.rows.device
    need = topk_workspace_bytes(n_r, n_q, k, form)
    ws_full = torch.full((need + 8192,), 0xAB, dtype=torch.uint8, device=dev)
    s_full = torch.full((n_q + 8, k), -7, dtype=torch.int32, device=dev)
    x_full = torch.full((n_q + 8, k), -7, dtype=torch.int64, device=dev)
    out = (s_full[:n_q], x_full[:n_q])
    s, x = db.topk_device(dq, k, None, ws_full[:need], out)
    torch.cuda.synchronize()
    assert (ws_full[need:] == 0xAB).all(), "write past the advertised workspace"
    assert (s_full[n_q:] == -7).all() and (x_full[n_q:] == -7).all(), "write past the outputs"
    es, ex, _ = oracle.topk(r, q, k)
    assert np.array_equal(s.cpu().numpy().view(np.uint32), es) and np.array_equal(x.cpu().numpy(), ex)


@pytest.mark.parametrize("n_q", [1, 100, 128])
def test_popc_topk_few_unknowns_many_knowns(rng, n_q):
    """CUDA-core top-k with one unknown group (<= 128 unknowns) and >= 80k knowns:
    the slice count is capped so the partial lists stay within the merge's
    768-list capacity; the result equals the oracle."""
    m = fb()
    L, n_r = 256, 90_000
    r, _ = rand_words(rng, n_r, 4, 64, L)
    q, _ = rand_words(rng, n_q, 4, 64, L)
    q[: max(1, n_q // 3)] = r[rng.integers(0, n_r, max(1, n_q // 3))]
    R, Q = m.Panel(tuple(range(n_r)), r, L), m.Panel(tuple(range(n_q)), q, L)
    res = m.topk(R, Q, 16, formulation="popc")
    es, ex, _ = oracle.topk(r, q, 16)
    assert np.array_equal(res.scores, es) and np.array_equal(res.index, ex)


@pytest.mark.parametrize("n_r,n_q", [(22_222, 300), (38_477, 2048), (192 * 37 * 2 + 1, 512)])
def test_dual_tile_pairs_streamed_unknowns(rng, n_r, n_q):
    """Dual-tile CTA pairs (streamed unknowns, L > 2048: each A stage feeds two
    known tiles): slices with odd and even tile counts, a one-tile remainder, the
    spare-pair grid (2048 unknowns: 72 regular pairs + 2 spares), ragged unknown
    groups -- top-k, threshold and the full matrix equal the oracle."""
    m = fb()
    from paper_1707_00516_b200.search import KnownDatabase

    L = 5000
    nw = -(-L // 64)
    r, _ = rand_words(rng, n_r, nw, 64, L)
    q, _ = rand_words(rng, n_q, nw, 64, L)
    q[:40] = r[rng.integers(0, n_r, 40)]
    r[-2:] = r[:2]  # ties across the first and last tiles
    db = KnownDatabase(r, L, formulation="tensor_f4")
    for k in (16, 5):
        s, x = db.search_words(q, k)
        es, ex, _ = oracle.topk(r, q, k, 0xFFFFFFFE)
        assert np.array_equal(s, es), (n_r, n_q, k)
        assert np.array_equal(x, ex), (n_r, n_q, k)
    if n_r * n_q <= 50_000_000:
        exp = oracle.blocked(r, np.ascontiguousarray(q.T), 64, 16, os.cpu_count() or 1)
        thr = int(np.percentile(exp[:, :8], 1))
        hits = db.threshold(m.Panel(tuple(range(n_q)), q, L), thr)
        hq, hr, hs = oracle.threshold_from_matrix(exp, thr)
        assert np.array_equal(hits.query, hq) and np.array_equal(hits.ref, hr) and np.array_equal(hits.score, hs)
        full = db.full_device(m.DevicePanel.from_words(q, L)).cpu().numpy().view(np.uint32)
        assert np.array_equal(full, exp)


def test_search_many_pipelined(rng):
    """KnownDatabase.search_many (batch i+1 staged before batch i is read back):
    every batch's lists equal the oracle's, across changing contents, a changing
    batch shape (new stagers mid-stream) and k."""
    from paper_1707_00516_b200.search import KnownDatabase

    L, n_r = 1024, 20_000
    r, _ = rand_words(rng, n_r, 16, 64, L)
    db = KnownDatabase(r, L)
    batches = []
    for n_q in (256, 256, 100, 256, 256):
        q, _ = rand_words(rng, n_q, 16, 64, L)
        q[:10] = r[rng.integers(0, n_r, 10)]
        batches.append(q)
    got = list(db.search_many(batches, 8))
    assert len(got) == len(batches)
    for q, (s, x) in zip(batches, got):
        es, ex, _ = oracle.topk(r, q, 8, 0xFFFFFFFE)
        assert np.array_equal(s, es) and np.array_equal(x, ex)
    assert list(db.search_many([], 8)) == []


@pytest.mark.parametrize("n_r,n_q,L", [(30_000, 2048, 1024), (9_000, 100, 5000), (500, 1, 1024)])
def test_graphed_search(rng, n_r, n_q, L):
    """The host-buffer top-k captured as one CUDA graph (H2D, encode, compare +
    top-k incl. the spare grid, merge, D2H): replays with new unknowns equal the
    oracle; wrong shapes and nonzero padding are rejected as search_words does."""
    m = fb()
    from paper_1707_00516_b200.search import KnownDatabase

    nw = -(-L // 64)
    r, _ = rand_words(rng, n_r, nw, 64, L)
    db = KnownDatabase(r, L)
    g = db.graphed_search(n_q, 16)
    for _ in range(3):
        q, _ = rand_words(rng, n_q, nw, 64, L)
        q[: min(8, n_q)] = r[rng.integers(0, n_r, min(8, n_q))]
        s, x = g.run(q)
        es, ex, _ = oracle.topk(r, q, 16, 0xFFFFFFFE)
        assert np.array_equal(s, es) and np.array_equal(x, ex)
    with pytest.raises(m.PanelMismatchError):
        g.run(np.zeros((n_q + 1, nw), np.uint64))
    if L % 64:
        bad = np.zeros((n_q, nw), np.uint64)
        bad[0, -1] = np.uint64(1)
        with pytest.raises(m.CorruptProfileError):
            g.run(bad)


@pytest.mark.parametrize("n_r,n_q,L,chunk", [(40_000, 300, 1024, 192 * 40), (12_000, 64, 5000, 192 * 9),
                                             (3_000, 2048, 1024, 192)])
def test_chunked_image(rng, n_r, n_q, L, chunk):
    """A panel searched through a chunked tensor image (one reusable image buffer,
    each chunk built in turn, fastid_db_create_in): top-k, full matrix and
    threshold hits equal the oracle across chunk boundaries, with a ref_base
    offset and ties that straddle chunks."""
    m = fb()
    from paper_1707_00516_b200.search import ChunkedImage, KnownDatabase

    nw = -(-L // 64)
    r, _ = rand_words(rng, n_r, nw, 64, L)
    q, _ = rand_words(rng, n_q, nw, 64, L)
    q[:20] = r[rng.integers(0, n_r, 20)]
    r[-2:] = r[:2]
    db = KnownDatabase(r, L, ref_base=5, image_chunk_rows=chunk)
    assert isinstance(db.image, ChunkedImage)
    db.chunked_min_queries = 1  # every batch through the chunks (the default sends small batches packed)
    for k in (16, 3):
        s, x = db.search_words(q, k)
        es, ex, _ = oracle.topk(r, q, k, 0xFFFFFFFE)
        assert np.array_equal(s, es) and np.array_equal(x, np.where(ex >= 0, ex + 5, -1)), k
    if n_r * n_q <= 40_000_000:
        exp = oracle.blocked(r, np.ascontiguousarray(q.T), 64, 16, os.cpu_count() or 1)
        full = db.full_device(m.DevicePanel.from_words(q, L)).cpu().numpy().view(np.uint32)
        assert np.array_equal(full, exp)
        thr = int(np.percentile(exp[:, :4], 1))
        hits = db.threshold(m.Panel(tuple(range(n_q)), q, L), thr)
        hq, hr, hs = oracle.threshold_from_matrix(exp, thr)
        assert np.array_equal(hits.query, hq) and np.array_equal(hits.ref, hr + 5) and np.array_equal(hits.score, hs)


def test_chunked_image_small_batches_use_packed_operands(rng):
    """Below CHUNKED_IMAGE_MIN_QUERIES a database on a chunked image answers through
    the packed-operand kernels (cheaper than building every chunk's image): same result."""
    from paper_1707_00516_b200.search import KnownDatabase

    L = 1024
    r, _ = rand_words(rng, 20_000, 16, 64, L)
    q, _ = rand_words(rng, 40, 16, 64, L)
    db = KnownDatabase(r, L, image_chunk_rows=192 * 7)
    assert not db._chunked_for(40)
    s, x = db.search_words(q, 8)
    es, ex, _ = oracle.topk(r, q, 8, 0xFFFFFFFE)
    assert np.array_equal(s, es) and np.array_equal(x, ex)


@pytest.mark.parametrize("n_q", [1, 2, 7, 16])
@pytest.mark.parametrize("L,width", [(1024, 64), (777, 32), (5000, 64), (64, 64)])
def test_popc_scan_few_unknowns(rng, n_q, L, width):
    """The CUDA-core scan for <= 16 unknowns (one packed row per lane, per-warp
    lists across the lanes, a shared bound, a per-CTA merge): top-k for k = 1, 16,
    32 with and without a score cap, planted copies and duplicate knowns (ties
    across warps and CTAs) equal the oracle."""
    m = fb()
    n_r = 150_003
    nw = -(-L // width)
    r, _ = rand_words(rng, n_r, nw, width, L)
    q, _ = rand_words(rng, n_q, nw, width, L)
    q[0] = r[77]
    r[100_000] = r[77]  # the same known twice: a tie at score 0
    r[5:9] = r[150_000]
    R, Q = m.Panel(tuple(range(n_r)), r, L), m.Panel(tuple(range(n_q)), q, L)
    for k, ms in ((16, None), (1, None), (32, L // 5), (5, 0)):
        res = m.topk(R, Q, k, max_score=ms, formulation="popc")
        es, ex, _ = oracle.topk(r, q, k, 0xFFFFFFFE if ms is None else ms)
        assert np.array_equal(res.scores, es) and np.array_equal(res.index, ex), (k, ms)
    assert 77 in res.index[0] or k < 2


@pytest.mark.parametrize("n_q", [1, 3, 16])
@pytest.mark.parametrize("L", [1024, 5000, 130])
def test_popc_scan_threshold(rng, n_q, L):
    """Threshold hits of <= 16 unknowns through the CUDA-core scan (one packed row
    per lane, warp-aggregated hit slots): the (unknown, known, score) list equals
    the oracle's, with planted copies, duplicate knowns and a capacity overflow
    that the two-pass wrapper recovers from."""
    m = fb()
    n_r = 120_001
    nw = -(-L // 64)
    r, _ = rand_words(rng, n_r, nw, 64, L)
    q, _ = rand_words(rng, n_q, nw, 64, L)
    q[0] = r[9]
    r[60_000] = r[9]
    R, Q = m.Panel(tuple(range(n_r)), r, L), m.Panel(tuple(range(n_q)), q, L)
    exp = oracle.naive(r, q) if n_r * n_q * L <= 3e9 else oracle.blocked(r, np.ascontiguousarray(q.T), 64, 16, os.cpu_count() or 1)
    t = int(np.percentile(exp, 0.5))
    hits = m.threshold_hits(R, Q, t, capacity=7, formulation="popc")
    hq, hr, hs = oracle.threshold_from_matrix(exp, t)
    assert np.array_equal(hits.query, hq) and np.array_equal(hits.ref, hr) and np.array_equal(hits.score, hs)
