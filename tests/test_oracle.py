"""Pin the CPU oracle against the reference's own outputs (tests/golden) and
against an independent numpy restatement.  CPU only."""

import numpy as np
import pytest

import oracle

from conftest import rand_words


def test_oracle_matches_reference_goldens(kernel_cases):
    assert len(kernel_cases) >= 20
    for c in kernel_cases:
        got = oracle.naive(c["refs"], c["queries"])
        assert np.array_equal(got, c["scores"]), c["name"]


def test_blocked_oracle_matches_goldens(kernel_cases):
    for c in kernel_cases:
        qt = np.ascontiguousarray(c["queries"].T)
        for block, cells, workers in ((16, 1, 1), (32, 3, 2), (64, 16, 8)):
            got = oracle.blocked(c["refs"], qt, block, cells, workers)
            assert np.array_equal(got, c["scores"]), (c["name"], block, workers)


def test_numpy_restatement_matches_goldens(kernel_cases):
    for c in kernel_cases:
        if c["refs"].shape[0] * c["queries"].shape[0] * c["refs"].shape[1] > 5e6:
            continue
        assert np.array_equal(oracle.np_scores(c["refs"], c["queries"]), c["scores"]), c["name"]


def test_golden_4x4_and_worked_word(kernel_cases):
    by = {c["name"]: c for c in kernel_cases}
    assert by["golden_4x4"]["scores"].tolist() == [[0, 4, 2, 2], [4, 0, 4, 2], [4, 4, 6, 4], [0, 0, 0, 0]]
    assert by["worked_word"]["scores"].tolist() == [[3]]
    assert oracle.score_word(0x06001440, 0x00000440) == 3
    # popcount(0x06001440) is 5 (test_kernel.py:58-60), not the 6 of SPEC.md:433
    assert oracle.score_word(0x06001440, 0) == 5
    assert by["all_ones_96"]["scores"][0].tolist() == [96] * 5


def test_golden_csv_bytes(kernel_cases):
    # the reference's golden CSV (pkg/tests/golden/scores_4x4.csv) restated from the matrix
    s = {c["name"]: c for c in kernel_cases}["golden_4x4"]["scores"]
    lines = ["ref_id," + ",".join(f"q{j}" for j in range(4))]
    lines += [f"r{i}," + ",".join(str(int(v)) for v in s[i]) for i in range(4)]
    assert "\n".join(lines) + "\n" == "ref_id,q0,q1,q2,q3\nr0,0,4,2,2\nr1,4,0,4,2\nr2,4,4,6,4\nr3,0,0,0,0\n"


def test_pack_matches_reference(pack_cases):
    for L in pack_cases["lengths"]:
        bits = pack_cases[f"L{L}_bits"]
        for width in (32, 64):
            assert np.array_equal(oracle.pack_bits(bits, width), pack_cases[f"L{L}_w{width}"]), (L, width)
    assert oracle.pack_bits(pack_cases["example_bits"], 32).tolist() == [[100668480]]


def test_topk_oracle_matches_reference_derivation(topk_cases):
    for c in topk_cases:
        k = int(c["k"])
        s, x, cnt = oracle.topk(c["refs"], c["queries"], k)
        assert np.array_equal(s, c["top_scores"]), c["name"]
        assert np.array_equal(x, c["top_index"]), c["name"]
        assert (cnt == k).all()
        hq, hr, hs, n = oracle.threshold(c["refs"], c["queries"], int(c["threshold"]))
        assert n == len(c["hit_query"])
        assert np.array_equal(hq, c["hit_query"]) and np.array_equal(hr, c["hit_ref"])
        assert np.array_equal(hs, c["hit_score"])


def test_scan_oracle_matches_reference_derivation(topk_cases):
    """The database-scale oracle (row ranges on all threads, merged in row order)
    reproduces the reference-derived top-k and threshold goldens."""
    for c in topk_cases:
        k = int(c["k"])
        for workers in (1, 3, 8):
            top, hits = oracle.scan(c["refs"], c["queries"], k, threshold=int(c["threshold"]), workers=workers)
            assert np.array_equal(top[0], c["top_scores"]) and np.array_equal(top[1], c["top_index"]), c["name"]
            assert np.array_equal(hits[0], c["hit_query"]) and np.array_equal(hits[1], c["hit_ref"])
            assert np.array_equal(hits[2], c["hit_score"]) and hits[3] == len(c["hit_query"])


@pytest.mark.parametrize("width", [32, 64])
def test_scan_oracle_matches_topk_oracle(rng, width):
    """Ties across row ranges, score caps, k larger than the panel, 32-bit words,
    partial row blocks: the scan oracle equals the per-unknown oracle."""
    for n_r, n_q, L in ((3, 4, 64), (700, 19, 1000), (2049, 7, 5000)):
        nw = -(-L // width)
        r, _ = rand_words(rng, n_r, nw, width, L)
        q, _ = rand_words(rng, n_q, nw, width, L)
        r[n_r // 2:] = r[: n_r - n_r // 2]  # every row duplicated across the two halves
        q[: n_q // 2] = r[rng.integers(0, n_r, n_q // 2)]
        for k, ms in ((1, 0xFFFFFFFF), (16, 0xFFFFFFFF), (32, L // 3), (5, 0)):
            top, _ = oracle.scan(r, q, k, ms, workers=6)
            for a, b in zip(top, oracle.topk(r, q, k, ms)):
                assert np.array_equal(a, b), (n_r, n_q, L, k, ms)
        _, hits = oracle.scan(r, q, 0, threshold=L // 4, workers=5)
        exp = oracle.threshold(r, q, L // 4)
        assert hits[3] == exp[3] and all(np.array_equal(a, b) for a, b in zip(hits[:3], exp[:3]))


def test_topk_max_score_and_small_panels(rng):
    r, L = rand_words(rng, 50, 2, 64)
    q, _ = rand_words(rng, 9, 2, 64)
    full = oracle.naive(r, q)
    for k, ms in ((1, 0xFFFFFFFF), (5, 60), (32, 64), (8, 0)):
        got = oracle.topk(r, q, k, ms)
        exp = oracle.topk_from_matrix(full, k, ms)
        for a, b in zip(got, exp):
            assert np.array_equal(a, b)


def test_checksum_convention_matches_reference(checksum_rows):
    row = next(r for r in checksum_rows if r["label"].startswith("baseline_config1"))
    refs = oracle.synth_words(row["n_refs"], row["n_words"], row["word_width"], row["seed"], 0)
    queries = oracle.synth_words(row["n_queries"], row["n_words"], row["word_width"], row["seed"], 1)
    scores = oracle.blocked(refs, np.ascontiguousarray(queries.T), 64, 16, 8)
    assert oracle.score_checksum(scores) == row["checksum"]


@pytest.mark.parametrize("width", [32, 64])
def test_c_and_numpy_agree_random(rng, width):
    for L in (1, 33, 200, 1000):
        nw = -(-L // width)
        r, _ = rand_words(rng, 40, nw, width, L)
        q, _ = rand_words(rng, 23, nw, width, L)
        assert np.array_equal(oracle.naive(r, q), oracle.np_scores(r, q))


def fidm_bytes(scores: np.ndarray) -> bytes:
    """The packed-binary score file (io.py:29-31 header, then row-major <u4 cells), restated."""
    import struct

    n_r, n_q = scores.shape
    return struct.pack("<4sBQQ", b"FIDM", 1, n_r, n_q) + np.ascontiguousarray(scores, "<u4").tobytes()


def test_fidm_format_matches_reference_files():
    """The oracle's scores in the FIDM layout equal the files the reference's own
    write_scores produced (tests/golden/fidm_cases.npz)."""
    from conftest import GOLDEN

    d = np.load(GOLDEN / "fidm_cases.npz")
    for name in ("golden_4x4", "rand_37x23_L100"):
        r, q = d[f"{name}__refs"], d[f"{name}__queries"]
        assert fidm_bytes(oracle.naive(r, q)) == d[f"{name}__fidm"].tobytes(), name


def test_operator_restatements(rng):
    """np_scores_op: "andnot" is Eq. 1 (== the pinned C oracle); "and" / "xor"
    follow their definitions and the identity the tensor epilogue uses
    (xor = popc(r) + popc(q) - 2 and).  AND and XOR are parity-unpinned
    extensions (the reference computes AND-NOT only)."""
    r, _ = rand_words(rng, 70, 5, 64, 300)
    q, _ = rand_words(rng, 9, 5, 64, 300)
    assert np.array_equal(oracle.np_scores_op(r, q, "andnot"), oracle.naive(r, q))
    both = oracle.np_scores_op(r, q, "and", block=16).astype(np.int64)
    pr = np.bitwise_count(r).sum(axis=1, dtype=np.int64)
    pq = np.bitwise_count(q).sum(axis=1, dtype=np.int64)
    assert np.array_equal(oracle.np_scores_op(r, q, "xor"), pr[:, None] + pq[None, :] - 2 * both)
    assert np.array_equal(oracle.np_scores_op(r, q, "andnot").astype(np.int64), pr[:, None] - both)
    with pytest.raises(KeyError):
        oracle.np_scores_op(r, q, "or")


@pytest.mark.parametrize("op", ["andnot", "and", "xor"])
@pytest.mark.parametrize("width", [32, 64])
def test_scan_operators_match_numpy(rng, op, width):
    """oracle.scan(op=...) (the C scan bench.py verifies with) == the numpy
    operator restatement, top-k and threshold."""
    L = 700
    nw = -(-L // width)
    r, _ = rand_words(rng, 3000, nw, width, L)
    q, _ = rand_words(rng, 7, nw, width, L)
    exp = oracle.np_scores_op(r, q, op)
    t = int(np.percentile(exp, 1))
    (s, x, _), (hq, hr, hs, n) = oracle.scan(r, q, 9, threshold=t, workers=3, op=op)
    es, ex, _ = oracle.topk_from_matrix(exp, 9)
    assert np.array_equal(s, es) and np.array_equal(x, ex)
    eq, er, esc = oracle.threshold_from_matrix(exp, t)
    assert n == len(eq) and np.array_equal(hq, eq) and np.array_equal(hr, er) and np.array_equal(hs, esc)
