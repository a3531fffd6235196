"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container only (the reference is not present on GPU boxes):

    python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src
(numba's cache is redirected to /tmp so nothing is written into the
reference tree) and records, for a set of seeded inputs:

* kernel_cases.npz  -- refs / queries words, bit length, and the score matrix
                       from ``compare_naive`` (kernel.py:283-292), each also
                       checked against ``compare_blocked`` (kernel.py:295-314)
                       at several tile/worker settings before being saved;
* topk_cases.npz    -- planted near-copy panels plus the top-k / threshold
                       derivations of the reference's own score matrix
                       (ordering: score asc, known index asc);
* pack_cases.npz    -- 0/1 bit matrices and ``codec.pack`` words at widths
                       32 and 64 (codec.py:118-127);
* checksums.json    -- ``bench.score_checksum`` (bench.py:57-58) of
                       ``compare_blocked`` on ``synth_panel`` inputs
                       (bench.py:41-54), incl. BASELINE config 1;
* genotype.json     -- ``codec.encode_genotype`` examples (codec.py:99-115);
* fidm_cases.npz    -- panels and the packed-binary score files the reference's
                       own ``io.write_scores(..., ScoreOutput(path, "binary"))``
                       writes for them (io.py:160-172), byte for byte.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_cache_"))
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF_SRC))

import numpy as np  # noqa: E402

from fastid import codec, kernel  # noqa: E402
from fastid.bench import score_checksum, synth_panel  # noqa: E402

OUT = Path(__file__).resolve().parent


def rand_words(rng, n, n_words, width, bit_length=None):
    dtype = np.uint32 if width == 32 else np.uint64
    w = rng.integers(0, 2**width, size=(n, n_words), dtype=dtype)
    bit_length = bit_length or n_words * width
    tail = bit_length % width
    if tail and n_words:
        w[:, -1] &= dtype((2**width - 1) ^ ((1 << (width - tail)) - 1))
    return w, bit_length


def panel(words, bit_length, prefix):
    return kernel.Panel(tuple(f"{prefix}{i}" for i in range(words.shape[0])), words, bit_length)


def reference_scores(refs_w, q_w, bit_length):
    refs = panel(refs_w, bit_length, "r")
    queries = panel(q_w, bit_length, "q")
    expected = kernel.compare_naive(refs, queries).scores
    layout = kernel.relayout_queries(queries)
    for tile, workers in ((16, 1), (32, 2), (64, 8)):
        got = kernel.compare_blocked(refs, layout, kernel.TileConfig(tile), workers).scores
        assert np.array_equal(got, expected)
    return np.array(expected, dtype=np.uint32)


def kernel_cases():
    rng = np.random.default_rng(20260809)
    cases = []

    def add(name, r, q, L):
        cases.append((name, r, q, L, reference_scores(r, q, L)))

    # acceptance criterion 8 (test_acceptance.py:234-256), L = 8, u32
    r = np.array([[0xF0000000], [0x0F000000], [0xFF000000], [0]], dtype=np.uint32)
    q = np.array([[0xF0000000], [0x0F000000], [0xA0000000], [0xCC000000]], dtype=np.uint32)
    add("golden_4x4", r, q, 8)
    # worked word (test_kernel.py:35-38)
    add("worked_word", np.array([[0x06001440]], np.uint32), np.array([[0x00000440]], np.uint32), 32)
    # single zero profile (test_kernel.py:155-159)
    add("zero_1x1", np.zeros((1, 1), np.uint32), np.zeros((1, 1), np.uint32), 32)
    # all-ones ref row at L = 96 (test_kernel.py:200-210)
    ones = np.zeros((2, 2), np.uint64)
    ones[0] = [2**64 - 1, np.uint64(0xFFFFFFFF) << np.uint64(32)]
    add("all_ones_96", ones, np.zeros((5, 2), np.uint64), 96)
    # partial last word L = 50 (test_kernel.py:145-150)
    a, L = rand_words(rng, 6, 2, 32, 50)
    b, _ = rand_words(rng, 5, 2, 32, 50)
    add("partial_50_u32", a, b, L)
    for width in (32, 64):
        a, L = rand_words(rng, 9, 2, width)
        b, _ = rand_words(rng, 7, 2, width)
        add(f"bitloop_9x7_w{width}", a, b, L)
    a, L = rand_words(rng, 12, 3, 64)
    add("self_12", a, a.copy(), L)
    # tile-edge and multi-word shapes for the device kernels
    for name, n_r, n_q, L, width in (
        ("edge_300x200_L1024_w64", 300, 200, 1024, 64),
        ("edge_257x129_L5000_w64", 257, 129, 5000, 64),
        ("edge_130x67_L1000_w32", 130, 67, 1000, 32),
        ("edge_513x300_L2048_w32", 513, 300, 2048, 32),
        ("edge_1x1_L1", 1, 1, 1, 64),
        ("edge_77x33_L127_w32", 77, 33, 127, 32),
        ("edge_129x257_L40000_w64", 129, 257, 40000, 64),
    ):
        nw = -(-L // width)
        a, _ = rand_words(rng, n_r, nw, width, L)
        b, _ = rand_words(rng, n_q, nw, width, L)
        add(name, a, b, L)
    # criterion-2 style draws (test_acceptance.py:51-80), seed 0xFA57
    crng = np.random.default_rng(0xFA57)
    for t in range(12):
        n_words = int(crng.choice([4, 8, 16]))
        n_r = int(crng.integers(1, 257))
        n_q = int(crng.integers(1, 257))
        a = crng.integers(0, 2**32, (n_r, n_words), dtype=np.uint32)
        b = crng.integers(0, 2**32, (n_q, n_words), dtype=np.uint32)
        add(f"c2_draw{t}", a, b, n_words * 32)

    arrays = {}
    names = []
    for idx, (name, r, q, L, s) in enumerate(cases):
        names.append(name)
        arrays[f"{idx}_refs"] = r
        arrays[f"{idx}_queries"] = q
        arrays[f"{idx}_bits"] = np.array(L, dtype=np.int64)
        arrays[f"{idx}_scores"] = s
    arrays["names"] = np.array(names)
    np.savez_compressed(OUT / "kernel_cases.npz", **arrays)
    print(f"kernel_cases.npz: {len(cases)} cases")


def planted(rng, n_r, n_q, L, width, flips):
    nw = -(-L // width)
    refs, _ = rand_words(rng, n_r, nw, width, L)
    src = rng.integers(0, n_r, n_q)
    q = refs[src].copy()
    for j in range(n_q):
        for _ in range(int(rng.integers(0, flips + 1))):
            bit = int(rng.integers(0, L))
            q[j, bit // width] ^= q.dtype.type(1) << q.dtype.type(width - 1 - bit % width)
    # duplicate some refs so ties on score exist (tie-break = known index)
    refs[n_r // 2 : n_r // 2 + 8] = refs[src[:8]]
    return refs, q, src


def topk_cases():
    rng = np.random.default_rng(0x70B1)
    arrays = {}
    names = []
    specs = (
        ("planted_2000x37_L1024_w64", 2000, 37, 1024, 64, 16, 16, 40),
        ("planted_1500x130_L5000_w64", 1500, 130, 5000, 64, 24, 8, 150),
        ("planted_700x64_L512_w32", 700, 64, 512, 32, 6, 32, 10),
    )
    for idx, (name, n_r, n_q, L, width, flips, k, thr) in enumerate(specs):
        refs, q, _ = planted(rng, n_r, n_q, L, width, flips)
        s = reference_scores(refs, q, L)
        order = np.lexsort((np.broadcast_to(np.arange(n_r)[:, None], s.shape), s), axis=0)
        top_idx = order[:k].T.astype(np.int64)
        top_s = np.take_along_axis(s, order[:k], axis=0).T.astype(np.uint32)
        hj, hi = np.nonzero(s.T <= thr)
        names.append(name)
        arrays[f"{idx}_refs"] = refs
        arrays[f"{idx}_queries"] = q
        arrays[f"{idx}_bits"] = np.array(L, dtype=np.int64)
        arrays[f"{idx}_k"] = np.array(k, dtype=np.int64)
        arrays[f"{idx}_top_scores"] = top_s
        arrays[f"{idx}_top_index"] = top_idx
        arrays[f"{idx}_threshold"] = np.array(thr, dtype=np.int64)
        arrays[f"{idx}_hit_query"] = hj.astype(np.uint32)
        arrays[f"{idx}_hit_ref"] = hi.astype(np.int64)
        arrays[f"{idx}_hit_score"] = s[hi, hj].astype(np.uint32)
    arrays["names"] = np.array(names)
    np.savez_compressed(OUT / "topk_cases.npz", **arrays)
    print(f"topk_cases.npz: {len(names)} cases")


def pack_cases():
    rng = np.random.default_rng(0xC0DE)
    arrays = {}
    lengths = (1, 8, 31, 32, 33, 50, 63, 64, 65, 100, 127, 128, 129, 1024, 5000)
    for L in lengths:
        bits = rng.integers(0, 2, size=(7, L), dtype=np.uint8)
        arrays[f"L{L}_bits"] = bits
        for width in (32, 64):
            words = np.array(
                [codec.pack(codec.ProfileBits(f"p{i}", bits[i]), width).words for i in range(7)],
                dtype=np.uint32 if width == 32 else np.uint64,
            )
            arrays[f"L{L}_w{width}"] = words
    # the paper's worked example (codec.py:3-6)
    ex = np.array([[int(c) for c in "00000110000000000001010001000000"]], dtype=np.uint8)
    arrays["example_bits"] = ex
    arrays["example_w32"] = np.array(
        [codec.pack(codec.ProfileBits("S1", ex[0]), 32).words], dtype=np.uint32
    )
    arrays["lengths"] = np.array(lengths, dtype=np.int64)
    np.savez_compressed(OUT / "pack_cases.npz", **arrays)
    print(f"pack_cases.npz: {len(lengths)} lengths")


def checksums():
    rows = []
    specs = (
        # (label, n_refs, n_queries, n_words, width, seed)
        ("baseline_config1_10000x64_L1024", 10_000, 64, 16, 64, 0),
        ("criterion5_100000x2048_w32", 100_000, 2048, 16, 32, 5),
        ("L5056_20000x300_w64", 20_000, 300, 79, 64, 3),
        ("L512_50000x1024_w32", 50_000, 1024, 16, 32, 7),
    )
    for label, n_r, n_q, nw, width, seed in specs:
        refs = synth_panel(n_r, nw, width, seed, 0, "r")
        queries = synth_panel(n_q, nw, width, seed, 1, "q")
        m = kernel.compare_blocked(
            refs, kernel.relayout_queries(queries), kernel.TileConfig(64), os.cpu_count() or 1
        )
        if n_r * n_q <= 1_000_000:
            assert np.array_equal(m.scores, kernel.compare_naive(refs, queries).scores)
        rows.append(
            {
                "label": label,
                "n_refs": n_r,
                "n_queries": n_q,
                "n_words": nw,
                "word_width": width,
                "seed": seed,
                "checksum": score_checksum(m.scores),
                "sum": int(m.scores.sum(dtype=np.uint64)),
            }
        )
        print(label, rows[-1]["checksum"])
    (OUT / "checksums.json").write_text(json.dumps(rows, indent=1) + "\n")


def genotypes():
    examples = [["MM"], ["mm"], ["Mm", "mM", "MM"], ["Mm", "mM"], ["mm", "Mm", "MM", "mM", "mm"]]
    rows = []
    for g in examples:
        bits = codec.encode_genotype(g).bits
        rows.append({"codes": g, "bits": [int(b) for b in bits],
                     "w32": list(codec.pack(codec.encode_genotype(g), 32).words)})
    (OUT / "genotype.json").write_text(json.dumps(rows, indent=1) + "\n")


def fidm_cases():
    from fastid import io as ref_io

    rng = np.random.default_rng(0xF1D)
    cases = {}
    r4 = np.array([[0xF0000000], [0x0F000000], [0xFF000000], [0x00000000]], np.uint32)
    q4 = np.array([[0xF0000000], [0x0F000000], [0xA0000000], [0xCC000000]], np.uint32)
    r_rand, _ = rand_words(rng, 37, 2, 64, 100)
    q_rand, _ = rand_words(rng, 23, 2, 64, 100)
    for name, r, q, L in (("golden_4x4", r4, q4, 8), ("rand_37x23_L100", r_rand, q_rand, 100)):
        m = kernel.compare_naive(panel(r, L, "r"), panel(q, L, "q"))
        with tempfile.TemporaryDirectory() as d:
            path = Path(d) / "scores.fidm"
            ref_io.write_scores(m, ref_io.ScoreOutput(path=str(path), format="binary"))
            blob = np.frombuffer(path.read_bytes(), np.uint8)
        cases[f"{name}__refs"] = r
        cases[f"{name}__queries"] = q
        cases[f"{name}__bits"] = np.array(L)
        cases[f"{name}__fidm"] = blob
    np.savez_compressed(OUT / "fidm_cases.npz", **cases)


if __name__ == "__main__":
    fidm_cases()
    kernel_cases()
    topk_cases()
    pack_cases()
    genotypes()
    checksums()
