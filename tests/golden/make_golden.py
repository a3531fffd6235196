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
* panel_cases.json  -- panel texts (valid and malformed) and what the
                       reference's ``io.load_panel`` returns for them at word
                       widths 32 and 64: ids, bit length, hex words -- or the
                       exception type and message (io.py:45-127);
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


def panel_texts():
    rng = np.random.default_rng(0x1A57)
    texts = {
        "worked_example": "#bits=32\nS1\t06001440\n",
        "empty_body": "#bits=64\n",
        "ids_in_order": "#bits=8\nba\t00\nc\tFF\nab\t0F\n",
        "comments": "# comment\n#bits=8\n# another\nx\tA5\n",
        "missing_header": "S1\t06001440\n",
        "before_header": "S1\t00\n#bits=8\n",
        "duplicate_id": "#bits=8\na\t00\na\tFF\n",
        "length_mismatch": "#bits=8\na\t00\nb\t0000\n",
        "tail_padding": "#bits=4\na\t01\n",
        "surplus_padding": "#bits=32\na\t0600144000000001\n",
        "comma_id": "#bits=8\na,b\t00\n",
        "bad_hex": "#bits=8\na\tZZ\n",
        "bad_hex_mixed": "#bits=8\na\t0q\nb\tz!\n",
        "short_hex": "#bits=64\na\t00\n",
        "duplicate_header": "#bits=8\n#bits=8\na\t00\n",
        "duplicate_header_after_profile": "#bits=8\na\t00\n#bits=16\n",
        "bad_header": "#bits=abc\n",
        "zero_bits": "#bits=0\n",
        "negative_bits": "#bits=-3\n",
        "header_spaces_underscore": "#  bits= 1_6 \na\tFFFF\n",
        "three_fields": "#bits=8\na\t00\tff\n",
        "no_tab": "#bits=8\na 00\n",
        "empty_id": "#bits=8\n\t00\n",
        "empty_hex_short": "#bits=8\na\t\n",
        "crlf_and_cr": "#bits=12\r\na\tABC\r\nb\t123\rc\tfff\n\n\r\n",
        "lowercase_zero_extend_truncate": "#bits=40\np1\tdeadbeef12\np2\t0000000000\n",
        "truncate_zero_surplus": "#bits=8\np\tA500000000000000000000\n",
        "dup_vs_bad_hex_same_line": "#bits=8\na\t00\na\tZZ\n",
        "error_order_first_line_wins": "#bits=8\na\t00\nb\tZZ\nb\t00\n",
        "missing_header_no_profiles": "# only a comment\n\n",
        "unicode_id": "#bits=8\n\u00e9t\u00e9\t7F\n",
    }
    for L in (1, 50, 64, 100, 1000):
        n_digits = -(-L // 4)
        lines = [f"#bits={L}", "# generated"]
        for i in range(60):
            bits = rng.integers(0, 2, L)
            val = int("".join(map(str, bits)), 2) << (4 * n_digits - L) if L else 0
            h = f"{val:0{n_digits}x}" if i % 2 else f"{val:0{n_digits}X}"
            h = h + "0" * (L % 3 + (L == 64))  # surplus zero digits (same on every line): truncated
            lines.append(f"id{i}_{L}\t{h}")
            if i % 11 == 5:
                lines.append("")
        texts[f"random_L{L}"] = "\n".join(lines) + "\n"
    return texts


def panel_cases():
    from fastid import errors as ref_errors
    from fastid import io as ref_io

    out = []
    for name, text in panel_texts().items():
        row = {"name": name, "text": text, "results": {}}
        for width in (32, 64):
            with tempfile.TemporaryDirectory() as d:
                path = Path(d) / "p.panel"
                path.write_bytes(text.encode("utf-8"))
                try:
                    p = ref_io.load_panel(path, width)
                    row["results"][str(width)] = {"ids": list(p.ids), "bit_length": p.bit_length,
                                                  "words": [[f"{int(w):x}" for w in r] for r in p.words]}
                except (ref_errors.PanelFormatError, ref_errors.CorruptProfileError) as e:
                    msg = str(e).replace(str(path), "<path>")
                    row["results"][str(width)] = {"error": type(e).__name__, "message": msg}
        out.append(row)
    (OUT / "panel_cases.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    panel_cases()
    fidm_cases()
    kernel_cases()
    topk_cases()
    pack_cases()
    genotypes()
    checksums()
