"""CPU oracle for the FastID comparison path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module.  The
product package ``paper_1707_00516_b200`` never imports it: its compare entry
points fail loudly when the CUDA library is missing.

Two independent restatements of the reference algorithm live here:

* ``fastid_oracle.c`` (loaded with ctypes): Algorithm 2 as in
  ``_naive_kernel`` (/root/reference/pkg/src/fastid/kernel.py:224-235), the
  tiled thread-pool kernel as in ``_blocked_worker`` / ``run_blocked_kernel``
  (kernel.py:238-269, 317-347), ``codec.pack`` (codec.py:118-127) and the
  top-k / threshold derivations of the score matrix.
* numpy one-liners over ``np.bitwise_count`` (``np_scores`` etc.) used for
  small cases and to cross-check the C code.

Both are pinned against the reference itself through the fixtures in
``tests/golden`` (made by ``tests/golden/make_golden.py``, which imports the
reference package read-only).
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_build" / "libfastid_oracle.so"

_lib = None


def build() -> Path:
    """Compile the C oracle in-tree (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        vp, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint32
        L.oracle_naive.argtypes = [vp, i64, vp, i64, i64, i32, vp]
        L.oracle_naive.restype = i32
        L.oracle_blocked.argtypes = [vp, i64, vp, i64, i64, i32, i32, i32, i32, vp]
        L.oracle_blocked.restype = i32
        L.oracle_pack_bits.argtypes = [vp, i64, i64, i32, vp]
        L.oracle_pack_bits.restype = i32
        L.oracle_topk.argtypes = [vp, i64, vp, i64, i64, i32, i32, u32, i32, vp, vp, vp]
        L.oracle_topk.restype = i32
        L.oracle_threshold.argtypes = [vp, i64, vp, i64, i64, i32, u32, i64, vp, vp, vp]
        L.oracle_threshold.restype = i64
        L.oracle_scan.argtypes = [vp, i64, vp, i64, i64, i32, i32, u32, i32, u32, i32, vp, vp, vp, i64, vp, vp, vp]
        L.oracle_scan.restype = i64
        L.oracle_scan_op.argtypes = L.oracle_scan.argtypes + [i32]
        L.oracle_scan_op.restype = i64
        L.oracle_score_word.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.oracle_score_word.restype = u32
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _words(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    if a.dtype not in (np.uint32, np.uint64) or a.ndim != 2:
        raise ValueError("word arrays must be 2-D uint32/uint64")
    return a


# ---------------------------------------------------------------------------
# C restatement
# ---------------------------------------------------------------------------

def naive(refs: np.ndarray, queries: np.ndarray) -> np.ndarray:
    """compare_naive's matrix (kernel.py:283-292 -> _naive_kernel 224-235)."""
    refs, queries = _words(refs), _words(queries)
    assert refs.dtype == queries.dtype and refs.shape[1] == queries.shape[1]
    out = np.zeros((refs.shape[0], queries.shape[0]), dtype=np.uint32)
    if out.size:
        rc = lib().oracle_naive(_ptr(refs), refs.shape[0], _ptr(queries), queries.shape[0],
                                refs.shape[1], refs.dtype.itemsize * 8, _ptr(out))
        assert rc == 0
    return out


def blocked(refs: np.ndarray, queries_t: np.ndarray, block: int = 64, cells: int = 16,
            workers: int = 1) -> np.ndarray:
    """compare_blocked's matrix over the transposed query layout (kernel.py:295-347)."""
    refs, queries_t = _words(refs), _words(queries_t)
    out = np.zeros((refs.shape[0], queries_t.shape[1]), dtype=np.uint32)
    if out.size:
        rc = lib().oracle_blocked(_ptr(refs), refs.shape[0], _ptr(queries_t), queries_t.shape[1],
                                  refs.shape[1], refs.dtype.itemsize * 8, block, cells, workers,
                                  _ptr(out))
        assert rc == 0
    return out


def pack_bits(bits: np.ndarray, word_bits: int = 64) -> np.ndarray:
    """codec.pack over a (rows, L) 0/1 matrix (codec.py:118-127)."""
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    rows, length = bits.shape
    n_words = -(-length // word_bits)
    out = np.zeros((rows, n_words), dtype=np.uint64 if word_bits == 64 else np.uint32)
    rc = lib().oracle_pack_bits(_ptr(bits), rows, length, word_bits, _ptr(out))
    assert rc == 0
    return out


def topk(refs: np.ndarray, queries: np.ndarray, k: int, max_score: int = 0xFFFFFFFF,
         workers: int | None = None):
    """Per unknown j: first k of column j by (score asc, known index asc), score <= max_score.

    Returns (scores u32 [N_Q, k], index i64 [N_Q, k], counts i32 [N_Q]); missing
    slots hold 0xFFFFFFFF / -1.
    """
    refs, queries = _words(refs), _words(queries)
    nq = queries.shape[0]
    s = np.full((nq, k), 0xFFFFFFFF, dtype=np.uint32)
    x = np.full((nq, k), -1, dtype=np.int64)
    c = np.zeros(nq, dtype=np.int32)
    if nq:
        rc = lib().oracle_topk(_ptr(refs), refs.shape[0], _ptr(queries), nq, refs.shape[1],
                               refs.dtype.itemsize * 8, k, max_score,
                               workers or os.cpu_count() or 1, _ptr(s), _ptr(x), _ptr(c))
        assert rc == 0
    return s, x, c


def threshold(refs: np.ndarray, queries: np.ndarray, t: int, capacity: int | None = None):
    """All (unknown j, known i, score) with score <= t, ordered by (j, i)."""
    refs, queries = _words(refs), _words(queries)
    cap = capacity if capacity is not None else refs.shape[0] * queries.shape[0]
    hq = np.zeros(max(cap, 1), dtype=np.uint32)
    hr = np.zeros(max(cap, 1), dtype=np.int64)
    hs = np.zeros(max(cap, 1), dtype=np.uint32)
    n = lib().oracle_threshold(_ptr(refs), refs.shape[0], _ptr(queries), queries.shape[0],
                               refs.shape[1], refs.dtype.itemsize * 8, t, cap,
                               _ptr(hq), _ptr(hr), _ptr(hs))
    m = min(n, cap)
    return hq[:m].copy(), hr[:m].copy(), hs[:m].copy(), int(n)


_SCAN_OPS = {"andnot": 0, "and": 1, "xor": 2}


def scan(refs: np.ndarray, queries: np.ndarray, k: int = 0, max_score: int = 0xFFFFFFFF,
         threshold: int | None = None, capacity: int = 1 << 24, workers: int | None = None, op: str = "andnot"):
    """Database-scale derivations with all host threads (oracle_scan): the top-k
    of ``topk`` (k > 0) and/or the hits of ``threshold``, over row ranges merged
    in row order.  Returns (scores, index, counts) for k > 0 (else None) and
    (query, ref, score, total) when ``threshold`` is given (else None).  ``op``
    "and" / "xor" score popcount(r AND q) / popcount(r XOR q) instead of Eq. 1
    (operator extensions without a reference implementation: parity unpinned)."""
    refs, queries = _words(refs), _words(queries)
    assert refs.dtype == queries.dtype and refs.shape[1] == queries.shape[1]
    nq = queries.shape[0]
    kk = max(k, 1)
    s = np.full((nq, kk), 0xFFFFFFFF, dtype=np.uint32)
    x = np.full((nq, kk), -1, dtype=np.int64)
    c = np.zeros(max(nq, 1), dtype=np.int32)
    want = threshold is not None
    cap = capacity if want else 0
    hq = np.zeros(max(cap, 1), dtype=np.uint32)
    hr = np.zeros(max(cap, 1), dtype=np.int64)
    hs = np.zeros(max(cap, 1), dtype=np.uint32)
    n = lib().oracle_scan_op(_ptr(refs), refs.shape[0], _ptr(queries), nq, refs.shape[1], refs.dtype.itemsize * 8,
                             k, max_score, int(want), int(threshold or 0), workers or os.cpu_count() or 1,
                             _ptr(s), _ptr(x), _ptr(c), cap, _ptr(hq), _ptr(hr), _ptr(hs), _SCAN_OPS[op])
    assert n >= 0, "oracle_scan failed"
    top = (s, x, c[:nq]) if k > 0 else None
    hits = None
    if want:
        m = min(n, cap)
        hits = (hq[:m].copy(), hr[:m].copy(), hs[:m].copy(), int(n))
    return top, hits


def score_word(r: int, q: int) -> int:
    return int(lib().oracle_score_word(r, q))


# ---------------------------------------------------------------------------
# numpy restatement (independent of the C code)
# ---------------------------------------------------------------------------

def np_scores(refs: np.ndarray, queries: np.ndarray) -> np.ndarray:
    """sum_k popcount(r_k AND NOT q_k) -- SPEC.md:131 form of Eq. 1."""
    r = refs[:, None, :]
    q = queries[None, :, :]
    return np.bitwise_count(r & ~q).sum(axis=2, dtype=np.uint32)


def np_scores_op(refs: np.ndarray, queries: np.ndarray, op: str = "andnot", block: int = 4096) -> np.ndarray:
    """sum_k popcount(op(r_k, q_k)) for op in {"andnot", "and", "xor"}.

    "andnot" is Eq. 1 (pinned by the golden fixtures through np_scores and
    the C oracle).  "and" and "xor" are operator extensions the reference
    does not implement -- their restatement is the definition itself
    (popcount of the word-wise AND / XOR), PARITY UNPINNED against the
    reference.  Blocked over known rows to bound the temporary."""
    fn = {"andnot": lambda r, q: r & ~q, "and": lambda r, q: r & q, "xor": lambda r, q: r ^ q}[op]
    out = np.empty((refs.shape[0], queries.shape[0]), dtype=np.uint32)
    q = queries[None, :, :]
    for r0 in range(0, refs.shape[0], block):
        r = refs[r0:r0 + block, None, :]
        out[r0:r0 + block] = np.bitwise_count(fn(r, q)).sum(axis=2, dtype=np.uint32)
    return out


def topk_from_matrix(scores: np.ndarray, k: int, max_score: int = 0xFFFFFFFF):
    """The same top-k derivation from a full (N_R, N_Q) matrix (numpy, stable)."""
    n_r, n_q = scores.shape
    s = np.full((n_q, k), 0xFFFFFFFF, dtype=np.uint32)
    x = np.full((n_q, k), -1, dtype=np.int64)
    c = np.zeros(n_q, dtype=np.int32)
    for j in range(n_q):
        col = scores[:, j]
        order = np.lexsort((np.arange(n_r), col))
        order = order[col[order] <= max_score][:k]
        c[j] = len(order)
        s[j, : len(order)] = col[order]
        x[j, : len(order)] = order
    return s, x, c


def threshold_from_matrix(scores: np.ndarray, t: int):
    j, i = np.nonzero(scores.T <= t)
    return j.astype(np.uint32), i.astype(np.int64), scores[i, j].astype(np.uint32)


# ---------------------------------------------------------------------------
# measurement conventions restated from the reference bench (bench.py:41-58)
# ---------------------------------------------------------------------------

def synth_words(n_rows: int, n_words: int, word_width: int = 64, seed: int = 0,
                stream: int = 0) -> np.ndarray:
    """Words of synth_panel(n_rows, n_words, word_width, seed, stream) (bench.py:41-54)."""
    rng = np.random.default_rng([seed, stream, n_rows, n_words, word_width])
    dtype = np.uint32 if word_width == 32 else np.uint64
    return rng.integers(0, 2**word_width, size=(n_rows, n_words), dtype=dtype)


def score_checksum(scores: np.ndarray) -> str:
    """sha256[:16] of the little-endian u32 matrix (bench.py:57-58)."""
    return hashlib.sha256(np.ascontiguousarray(scores, dtype="<u4").tobytes()).hexdigest()[:16]


def mask_padding(words: np.ndarray, bit_length: int) -> np.ndarray:
    """Zero the bits past bit_length in the last word (tests/conftest.py:77-86 rule)."""
    width = words.dtype.itemsize * 8
    tail = bit_length % width
    if tail and words.shape[1]:
        words = words.copy()
        keep = ((1 << width) - 1) ^ ((1 << (width - tail)) - 1)
        words[:, -1] &= words.dtype.type(keep)
    return words


def merge_lists(scores: np.ndarray, index: np.ndarray, k: int):
    """Merge [lists, N_Q, k_in] candidate lists into the first k per query by (score, index)."""
    n_lists, n_q, k_in = scores.shape
    s_out = np.full((n_q, k), 0xFFFFFFFF, dtype=np.uint32)
    x_out = np.full((n_q, k), -1, dtype=np.int64)
    for j in range(n_q):
        s = scores[:, j, :].reshape(-1)
        x = index[:, j, :].reshape(-1)
        keep = x >= 0
        s, x = s[keep], x[keep]
        order = np.lexsort((x, s))[:k]
        s_out[j, : len(order)] = s[order]
        x_out[j, : len(order)] = x[order]
    return s_out, x_out
