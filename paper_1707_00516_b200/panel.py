"""Host-side panel types with the reference's names and validation rules.

These mirror ``Panel`` / ``QueryLayout`` / ``ScoreMatrix`` / ``TileConfig``
of the reference (pkg/src/fastid/kernel.py:62-207) so that parity tests and
callers read the same.  The comparison entry points in ``compare.py`` accept
either these classes or the reference's own objects (duck-typed on
``words`` / ``bit_length`` / ``ids``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import CodecError, CorruptProfileError

WORD_WIDTHS = (32, 64)
TILE_SIZES = (16, 32, 64)          # the paper's §IV-B block sizes (kernel.py:28)
DEFAULT_TILE_SIZE = 64
DEFAULT_CELLS_PER_TASK = 16        # "16 output elements per thread" (kernel.py:30)


def words_per_profile(bit_length: int, word_width: int) -> int:
    """ceil(L / B) (codec.py:40-42)."""
    return -(-bit_length // word_width)


def word_dtype(word_width: int) -> np.dtype:
    """uint32 / uint64 for B = 32 / 64 (codec.py:32-37)."""
    if word_width not in WORD_WIDTHS:
        raise CodecError(f"unsupported word width {word_width}, expected one of {WORD_WIDTHS}")
    return np.dtype(np.uint32 if word_width == 32 else np.uint64)


def padding_mask(bit_length: int, word_width: int) -> int:
    """Bits of the last word that lie past bit_length (must be zero)."""
    tail = bit_length % word_width
    return (1 << (word_width - tail)) - 1 if tail else 0


def _frozen_words(words) -> np.ndarray:
    arr = np.ascontiguousarray(words)
    if arr is words and arr.flags.writeable:
        arr = arr.copy()
    arr.setflags(write=False)
    return arr


@dataclass(frozen=True)
class Panel:
    """Row-major (N, ceil(L/B)) u32/u64 profile words, zero padded past L, read-only."""

    ids: tuple
    words: np.ndarray
    bit_length: int

    def __post_init__(self):
        w = np.ascontiguousarray(self.words)
        if w.ndim != 2:
            raise ValueError("panel words must be a 2-D array (rows x words)")
        if w.dtype not in (np.dtype(np.uint32), np.dtype(np.uint64)):
            raise ValueError(f"panel dtype must be uint32 or uint64, got {w.dtype}")
        ids = tuple(self.ids)
        if len(ids) != w.shape[0]:
            raise ValueError(f"{len(ids)} ids for {w.shape[0]} profile rows")
        if self.bit_length <= 0:
            raise ValueError("panel bit length must be positive")
        width = w.dtype.itemsize * 8
        need = words_per_profile(self.bit_length, width)
        if w.shape[1] != need:
            raise ValueError(f"expected {need} words for {self.bit_length} bits at width {width}, "
                             f"got {w.shape[1]}")
        mask = padding_mask(self.bit_length, width)
        if mask and w.size and np.any(w[:, -1] & w.dtype.type(mask)):
            raise CorruptProfileError(f"nonzero padding past bit {self.bit_length}")
        object.__setattr__(self, "words", _frozen_words(w))
        object.__setattr__(self, "ids", ids)

    @property
    def n_profiles(self) -> int:
        return self.words.shape[0]

    @property
    def n_words(self) -> int:
        return self.words.shape[1]

    @property
    def word_width(self) -> int:
        return self.words.dtype.itemsize * 8


@dataclass(frozen=True)
class QueryLayout:
    """The query panel stored word-major (N_W, N_Q) -- the paper's transposed B (§IV-B)."""

    ids: tuple
    words: np.ndarray
    bit_length: int

    def __post_init__(self):
        w = np.ascontiguousarray(self.words)
        if w.ndim != 2:
            raise ValueError("query layout words must be 2-D (words x queries)")
        object.__setattr__(self, "words", _frozen_words(w))
        object.__setattr__(self, "ids", tuple(self.ids))

    @property
    def n_queries(self) -> int:
        return self.words.shape[1]

    @property
    def n_words(self) -> int:
        return self.words.shape[0]

    @property
    def word_width(self) -> int:
        return self.words.dtype.itemsize * 8


def relayout_queries(queries) -> QueryLayout:
    """Column-major copy of a query panel (kernel.py:161-163)."""
    return QueryLayout(queries.ids, np.ascontiguousarray(np.asarray(queries.words).T), queries.bit_length)


def restore_queries(layout) -> Panel:
    """Inverse of relayout_queries (kernel.py:166-168)."""
    return Panel(layout.ids, np.ascontiguousarray(np.asarray(layout.words).T), layout.bit_length)


@dataclass(frozen=True)
class ScoreMatrix:
    """N_R x N_Q u32 scores with row (known) and column (unknown) ids, read-only."""

    ref_ids: tuple
    query_ids: tuple
    scores: np.ndarray

    def __post_init__(self):
        s = np.ascontiguousarray(self.scores, dtype=np.uint32)
        rid, qid = tuple(self.ref_ids), tuple(self.query_ids)
        if s.shape != (len(rid), len(qid)):
            raise ValueError(f"score shape {s.shape} does not match {len(rid)} refs x {len(qid)} queries")
        s.setflags(write=False)
        object.__setattr__(self, "scores", s)
        object.__setattr__(self, "ref_ids", rid)
        object.__setattr__(self, "query_ids", qid)

    @property
    def shape(self) -> tuple:
        return self.scores.shape


@dataclass(frozen=True)
class TileConfig:
    """Accepted for API compatibility (kernel.py:196-207); the device tiling is fixed
    by the CTA / TMEM shapes, so these values only go through validation."""

    block_size: int = DEFAULT_TILE_SIZE
    cells_per_task: int = DEFAULT_CELLS_PER_TASK

    def __post_init__(self):
        if self.block_size not in TILE_SIZES:
            raise ValueError(f"tile size must be one of {TILE_SIZES}, got {self.block_size}")
        if self.cells_per_task < 1:
            raise ValueError("cells_per_task must be at least 1")


@dataclass(frozen=True)
class TopKResult:
    """Per unknown: the k best (score, known index) pairs, score asc then index asc.

    ``scores`` u32 [N_Q, k] (0xFFFFFFFF = empty slot), ``index`` i64 [N_Q, k]
    (-1 = empty), ``ref_ids`` resolves indices when the known panel had ids.
    """

    query_ids: tuple
    scores: np.ndarray
    index: np.ndarray
    ref_ids: tuple | None = None

    @property
    def counts(self) -> np.ndarray:
        return (self.index >= 0).sum(axis=1).astype(np.int32)


@dataclass(frozen=True)
class ThresholdHits:
    """All (unknown j, known i, score) with score <= threshold, ordered by (j, i)."""

    query: np.ndarray
    ref: np.ndarray
    score: np.ndarray
    threshold: int

    def __len__(self) -> int:
        return int(self.query.shape[0])
