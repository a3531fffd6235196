"""Database-scale search: a known panel resident in HBM, queried in batches.

This is the shape of the paper's headline job (2048 unknowns x 20M knowns,
PAPER.md:13): the known database is uploaded once (PAPER.md:151-153 batch
the knowns because a K80 could not hold them; a B200's 180 GB holds 20M x
1,024 loci = 2.56 GB seventy times over), and each batch of unknowns is
scored against all of it with a fused top-k or threshold epilogue, so the
N_R x N_Q count matrix is never materialised.

``KnownDatabase.search`` is the host-buffer public call: unknowns from host
memory (pinned staging) -> device, compare + epilogue on the device, results
back to host.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from .compare import (DevicePanel, _check_panels, _require_cuda, compare_device, threshold_hits, topk_device,
                      topk_workspace_bytes)
from .panel import ThresholdHits, TopKResult

__all__ = ["KnownDatabase", "PreparedImage", "ChunkedImage", "QueryStager", "GraphedSearch", "DB_OPTIONS"]

# Execution variants of a prepared database (fastid_db_option, include/fastid_b200.h).
# Each computes the same result; they select among kernel paths.
DB_OPTIONS = {
    "no_cta_pairs": 1,       # single-CTA split-B kernel instead of CTA pairs
    "no_tma_store": 2,       # full matrix by per-element stores
    "no_spare_pairs": 4,     # no spare-pair grid on the SMs the regular grid leaves free
    "narrow_tma_store": 8,   # per-warp (32-unknown) TMA-store blocks
}


class PreparedImage:
    """Owner of a C-ABI ``fastid_db`` handle: the known panel's tensor image.

    For the tcgen05 formulations the image holds every known tile already in
    the MMA operand layout (e2m1 nibbles / u8 bytes, ~4x / 8x the packed
    rows), so query batches stream it with bulk copies and no per-batch bit
    unpacking.  Built once per database (fastid_db_create).
    """

    def __init__(self, panel: DevicePanel, formulation: str | int, op: str = "andnot"):
        from . import _native

        self.panel = panel  # keeps the packed rows alive for the handle
        self.op = op
        self.handle = ctypes.c_void_p()
        L = _native.lib()
        with torch.cuda.device(panel.device):
            _native.check(L.fastid_db_create(panel.rows.data_ptr() if panel.n_profiles else 0, panel.n_profiles,
                                             panel.stride, panel.bit_length, _native.formulation_code(formulation, op),
                                             torch.cuda.current_stream(panel.device).cuda_stream,
                                             ctypes.byref(self.handle)), "fastid_db_create")
        self.formulation = L.fastid_db_formulation(self.handle)
        self.image_bytes = L.fastid_db_image_bytes(panel.n_profiles, panel.bit_length, self.formulation)

    def set_option(self, name: str, enabled: bool = True) -> None:
        """Switch one DB_OPTIONS execution variant on or off for later calls."""
        from . import _native

        if name not in DB_OPTIONS:
            raise ValueError(f"option must be one of {sorted(DB_OPTIONS)}, got {name!r}")
        _native.check(_native.lib().fastid_db_set_option(self.handle, DB_OPTIONS[name], int(bool(enabled))),
                      "fastid_db_set_option")

    def set_operator(self, op: str) -> None:
        """The operator of later calls (fastid_db_set_operator); the image is reused."""
        from . import _native

        _native.check(_native.lib().fastid_db_set_operator(self.handle, _native.operator_code(op)),
                      "fastid_db_set_operator")
        self.op = op

    @property
    def options(self) -> set:
        from . import _native

        bits = _native.lib().fastid_db_options(self.handle)
        return {n for n, b in DB_OPTIONS.items() if bits & b}

    def __del__(self):
        try:
            from . import _native

            if self.handle:
                _native.lib().fastid_db_destroy(self.handle)
                self.handle = ctypes.c_void_p()
        except Exception:
            pass


class QueryStager:
    """Pinned host staging + device buffers for repeated query batches of one shape."""

    def __init__(self, n_queries: int, n_words: int, word_width: int, bit_length: int, k: int, device):
        self.device = device
        self.word_width = word_width
        self.bit_length = bit_length
        nbytes = n_words * word_width // 8
        self.host_in = torch.empty((n_queries, nbytes), dtype=torch.uint8).pin_memory()
        self.dev_in = torch.empty((n_queries, nbytes), dtype=torch.uint8, device=device)
        self.panel = DevicePanel.empty(n_queries, bit_length, word_width, device)
        self.out_s = torch.empty((n_queries, k), dtype=torch.int32, device=device)
        self.out_x = torch.empty((n_queries, k), dtype=torch.int64, device=device)
        self.host_s = torch.empty((n_queries, k), dtype=torch.int32).pin_memory()
        self.host_x = torch.empty((n_queries, k), dtype=torch.int64).pin_memory()
        self.workspace = None
        self.done = torch.cuda.Event()  # recorded after this stager's D2H (pipelined searches)

    @property
    def h2d_bytes(self) -> int:
        return self.host_in.numel()

    @property
    def d2h_bytes(self) -> int:
        return self.host_s.numel() * 4 + self.host_x.numel() * 8


class ChunkedImage:
    """The tensor image of a known panel too large for one image in device memory.

    One reusable device buffer holds the image of ``chunk_rows`` rows (a
    multiple of the 192-row tile); each search builds the chunks' images into
    it in turn (fastid_db_create_in: an image-build kernel into the caller's
    buffer, stream-ordered after the previous chunk's comparison) and runs the
    image kernels per chunk with the chunk's row offset, so a panel whose
    packed rows fit but whose 4-bit image does not (e.g. 20M x 16384 loci:
    41 GB packed, 164 GB image) is still searched by the CTA-pair kernels; the
    chunks' results combine exactly (top-k lists merged with the (score,
    index) order, full-matrix rows and threshold hits by row range).
    """

    def __init__(self, panel: DevicePanel, formulation: str | int, chunk_rows: int | None = None,
                 op: str = "andnot"):
        from . import _native
        from .errors import DeviceError

        L = _native.lib()
        self.panel = panel
        self.op = op
        code = _native.formulation_code(formulation)
        if code == 0:  # auto: the tensor formulation that runs this length
            code = _native.FORMULATIONS["tensor_f4"] if _native.supports("tensor_f4", panel.bit_length) else 1
        self.code = code
        tile = 192
        per_tile = L.fastid_db_image_bytes(tile, panel.bit_length, code)
        if per_tile == 0:
            raise DeviceError("formulation has no tensor image")
        if chunk_rows is None:
            free = torch.cuda.mem_get_info(panel.device)[0]
            chunk_rows = int(free * 0.6) // per_tile * tile
        chunk_rows = min(int(chunk_rows) // tile * tile, -(-panel.n_profiles // tile) * tile)
        if chunk_rows < tile:
            raise DeviceError(f"cannot allocate even one {tile}-row chunk of the tensor image")
        self.chunk_rows = chunk_rows
        try:
            self.buf = torch.empty(L.fastid_db_image_bytes(chunk_rows, panel.bit_length, code), dtype=torch.uint8,
                                   device=panel.device)
        except torch.cuda.OutOfMemoryError as e:
            raise DeviceError(f"cannot allocate a {chunk_rows}-row image chunk: {e}") from None
        self._bits = 0

    def set_option(self, name: str, enabled: bool = True) -> None:
        """Switch one DB_OPTIONS execution variant for every chunk's handle."""
        if name not in DB_OPTIONS:
            raise ValueError(f"option must be one of {sorted(DB_OPTIONS)}, got {name!r}")
        self._bits = (self._bits | DB_OPTIONS[name]) if enabled else (self._bits & ~DB_OPTIONS[name])

    def set_operator(self, op: str) -> None:
        """The operator of the chunk handles built from now on."""
        from . import _native

        _native.operator_code(op)
        self.op = op

    @property
    def options(self) -> set:
        return {n for n, b in DB_OPTIONS.items() if self._bits & b}

    def chunks(self):
        """(first row, rows, the chunk's prepared image) per chunk, in row order; each
        image is built on the current stream into the shared buffer."""
        from . import _native

        L = _native.lib()
        n = self.panel.n_profiles
        for r0 in range(0, n, self.chunk_rows):
            nr = min(self.chunk_rows, n - r0)
            sub = self.panel.slice(r0, r0 + nr)
            h = ctypes.c_void_p()
            with torch.cuda.device(self.panel.device):
                _native.check(L.fastid_db_create_in(
                    sub.rows.data_ptr(), nr, sub.stride, sub.bit_length, self.code | _native.operator_code(self.op),
                    self.buf.data_ptr(),
                    self.buf.numel(), torch.cuda.current_stream(self.panel.device).cuda_stream, ctypes.byref(h)),
                    "fastid_db_create_in")
            for name, bit in DB_OPTIONS.items():
                if self._bits & bit:
                    _native.check(L.fastid_db_set_option(h, bit, 1), "fastid_db_set_option")
            view = _ChunkView(h, self.op)
            try:
                yield r0, nr, sub, view
            finally:
                L.fastid_db_destroy(h)  # the handle is host state only; kernels already enqueued


# Below this many unknowns a chunked image costs more to build per search than it
# saves: 20M x 16384 loci, top-16 (tools/chunked_vs_packed.py): 64 unknowns 72 ms
# chunked vs 20 ms packed, 512: 101 vs 75, 1024: 139 vs 152, 2048: 226 vs 306.
CHUNKED_IMAGE_MIN_QUERIES = 1024
# Up to this many unknowns an "auto" top-k runs the CUDA-core scan over the packed
# rows instead of the tensor image (tools/small_batch.py, 20M x 1024 loci, top-16:
# 1 unknown 0.49 vs 1.61 ms, 2: 0.64 vs 1.57, 4: 1.12 vs 1.57, 8: 2.01 vs 1.59).
SCAN_MAX_QUERIES = 4
# Up to this many unknowns (one 128-row group of the single-CTA tensor kernel) an
# "auto" top-k reads the packed rows, unpacked in shared memory, instead of the
# 4-bit image: 20M x 1024 loci 8-128 unknowns 1.23-1.35 vs 1.54-1.75 ms; 10M x
# 2048 loci 1.25-1.36 vs 1.51-1.67; 5M x 5000 1.63-1.79 vs 1.90-2.05; at 256
# unknowns the image wins (2.16 vs 2.33, 1.92 vs 2.40, 2.14 vs 3.39).
PACKED_MAX_QUERIES = 128


class _ChunkView:
    """A chunk's fastid_db handle, shaped like PreparedImage for the compare helpers."""

    def __init__(self, handle, op: str):
        self.handle = handle
        self.op = op


class GraphedSearch:
    """One host-buffer top-k search of a fixed shape captured as a CUDA graph.

    The graph holds the whole step -- pinned host -> device copy of the
    unknowns, their encode into the row layout, the fused compare + top-k
    launches (regular and spare CTA-pair grids, joined) and the merge, and the
    device -> pinned host copy of the lists -- so a repeated query of the same
    shape costs one graph launch instead of a dozen host-side enqueues (the
    graphs the task names in place of a tracing compiler).  ``run(words)``
    copies the words into the pinned input, replays, waits, and returns the
    lists; the result equals ``KnownDatabase.search_words`` of the same words.
    Built by ``KnownDatabase.graphed_search``.
    """

    def __init__(self, db: "KnownDatabase", n_queries: int, k: int, max_score: int | None = None):
        from . import _native

        self.db, self.n_queries, self.k = db, int(n_queries), int(k)
        p = db.panel
        dev = db.device
        self.stager = QueryStager(self.n_queries, p.n_words, p.word_width, p.bit_length, self.k, dev)
        st = self.stager
        with torch.cuda.device(dev):
            st.workspace = torch.empty(topk_workspace_bytes(p.n_profiles, self.n_queries, self.k, db.formulation),
                                       dtype=torch.uint8, device=dev)
            self.stream = torch.cuda.Stream(dev)
            self.stream.wait_stream(torch.cuda.current_stream(dev))
            lib = _native.lib()

            def step():
                cs = torch.cuda.current_stream(dev)
                st.dev_in.copy_(st.host_in, non_blocking=True)
                _native.check(lib.fastid_load_words(
                    st.dev_in.data_ptr(), self.n_queries, st.dev_in.shape[1], st.panel.rows.data_ptr(),
                    st.panel.stride, cs.cuda_stream), "fastid_load_words")
                s, x = db.topk_device(st.panel, self.k, max_score, st.workspace, (st.out_s, st.out_x))
                st.host_s.copy_(s, non_blocking=True)
                st.host_x.copy_(x, non_blocking=True)

            # warm up on the capture stream (the library keeps launch scratch per stream;
            # a first use inside the capture would have to allocate), then capture
            with torch.cuda.stream(self.stream):
                step()
            self.stream.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=self.stream):
                step()

    def run(self, query_words: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """Top-k of a (n_queries, N_W) host word array through the captured graph."""
        from .errors import CorruptProfileError, PanelMismatchError
        from .panel import padding_mask

        p = self.db.panel
        qw = np.ascontiguousarray(query_words)
        if qw.dtype.itemsize * 8 != p.word_width or qw.shape != (self.n_queries, p.n_words):
            raise PanelMismatchError(f"query words {qw.shape}/{qw.dtype} do not match the captured search "
                                     f"({self.n_queries} x {p.n_words} {p.word_width}-bit words)")
        mask = padding_mask(p.bit_length, p.word_width)
        if mask and qw.size and np.any(qw[:, -1] & qw.dtype.type(mask)):
            raise CorruptProfileError(f"nonzero padding past bit {p.bit_length}")
        st = self.stager
        st.host_in.numpy()[:] = qw.view(np.uint8).reshape(self.n_queries, -1)
        with torch.cuda.stream(self.stream):  # replay() launches on the current stream
            self.graph.replay()
        self.stream.synchronize()
        return st.host_s.numpy().view(np.uint32).copy(), st.host_x.numpy().copy()


class KnownDatabase:
    """A known panel resident on one device (or one shard of it, ``ref_base`` = global offset)."""

    def __init__(self, refs, bit_length: int | None = None, device=None, ref_base: int = 0,
                 formulation: str | int = "auto", prepare: bool = True, image_chunk_rows: int | None = None,
                 op: str = "andnot"):
        self.device = _require_cuda(device)
        if isinstance(refs, DevicePanel):
            self.panel = refs
        elif hasattr(refs, "words"):
            self.panel = DevicePanel.from_panel(refs, self.device)
        else:
            if bit_length is None:
                raise ValueError("bit_length is required for raw word arrays")
            self.panel = DevicePanel.from_words(refs, bit_length, device=self.device)
        self.ref_base = int(ref_base)
        self.formulation = formulation
        from . import _native

        _native.operator_code(op)
        self.op = op  # the bitwise operator of every search (compare_device's op)
        self._stagers: dict = {}
        # the tensor image (built once) lets every query batch skip bit unpacking; a
        # database whose image does not fit in device memory (4 bits per locus for
        # mxf4) keeps only its packed rows and runs the unpacking kernels instead
        self.image = None
        self.chunked_min_queries = CHUNKED_IMAGE_MIN_QUERIES
        self.scan_max_queries = SCAN_MAX_QUERIES
        self.packed_max_queries = PACKED_MAX_QUERIES
        if prepare and self.panel.n_profiles:
            # image_chunk_rows: build the image chunk by chunk into one buffer of that
            # many rows (what a panel whose whole image does not fit falls back to)
            self.image = (ChunkedImage(self.panel, formulation, image_chunk_rows, op) if image_chunk_rows
                          else self._prepare(formulation))

    def _prepare(self, formulation):
        from .errors import DeviceError

        for attempt in range(2):
            try:
                return PreparedImage(self.panel, formulation, self.op)
            except DeviceError as e:
                if "allocate" not in str(e):
                    raise
                if attempt == 0:
                    torch.cuda.empty_cache()  # cached torch blocks may be what is missing
                    continue
                try:
                    return ChunkedImage(self.panel, formulation, op=self.op)
                except DeviceError as e2:
                    import warnings

                    warnings.warn(f"tensor image does not fit on {self.device} ({e}; {e2}); using packed operands",
                                  RuntimeWarning, stacklevel=3)
        return None

    def set_option(self, name: str, enabled: bool = True) -> None:
        """Select an execution variant of the prepared image (DB_OPTIONS); every
        variant returns the same result.  No effect without a tensor image."""
        if self.image is not None:
            self.image.set_option(name, enabled)

    def set_operator(self, op: str) -> None:
        """Switch the bitwise operator ("andnot", "and", "xor") of later searches;
        the prepared image serves every operator and is not rebuilt."""
        from . import _native

        _native.operator_code(op)
        if self.image is not None:
            self.image.set_operator(op)
        self.op = op

    @property
    def n_profiles(self) -> int:
        return self.panel.n_profiles

    @property
    def bit_length(self) -> int:
        return self.panel.bit_length

    def _queries_device(self, queries) -> DevicePanel:
        if isinstance(queries, DevicePanel):
            return queries
        return DevicePanel.from_panel(queries, self.device)

    # -- device-resident calls (inputs already in HBM) -------------------------
    def _chunked_for(self, n_queries: int) -> bool:
        """Whether a batch this size goes through the chunked image (large batches) or
        the packed-operand kernels (small ones), when the whole image did not fit."""
        return isinstance(self.image, ChunkedImage) and n_queries >= self.chunked_min_queries

    def _plain_image(self):
        return None if isinstance(self.image, ChunkedImage) else self.image

    def topk_device(self, queries: DevicePanel, k: int, max_score: int | None = None, workspace=None, out=None,
                    events=None):
        if self.formulation == "auto" and self.panel.n_profiles and events is None:
            n_q = queries.n_profiles
            if n_q <= self.scan_max_queries:
                # a handful of unknowns: the CUDA-core scan over the packed rows (HBM-bound)
                # beats streaming the 4-bit image (one unknown, 20M x 1024 loci: 0.70 vs 1.52 ms)
                return topk_device(self.panel, queries, k, max_score, self.ref_base, "popc", workspace, out,
                                   op=self.op)
            if n_q <= self.packed_max_queries:
                # one group of unknowns: the tensor kernel unpacking packed rows in shared
                # memory reads 4x fewer bytes than the image and is faster
                return topk_device(self.panel, queries, k, max_score, self.ref_base, "tensor_f4", workspace, out,
                                   op=self.op)
        if self._chunked_for(queries.n_profiles):
            return self._topk_chunked(queries, k, max_score, workspace, out)
        return topk_device(self.panel, queries, k, max_score, self.ref_base, self.formulation, workspace, out,
                           events=events, image=self._plain_image(), op=self.op)

    def _topk_chunked(self, queries: DevicePanel, k: int, max_score, workspace, out):
        """Per chunk: its image, the fused top-k with the chunk's row offset, and a merge
        of the chunk's lists into the running lists (two-list fastid_merge_topk)."""
        from . import _native

        n_q = queries.n_profiles
        dev = self.device
        if out is None:
            out = (torch.empty((n_q, k), dtype=torch.int32, device=dev),
                   torch.empty((n_q, k), dtype=torch.int64, device=dev))
        s, x = out
        if n_q == 0:
            return s, x
        cand_s = torch.empty((2, n_q, k), dtype=torch.int32, device=dev)
        cand_x = torch.empty((2, n_q, k), dtype=torch.int64, device=dev)
        L = _native.lib()
        first = True
        for r0, nr, sub, view in self.image.chunks():
            dst = (cand_s[0], cand_x[0]) if first else (cand_s[1], cand_x[1])
            topk_device(sub, queries, k, max_score, self.ref_base + r0, self.formulation, workspace, dst, image=view,
                        op=self.op)
            if not first:
                with torch.cuda.device(dev):
                    _native.check(L.fastid_merge_topk(cand_s.data_ptr(), cand_x.data_ptr(), 2, n_q, k, k,
                                                      s.data_ptr(), x.data_ptr(),
                                                      torch.cuda.current_stream(dev).cuda_stream),
                                  "fastid_merge_topk")
                cand_s[0].copy_(s)
                cand_x[0].copy_(x)
            first = False
        s.copy_(cand_s[0])
        x.copy_(cand_x[0])
        return s, x

    def full_device(self, queries: DevicePanel, out=None) -> torch.Tensor:
        if self._chunked_for(queries.n_profiles):
            if out is None:
                out = torch.empty((self.panel.n_profiles, queries.n_profiles), dtype=torch.int32, device=self.device)
            for r0, nr, sub, view in self.image.chunks():
                compare_device(sub, queries, out[r0:r0 + nr], self.formulation, image=view, op=self.op)
            return out
        return compare_device(self.panel, queries, out, self.formulation, image=self._plain_image(), op=self.op)

    # -- host-buffer public calls ------------------------------------------------
    def stager(self, n_queries: int, k: int, slot: int = 0) -> QueryStager:
        key = (n_queries, k, slot)
        st = self._stagers.get(key)
        if st is None:
            p = self.panel
            st = QueryStager(n_queries, p.n_words, p.word_width, p.bit_length, k, self.device)
            self._stagers[key] = st
        return st

    def stage_queries(self, query_words: np.ndarray, k: int, stager: QueryStager | None = None) -> QueryStager:
        """Host (N_Q, N_W) words -> the stager's device panel, enqueued on the current
        stream: copy into pinned staging, H2D, encode into the aligned row layout.
        Validates the words as the reference Panel does (width, word count,
        zero padding past L)."""
        from . import _native
        from .errors import CorruptProfileError, PanelMismatchError
        from .panel import padding_mask

        p = self.panel
        qw = np.ascontiguousarray(query_words)
        if qw.dtype.itemsize * 8 != p.word_width or qw.ndim != 2 or qw.shape[1] != p.n_words:
            raise PanelMismatchError(f"query words {qw.shape}/{qw.dtype} do not match the database "
                                     f"({p.n_words} x {p.word_width}-bit words)")
        mask = padding_mask(p.bit_length, p.word_width)
        if mask and qw.size and np.any(qw[:, -1] & qw.dtype.type(mask)):
            raise CorruptProfileError(f"nonzero padding past bit {p.bit_length}")
        n_q = qw.shape[0]
        st = stager or self.stager(n_q, k)
        st.host_in.numpy()[:] = qw.view(np.uint8).reshape(n_q, -1)
        stream = torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            st.dev_in.copy_(st.host_in, non_blocking=True)
            _native.check(_native.lib().fastid_load_words(
                st.dev_in.data_ptr(), n_q, st.dev_in.shape[1], st.panel.rows.data_ptr(), st.panel.stride,
                stream.cuda_stream), "fastid_load_words")
        return st

    def fetch_lists(self, st: QueryStager, s: torch.Tensor, x: torch.Tensor) -> tuple[np.ndarray, np.ndarray]:
        """D2H of a (scores, index) result through the stager's pinned buffers."""
        stream = torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            st.host_s.copy_(s, non_blocking=True)
            st.host_x.copy_(x, non_blocking=True)
            stream.synchronize()
        return st.host_s.numpy().view(np.uint32).copy(), st.host_x.numpy().copy()

    def search_words(self, query_words: np.ndarray, k: int = 16, max_score: int | None = None,
                     stager: QueryStager | None = None) -> tuple[np.ndarray, np.ndarray]:
        """Top-k of a (N_Q, N_W) host word array -> host (scores u32 [N_Q,k], index i64 [N_Q,k]).

        Per call: pinned H2D of the unknowns, on-device encode into the row
        layout, fused compare + top-k, D2H of the (score, index) lists.
        """
        st = self.stage_queries(query_words, k, stager)
        with torch.cuda.device(self.device):
            s, x = self.topk_device(st.panel, k, max_score, st.workspace, (st.out_s, st.out_x))
        return self.fetch_lists(st, s, x)

    def search_many(self, batches, k: int = 16, max_score: int | None = None, combine=None):
        """Pipelined top-k over a sequence of host query batches (a serving loop):
        batch i+1 is staged (pinned copy, H2D, encode) and its kernels enqueued
        before batch i's lists are read back, so the host work and the D2H of one
        batch overlap the device work of the next.  Yields host (scores, index)
        per batch, in order; each equals ``search_words`` of that batch.
        ``combine(s, x, k)`` is applied on the device before the read-back (the
        sharded driver's cross-rank gather + merge)."""
        stream = torch.cuda.current_stream(self.device)
        pending = None
        slot = 0
        for qw in batches:
            qw = np.ascontiguousarray(qw)
            st = self.stager(qw.shape[0], k, slot)
            st.done.synchronize()  # the slot's previous batch has been read back
            self.stage_queries(qw, k, st)
            with torch.cuda.device(self.device):
                s, x = self.topk_device(st.panel, k, max_score, st.workspace, (st.out_s, st.out_x))
                if combine is not None:
                    s, x = combine(s, x, k)
                st.host_s.copy_(s, non_blocking=True)
                st.host_x.copy_(x, non_blocking=True)
                st.done.record(stream)
            if pending is not None:
                yield self._read_back(pending)
            pending = st
            slot ^= 1
        if pending is not None:
            yield self._read_back(pending)

    @staticmethod
    def _read_back(st: QueryStager) -> tuple[np.ndarray, np.ndarray]:
        st.done.synchronize()
        return st.host_s.numpy().view(np.uint32).copy(), st.host_x.numpy().copy()

    def graphed_search(self, n_queries: int, k: int = 16, max_score: int | None = None) -> GraphedSearch:
        """Capture the host-buffer top-k of ``n_queries`` unknowns as a CUDA graph
        (GraphedSearch): for repeated queries of one shape, one graph launch per
        search."""
        return GraphedSearch(self, n_queries, k, max_score)

    def search(self, queries, k: int = 16, max_score: int | None = None) -> TopKResult:
        """Per unknown, the k closest knowns by (score asc, global index asc)."""
        _check_panels(self.bit_length, self.panel.word_width, queries.bit_length, queries.word_width)
        s, x = self.search_words(np.asarray(queries.words), k, max_score)
        return TopKResult(tuple(queries.ids), s, x, self.panel.ids)

    def threshold(self, queries, threshold: int, capacity: int | None = None) -> ThresholdHits:
        n_q = queries.n_profiles if isinstance(queries, DevicePanel) else len(queries.words)
        if self.formulation == "auto" and self.panel.n_profiles:
            if n_q <= self.scan_max_queries:
                # a handful of unknowns: the CUDA-core scan over the packed rows
                return threshold_hits(self.panel, queries, threshold, capacity, "popc", self.device,
                                      ref_base=self.ref_base, op=self.op)
            if n_q <= self.packed_max_queries:
                # one group of unknowns: packed rows unpacked in shared memory beat the image
                # (20M x 1024 loci, 32-128 unknowns: 1.26 vs 1.61 ms; 5M x 5000: 1.71-1.73 vs 2.01-2.04)
                return threshold_hits(self.panel, queries, threshold, capacity, "tensor_f4", self.device,
                                      ref_base=self.ref_base, op=self.op)
        if self._chunked_for(n_q):
            parts = [threshold_hits(sub, queries, threshold, capacity, self.formulation, self.device,
                                    ref_base=self.ref_base + r0, image=view, op=self.op)
                     for r0, nr, sub, view in self.image.chunks()]
            q = np.concatenate([h.query for h in parts])
            r = np.concatenate([h.ref for h in parts])
            sc = np.concatenate([h.score for h in parts])
            order = np.lexsort((r, q))
            return ThresholdHits(q[order], r[order], sc[order], int(threshold))
        return threshold_hits(self.panel, queries, threshold, capacity, self.formulation, self.device,
                              ref_base=self.ref_base, image=self._plain_image(), op=self.op)
