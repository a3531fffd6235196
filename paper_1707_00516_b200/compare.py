"""Drop-in comparison entry points over the sm_100a library.

Reference surface mirrored here (pkg/src/fastid/ in the reference):

=============================  ==============================================
reference                      this package
=============================  ==============================================
compare_naive(refs, queries)   compare_b200(refs, queries)     kernel.py:283
compare_blocked(refs, layout,  compare_blocked_b200(...)       kernel.py:295
  tile, parallelism)
run_naive_kernel(r, q, out)    run_b200_kernel(r, q, out)      kernel.py:350
run_blocked_kernel(r, qT, ..)  run_b200_kernel(r, qT, out,     kernel.py:317
                                 queries_transposed=True)
NaiveExecutor / Blocked...     B200Executor (run_pipeline seam) scheduler.py:221
(none)            topk / threshold_hits (fused epilogues)
=============================  ==============================================

Validation happens here, before any native call, and raises the reference's
exception types (``PanelMismatchError`` for bit-length/width mismatch,
kernel.py:272-280; ``ValueError`` for parallelism < 1, kernel.py:308-309).
Empty panels return empty results (kernel.py:289-291).

PyTorch is used only for device memory and the current stream; every score
is computed by the CUDA kernels in ``csrc/``.  There is no CPU fallback: if
the library is missing or no GPU is present the call raises.
"""

from __future__ import annotations

import ctypes
import os
import struct
import sys

import numpy as np
import torch

from . import _native
from .errors import CodecError, CorruptProfileError, PanelMismatchError
from .panel import (Panel, QueryLayout, ScoreMatrix, ThresholdHits, TileConfig, TopKResult, padding_mask, word_dtype,
                    words_per_profile)

__all__ = [
    "DevicePanel",
    "B200Executor",
    "compare_b200",
    "compare_blocked_b200",
    "compare_device",
    "run_b200_kernel",
    "topk",
    "topk_device",
    "threshold_hits",
    "row_stride",
]

EMPTY_SCORE = 0xFFFFFFFF


def row_stride(bit_length: int) -> int:
    """Bytes per device row: ceil(L / 128) * 16 (16-B aligned rows)."""
    return -(-bit_length // 128) * 16


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        from .errors import DeviceError

        raise DeviceError("no CUDA device is visible; the B200 path has no CPU fallback")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def _check_panels(ref_bits: int, ref_width: int, query_bits: int, query_width: int) -> None:
    """Same conditions and messages as the reference's _check_panels (kernel.py:272-280)."""
    if ref_bits != query_bits:
        raise PanelMismatchError(f"panel bit lengths differ: refs {ref_bits}, queries {query_bits}")
    if ref_width != query_width:
        raise PanelMismatchError(f"panel word widths differ: refs {ref_width}, queries {query_width}")


class DevicePanel:
    """A panel resident in HBM in the aligned row layout.

    ``rows`` is a uint8 tensor of shape (n_profiles, stride); row i holds the
    profile's words in native little-endian order, zero filled to ``stride``.
    This is how the known database stays resident between query batches.
    """

    def __init__(self, rows: torch.Tensor, bit_length: int, word_width: int, ids=None):
        if rows.dtype != torch.uint8 or rows.dim() != 2 or not rows.is_cuda:
            raise ValueError("rows must be a 2-D uint8 CUDA tensor")
        if rows.shape[1] != row_stride(bit_length):
            raise ValueError(f"row stride {rows.shape[1]} does not match {row_stride(bit_length)}")
        if rows.data_ptr() % 16:
            raise ValueError("rows must be 16-byte aligned")
        self.rows = rows
        self.bit_length = int(bit_length)
        self.word_width = int(word_width)
        self.ids = tuple(ids) if ids is not None else None

    # -- construction (the profile encoder) --------------------------------
    @classmethod
    def empty(cls, n: int, bit_length: int, word_width: int = 64, device=None) -> "DevicePanel":
        dev = _require_cuda(device)
        return cls(torch.zeros((n, row_stride(bit_length)), dtype=torch.uint8, device=dev),
                   bit_length, word_width)

    @classmethod
    def from_words(cls, words, bit_length: int, ids=None, device=None) -> "DevicePanel":
        """Upload a (N, N_W) u32/u64 word array (host numpy or CUDA tensor).

        The words are validated as the reference Panel validates them
        (kernel.py:60-63, 85-90): exactly ceil(L/B) words per row (ValueError)
        and zero padding past bit L (CorruptProfileError) -- before any device work.
        """
        if bit_length <= 0:
            raise ValueError("panel bit length must be positive")
        is_tensor = isinstance(words, torch.Tensor)
        if is_tensor:
            if words.dtype not in (torch.int32, torch.int64, torch.uint32, torch.uint64) or words.dim() != 2:
                raise ValueError("word tensors must be 2-D 32- or 64-bit integers")
            width = words.element_size() * 8
            n, n_words = words.shape
        else:
            arr = np.ascontiguousarray(words)
            if arr.dtype not in (np.uint32, np.uint64) or arr.ndim != 2:
                raise ValueError("word arrays must be 2-D uint32/uint64")
            width = arr.dtype.itemsize * 8
            n, n_words = arr.shape
        need = words_per_profile(bit_length, width)
        if n_words != need:
            raise ValueError(f"expected {need} words for {bit_length} bits at width {width}, got {n_words}")
        mask = padding_mask(bit_length, width)
        if mask and n and not is_tensor and np.any(arr[:, -1] & arr.dtype.type(mask)):
            raise CorruptProfileError(f"nonzero padding past bit {bit_length}")
        dev = _require_cuda(device)
        if is_tensor:
            src = words.to(dev).contiguous()
            # the tensor holds the words' bits as (possibly signed) integers: mask in that type
            m = mask - (1 << width) if mask >= 1 << (width - 1) else mask
            signed = src.view(torch.int64 if width == 64 else torch.int32)
            if mask and n and bool((signed[:, -1] & m).any()):
                raise CorruptProfileError(f"nonzero padding past bit {bit_length}")
        else:
            raw = arr.view(np.uint8).reshape(n, -1) if n else np.zeros((0, n_words * width // 8), np.uint8)
            if not raw.flags.writeable:
                raw = raw.copy()
            src = torch.from_numpy(raw).to(dev)
        out = cls.empty(n, bit_length, width, dev)
        out.ids = tuple(ids) if ids is not None else None
        if n:
            with torch.cuda.device(dev):
                _native.check(_native.lib().fastid_load_words(
                    src.data_ptr(), n, n_words * width // 8, out.rows.data_ptr(), out.stride,
                    _stream(dev)), "fastid_load_words")
                torch.cuda.current_stream(dev).synchronize()  # src must outlive the copy
        return out

    @classmethod
    def from_panel(cls, panel, device=None) -> "DevicePanel":
        return cls.from_words(np.asarray(panel.words), panel.bit_length, getattr(panel, "ids", None), device)

    @classmethod
    def from_bits(cls, bits, word_width: int = 64, ids=None, device=None) -> "DevicePanel":
        """Pack a (N, L) 0/1 byte matrix on the GPU exactly as codec.pack (codec.py:118-127)."""
        word_dtype(word_width)
        dev = _require_cuda(device)
        t = bits if isinstance(bits, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(bits, np.uint8))
        if t.dim() != 2 or t.dtype != torch.uint8:
            raise CodecError("profile bits must be a 2-D uint8 matrix")
        t = t.to(dev).contiguous()
        n, length = t.shape
        if length == 0:
            raise CodecError("profile bits must be non-empty")
        if n and int(t.max()) > 1:
            raise CodecError("profile bits must contain only 0 and 1")
        out = cls.empty(n, length, word_width, dev)
        out.ids = tuple(ids) if ids is not None else None
        if n:
            with torch.cuda.device(dev):
                _native.check(_native.lib().fastid_pack_bits(
                    t.data_ptr(), n, length, word_width, out.rows.data_ptr(), out.stride, _stream(dev)),
                    "fastid_pack_bits")
        return out

    @classmethod
    def from_genotypes(cls, codes, word_width: int = 64, ids=None, device=None) -> "DevicePanel":
        """Encode (N, loci) genotype codes 0=MM 1=Mm 2=mM 3=mm to 2 bits/locus (codec.py:99-115)."""
        word_dtype(word_width)
        dev = _require_cuda(device)
        t = codes if isinstance(codes, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(codes, np.uint8))
        if t.dim() != 2 or t.dtype != torch.uint8 or t.shape[1] == 0:
            raise CodecError("genotype codes must be a non-empty 2-D uint8 matrix")
        t = t.to(dev).contiguous()
        n, loci = t.shape
        if n and int(t.max()) > 3:
            bad = int(torch.nonzero(t.reshape(-1) > 3)[0])
            raise CodecError(f"unknown genotype code at position {bad % loci} of profile {bad // loci}")
        out = cls.empty(n, 2 * loci, word_width, dev)
        out.ids = tuple(ids) if ids is not None else None
        if n:
            with torch.cuda.device(dev):
                _native.check(_native.lib().fastid_pack_genotypes(
                    t.data_ptr(), n, loci, word_width, out.rows.data_ptr(), out.stride, _stream(dev)),
                    "fastid_pack_genotypes")
        return out

    # -- views ---------------------------------------------------------------
    @property
    def n_profiles(self) -> int:
        return int(self.rows.shape[0])

    @property
    def stride(self) -> int:
        return int(self.rows.shape[1])

    @property
    def device(self) -> torch.device:
        return self.rows.device

    @property
    def n_words(self) -> int:
        return -(-self.bit_length // self.word_width)

    def slice(self, start: int, stop: int) -> "DevicePanel":
        ids = self.ids[start:stop] if self.ids is not None else None
        return DevicePanel(self.rows[start:stop], self.bit_length, self.word_width, ids)

    def to_words(self) -> np.ndarray:
        """Download as a (N, N_W) word array (inverse of from_words)."""
        nbytes = self.n_words * self.word_width // 8
        host = self.rows[:, :nbytes].contiguous().cpu().numpy()
        return host.view(word_dtype(self.word_width)).reshape(self.n_profiles, self.n_words)

    def to_panel(self) -> Panel:
        ids = self.ids if self.ids is not None else tuple(f"p{i}" for i in range(self.n_profiles))
        return Panel(ids, self.to_words(), self.bit_length)


def _as_device(p, device) -> DevicePanel:
    if isinstance(p, DevicePanel):
        return p
    return DevicePanel.from_panel(p, device)


def _ptr(p: DevicePanel) -> int:
    return p.rows.data_ptr() if p.n_profiles else 0


def _check_image_op(image, op: str) -> None:
    _native.operator_code(op)
    if image is not None and getattr(image, "op", "andnot") != op:
        raise ValueError(f"the prepared image was built for op={image.op!r}, not {op!r}")


def compare_device(refs: DevicePanel, queries: DevicePanel, out: torch.Tensor | None = None,
                   formulation: str | int = "auto", image=None, op: str = "andnot") -> torch.Tensor:
    """Full (N_R, N_Q) u32 score matrix on the device (int32 storage, reinterpret as u32).

    ``op`` is the bitwise operator before the popcount: "andnot" (FastID Eq. 1,
    popcount(r AND NOT q)), "and" (popcount(r AND q)) or "xor" (Hamming distance).
    """
    _check_panels(refs.bit_length, refs.word_width, queries.bit_length, queries.word_width)
    _check_image_op(image, op)
    dev = refs.device
    if out is None:
        out = torch.empty((refs.n_profiles, queries.n_profiles), dtype=torch.int32, device=dev)
    if out.shape[0] != refs.n_profiles or out.shape[1] < queries.n_profiles or out.dtype != torch.int32:
        raise ValueError("out must be an int32 tensor of shape (N_R, >= N_Q)")
    if out.numel() and out.stride(1) != 1:
        raise ValueError("out rows must be contiguous")
    if refs.n_profiles and queries.n_profiles:
        with torch.cuda.device(dev):
            if image is not None:
                _native.check(_native.lib().fastid_db_compare_full(
                    image.handle, _ptr(queries), queries.n_profiles, out.data_ptr(), out.stride(0), _stream(dev)),
                    "fastid_db_compare_full")
            else:
                _native.check(_native.lib().fastid_compare_full(
                    _ptr(refs), refs.n_profiles, _ptr(queries), queries.n_profiles, refs.stride,
                    refs.bit_length, out.data_ptr(), out.stride(0), _native.formulation_code(formulation, op),
                    _stream(dev)), "fastid_compare_full")
    return out


def _score_matrix_type(panel):
    """The ScoreMatrix class that goes with the caller's panel type: the reference's
    own (fastid.kernel.ScoreMatrix) for reference panels, so isinstance checks and
    downstream writers (write_scores) behave as with compare_naive; else this
    package's mirror (panel.ScoreMatrix)."""
    mod = sys.modules.get(type(panel).__module__)
    cls = getattr(mod, "ScoreMatrix", None) if mod is not None else None
    return cls if isinstance(cls, type) else ScoreMatrix


def compare_b200(refs, queries, formulation: str | int = "auto", device=None, op: str = "andnot"):
    """``compare_naive`` on the B200 (kernel.py:283-292): same signature, errors,
    empties and result type (the reference's ScoreMatrix for reference panels).
    ``op`` as in compare_device (the reference computes "andnot" only)."""
    _native.operator_code(op)
    _check_panels(refs.bit_length, refs.word_width, queries.bit_length, queries.word_width)
    result = _score_matrix_type(refs)
    n_r, n_q = refs.words.shape[0], queries.words.shape[0]
    ref_ids = getattr(refs, "ids", tuple(f"r{i}" for i in range(n_r)))
    q_ids = getattr(queries, "ids", tuple(f"q{j}" for j in range(n_q)))
    if n_r == 0 or n_q == 0:
        return result(ref_ids, q_ids, np.zeros((n_r, n_q), dtype=np.uint32))
    dev = _require_cuda(device)
    if n_r * n_q * 4 > _PIPELINE_MIN_BYTES and isinstance(refs.words, np.ndarray) \
            and isinstance(queries.words, np.ndarray):
        # large host results stream through the chunked pinned pipeline of the
        # host-buffer ABI instead of one device-sized matrix and a pageable copy
        scores = np.empty((n_r, n_q), np.uint32)
        with torch.cuda.device(dev):
            run_b200_kernel(refs.words, queries.words, scores, formulation=formulation, op=op)
        return result(ref_ids, q_ids, scores)
    d = compare_device(_as_device(refs, dev), _as_device(queries, dev), formulation=formulation, op=op)
    scores = d.cpu().numpy().view(np.uint32)
    return result(ref_ids, q_ids, scores)


_PIPELINE_MIN_BYTES = 64 << 20  # fastid_run_kernel streams outputs above this (csrc/api.cu)


def compare_blocked_b200(refs, queries: QueryLayout, tile: TileConfig | None = None, parallelism: int = 1,
                         formulation: str | int = "auto", device=None):
    """``compare_blocked`` on the B200 (kernel.py:295-314): the same checks in the
    same order (tile, parallelism >= 1, panel compatibility), empty results for
    empty panels, and the transposed query words scored as given -- like the
    reference, a QueryLayout is not re-validated (the device undoes the
    transpose, run_b200_kernel(queries_transposed=True)).  ``tile`` and
    ``parallelism`` are otherwise ignored: the device tiling is fixed."""
    tile = tile or TileConfig()
    if parallelism < 1:
        raise ValueError("parallelism must be at least 1")
    _check_panels(refs.bit_length, refs.word_width, queries.bit_length, queries.word_width)
    n_r, n_q = refs.words.shape[0], queries.words.shape[1]
    out = np.zeros((n_r, n_q), dtype=np.uint32)
    if out.size:
        if device is not None:
            with torch.cuda.device(_require_cuda(device)):
                run_b200_kernel(refs.words, queries.words, out, queries_transposed=True, formulation=formulation)
        else:
            run_b200_kernel(refs.words, queries.words, out, queries_transposed=True, formulation=formulation)
    return _score_matrix_type(refs)(refs.ids, queries.ids, out)


def run_b200_kernel(ref_words: np.ndarray, query_words: np.ndarray, out: np.ndarray,
                    queries_transposed: bool = False, formulation: str | int = "auto", op: str = "andnot") -> None:
    """Raw-array dispatch through the C ABI's host-buffer entry (fastid_run_kernel).

    Matches run_naive_kernel (kernel.py:350-353) -- and run_blocked_kernel
    (kernel.py:317-347) with ``queries_transposed=True`` -- writing every cell
    of the caller-owned ``out`` (N_R, N_Q) u32 array.
    """
    ref_words = np.ascontiguousarray(ref_words)
    query_words = np.ascontiguousarray(query_words)
    if ref_words.dtype != query_words.dtype or ref_words.dtype not in (np.uint32, np.uint64):
        raise PanelMismatchError(f"word dtypes differ or unsupported: {ref_words.dtype} vs {query_words.dtype}")
    n_refs, n_words = ref_words.shape
    n_q = query_words.shape[1] if queries_transposed else query_words.shape[0]
    qw = query_words.shape[0] if queries_transposed else query_words.shape[1]
    if qw != n_words:
        raise PanelMismatchError(f"word counts differ: refs {n_words}, queries {qw}")
    if out.shape != (n_refs, n_q) or out.dtype != np.uint32 or not out.flags.c_contiguous:
        raise ValueError(f"out must be a C-contiguous uint32 array of shape {(n_refs, n_q)}")
    if out.size == 0:
        return
    _require_cuda()
    _native.check(_native.lib().fastid_run_kernel(
        ref_words.ctypes.data, n_refs, query_words.ctypes.data, n_q, n_words, ref_words.dtype.itemsize * 8,
        int(bool(queries_transposed)), out.ctypes.data, _native.formulation_code(formulation, op)),
        "fastid_run_kernel")


FIDM_MAGIC = b"FIDM"
FIDM_VERSION = 1
_FIDM_HEADER = struct.Struct("<4sBQQ")  # io.py:29-31: magic, version, N_R, N_Q (little-endian)


def compare_to_fidm(refs, queries, path, formulation: str | int = "auto", device=None) -> tuple[int, int]:
    """Score ``refs`` x ``queries`` straight into a packed-binary score file.

    Byte-identical to the reference's ``write_scores(compare_naive(refs, queries),
    ScoreOutput(path, "binary"))`` / ``BinaryScoreSink`` (io.py:160-172, 244-255):
    the "FIDM" header, then N_R x N_Q little-endian u32 cells in row order.  The
    rows stream from the device through pinned staging to the file in chunks
    (fastid_run_kernel_fd), never materialising the matrix in host memory.  A
    partial file is removed if scoring fails, as the reference's sinks do.
    Returns the matrix shape.
    """
    _check_panels(refs.bit_length, refs.word_width, queries.bit_length, queries.word_width)
    rw, qw = np.ascontiguousarray(refs.words), np.ascontiguousarray(queries.words)
    n_r, n_q = rw.shape[0], qw.shape[0]
    dev = _require_cuda(device) if n_r and n_q else None
    with open(path, "wb") as fh:
        try:
            fh.write(_FIDM_HEADER.pack(FIDM_MAGIC, FIDM_VERSION, n_r, n_q))
            fh.flush()
            if n_r and n_q:
                with torch.cuda.device(dev):
                    _native.check(_native.lib().fastid_run_kernel_fd(
                        rw.ctypes.data, n_r, qw.ctypes.data, n_q, rw.shape[1], rw.dtype.itemsize * 8, 0,
                        fh.fileno(), _native.formulation_code(formulation)), "fastid_run_kernel_fd")
        except BaseException:
            fh.close()
            os.unlink(path)
            raise
    return n_r, n_q


class B200Executor:
    """Executor for the reference pipeline's seam (scheduler.py:221-246):
    ``run_pipeline(plan, refs, queries, executor=B200Executor())``."""

    wants_transposed = False

    def __init__(self, formulation: str | int = "auto"):
        self.formulation = formulation
        self.calls = 0

    def run(self, ref_words: np.ndarray, query_words: np.ndarray, out: np.ndarray) -> None:
        self.calls += 1
        run_b200_kernel(ref_words, query_words, out, queries_transposed=self.wants_transposed,
                        formulation=self.formulation)


def topk_workspace_bytes(n_refs: int, n_queries: int, k: int, formulation: str | int = "auto") -> int:
    n = ctypes.c_size_t(0)
    _native.check(_native.lib().fastid_topk_workspace(n_refs, n_queries, k, _native.formulation_code(formulation),
                                                      ctypes.byref(n)), "fastid_topk_workspace")
    return int(n.value)


def topk_device(refs: DevicePanel, queries: DevicePanel, k: int, max_score: int | None = None,
                ref_base: int = 0, formulation: str | int = "auto", workspace: torch.Tensor | None = None,
                out: tuple | None = None, events: tuple | None = None, image=None, op: str = "andnot"):
    """Fused compare + top-k on the device -> (scores int32 [N_Q, k] as u32, index int64 [N_Q, k]).

    On the current stream: the comparison kernel (writing per-CTA candidate
    lists; with a prepared mxf4 image also the spare-pair grid, forked to a
    side stream and joined back) and the merge kernel.  ``events=(start, end)``
    are recorded around the comparison alone (roofline timing).  Every ``op``
    ranks by (score asc, index asc): nearest by AND-NOT or Hamming distance,
    fewest shared ones for "and".
    """
    _check_panels(refs.bit_length, refs.word_width, queries.bit_length, queries.word_width)
    _check_image_op(image, op)
    L = _native.lib()
    max_k = L.fastid_max_k()
    if not 1 <= k <= max_k:
        raise ValueError(f"k must be in [1, {max_k}]")
    dev = refs.device
    n_q = queries.n_profiles
    if out is None:
        out = (torch.empty((n_q, k), dtype=torch.int32, device=dev),
               torch.empty((n_q, k), dtype=torch.int64, device=dev))
    s, x = out
    if n_q == 0:
        return s, x
    ms = EMPTY_SCORE - 1 if max_score is None else int(max_score)
    if refs.n_profiles == 0:
        s.fill_(-1)
        x.fill_(-1)
        return s, x
    need = topk_workspace_bytes(refs.n_profiles, n_q, k, formulation)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    lists, kp = ctypes.c_int(0), ctypes.c_int(0)
    xo, so = ctypes.c_size_t(0), ctypes.c_size_t(0)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        if events is not None:
            events[0].record(stream)
        if image is not None:
            _native.check(L.fastid_db_topk_partials(
                image.handle, _ptr(queries), n_q, k, ms, ref_base, workspace.data_ptr(), workspace.numel(),
                stream.cuda_stream, ctypes.byref(lists), ctypes.byref(kp), ctypes.byref(xo), ctypes.byref(so)),
                "fastid_db_topk_partials")
        else:
            _native.check(L.fastid_topk_partials(
                _ptr(refs), refs.n_profiles, _ptr(queries), n_q, refs.stride, refs.bit_length, k, ms, ref_base,
                workspace.data_ptr(), workspace.numel(), _native.formulation_code(formulation, op), stream.cuda_stream,
                ctypes.byref(lists), ctypes.byref(kp), ctypes.byref(xo), ctypes.byref(so)), "fastid_topk_partials")
        if events is not None:
            events[1].record(stream)
        base = workspace.data_ptr()
        _native.check(L.fastid_merge_topk(base + so.value, base + xo.value, lists.value, n_q, kp.value, k,
                                          s.data_ptr(), x.data_ptr(), stream.cuda_stream), "fastid_merge_topk")
    return s, x


def topk(refs, queries, k: int, max_score: int | None = None, formulation: str | int = "auto",
         device=None, op: str = "andnot") -> TopKResult:
    """Per unknown, the k closest knowns by (score asc, known index asc), optionally score <= max_score."""
    _check_panels(refs.bit_length, refs.word_width, queries.bit_length, queries.word_width)
    dev = _require_cuda(device)
    dr, dq = _as_device(refs, dev), _as_device(queries, dev)
    s, x = topk_device(dr, dq, k, max_score, 0, formulation, op=op)
    q_ids = getattr(queries, "ids", None) or tuple(f"q{j}" for j in range(dq.n_profiles))
    return TopKResult(tuple(q_ids), s.cpu().numpy().view(np.uint32), x.cpu().numpy(),
                      getattr(refs, "ids", None))


def topk_streamed(refs, queries, k: int, max_score: int | None = None, formulation: str | int = "auto",
                  chunk_rows: int = 0, ref_base: int = 0, op: str = "andnot") -> TopKResult:
    """``topk`` for a known panel kept in HOST memory, larger than the device if need be.

    The panel's rows stream through the GPU in chunks (fastid_run_topk: pinned
    double-buffered uploads overlapped with the fused compare + top-k of the
    previous chunk, per-chunk lists merged on the device), so only one chunk
    (``chunk_rows``; 0 = ~512 MB of packed rows) and its tensor image are
    resident.  The result equals ``topk`` over the whole panel.  This is the
    device-side form of the reference's batch planner + pipeline
    (plan_batches scheduler.py:108-140, run_pipeline scheduler.py:270-419)
    with a top-k-reducing sink.  Arguments are Panel-like objects (``words``,
    ``bit_length``, ``word_width``, optional ``ids``) or the reference's Panel.
    """
    _check_panels(refs.bit_length, refs.word_width, queries.bit_length, queries.word_width)
    L = _native.lib()
    max_k = L.fastid_max_k()
    if not 1 <= k <= max_k:
        raise ValueError(f"k must be in [1, {max_k}]")
    if chunk_rows < 0:
        raise ValueError("chunk_rows must be >= 0")
    rw = np.ascontiguousarray(refs.words)
    qw = np.ascontiguousarray(queries.words)
    n_r, n_q = rw.shape[0], qw.shape[0]
    scores = np.empty((n_q, k), np.uint32)
    index = np.empty((n_q, k), np.int64)
    q_ids = getattr(queries, "ids", None) or tuple(f"q{j}" for j in range(n_q))
    if n_q:
        _require_cuda()
        ms = EMPTY_SCORE - 1 if max_score is None else int(max_score)
        _native.check(L.fastid_run_topk(
            rw.ctypes.data if n_r else None, n_r, qw.ctypes.data, n_q, rw.shape[1], rw.dtype.itemsize * 8, k, ms,
            int(ref_base), scores.ctypes.data, index.ctypes.data, int(chunk_rows),
            _native.formulation_code(formulation, op)), "fastid_run_topk")
    return TopKResult(tuple(q_ids), scores, index, getattr(refs, "ids", None))


def threshold_hits(refs, queries, threshold: int, capacity: int | None = None,
                   formulation: str | int = "auto", device=None, ref_base: int = 0, image=None,
                   op: str = "andnot") -> ThresholdHits:
    """Every (unknown j, known i, score) with score <= threshold, ordered by (j, i)."""
    _check_panels(refs.bit_length, refs.word_width, queries.bit_length, queries.word_width)
    _check_image_op(image, op)
    dev = _require_cuda(device)
    dr, dq = _as_device(refs, dev), _as_device(queries, dev)
    cap = int(capacity) if capacity is not None else max(1 << 16, 4 * dq.n_profiles)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    for _ in range(2):
        hq = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        hr = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
        hs = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        with torch.cuda.device(dev):
            if image is not None:
                _native.check(_native.lib().fastid_db_compare_threshold(
                    image.handle, _ptr(dq), dq.n_profiles, int(threshold), ref_base, hq.data_ptr(), hr.data_ptr(),
                    hs.data_ptr(), cap, count.data_ptr(), _stream(dev)), "fastid_db_compare_threshold")
            else:
                _native.check(_native.lib().fastid_compare_threshold(
                    _ptr(dr), dr.n_profiles, _ptr(dq), dq.n_profiles, dr.stride, dr.bit_length, int(threshold),
                    ref_base, hq.data_ptr(), hr.data_ptr(), hs.data_ptr(), cap, count.data_ptr(),
                    _native.formulation_code(formulation, op), _stream(dev)), "fastid_compare_threshold")
        n = int(count.item())
        if n <= cap:
            break
        cap = n  # second pass with an exact-size buffer
    q = hq[:n].cpu().numpy().view(np.uint32)
    r = hr[:n].cpu().numpy()
    sc = hs[:n].cpu().numpy().view(np.uint32)
    order = np.lexsort((r, q))
    return ThresholdHits(q[order], r[order], sc[order], int(threshold))
