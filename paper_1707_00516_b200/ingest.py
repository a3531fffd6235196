"""Bulk panel ingest: the reference's text panel format parsed
in native code.

``load_panel(path, word_width)`` is ``fastid.io.load_panel`` (io.py:45-127):
the same ``#bits=<L>`` header rule, comments, blank lines, ``<id><TAB><hex>``
profiles, universal newlines, zero-extension / truncation of the hex string,
and the same errors (``PanelFormatError`` / ``CorruptProfileError``, first
offending line wins, reference wording).  The parse runs multi-threaded in
``csrc/ingest.cu``; ``load_panel_device`` sends the words straight to the GPU
row layout.  Ids must be valid UTF-8 (``UnicodeDecodeError`` otherwise, as
the reference's text-mode read raises); other bytes are validated as hex.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import CorruptProfileError, PanelFormatError
from .panel import Panel, word_dtype


def parse_panel_text(data: bytes, word_width: int = 64, n_threads: int = 0):
    """Panel text -> (ids tuple[str], words ndarray (N, ceil(L/W)), bit_length)."""
    word_dtype(word_width)
    L = _native.lib()
    buf = np.frombuffer(data, dtype=np.uint8) if len(data) else np.zeros(1, np.uint8)
    handle = ctypes.c_void_p()
    status = L.fastid_parse_panel(buf.ctypes.data, len(data), int(word_width), int(n_threads), ctypes.byref(handle))
    if status != _native.FASTID_OK:
        msg = L.fastid_last_error().decode(errors="replace")
        if status == _native.E_FORMAT:
            raise PanelFormatError(msg)
        if status == _native.E_CORRUPT:
            raise CorruptProfileError(msg)
        _native.check(status, "fastid_parse_panel")
    try:
        n, bits, nw, nb = (ctypes.c_int64() for _ in range(4))
        _native.check(L.fastid_parsed_panel_shape(handle, ctypes.byref(n), ctypes.byref(bits), ctypes.byref(nw),
                                                  ctypes.byref(nb)), "fastid_parsed_panel_shape")
        words = np.empty((n.value, nw.value), dtype=word_dtype(word_width))
        id_bytes = np.empty(max(nb.value, 1), np.uint8)
        offsets = np.empty(n.value + 1, np.int64)
        _native.check(L.fastid_parsed_panel_copy(handle, words.ctypes.data, id_bytes.ctypes.data,
                                                 offsets.ctypes.data), "fastid_parsed_panel_copy")
    finally:
        L.fastid_parsed_panel_free(handle)
    # ids arrive joined by '\n' (an id holds neither a tab nor a line break)
    ids = tuple(id_bytes[: nb.value].tobytes().decode("utf-8").split("\n")) if n.value else ()
    return ids, words, bits.value


def load_panel(path, word_width: int = 64, n_threads: int = 0) -> Panel:
    """``fastid.io.load_panel`` on native code (io.py:45-127)."""
    with open(path, "rb") as fh:
        data = fh.read()
    try:
        ids, words, bit_length = parse_panel_text(data, word_width, n_threads)
    except PanelFormatError as e:
        if "missing #bits=<L> header" in str(e):
            raise PanelFormatError(f"{path}: missing #bits=<L> header") from None
        raise
    return Panel(ids, words, bit_length)


def load_panel_device(path, device=None, word_width: int = 64, n_threads: int = 0):
    """Parse a panel file and upload it to the device row layout (DevicePanel, ids kept)."""
    from .compare import DevicePanel

    p = load_panel(path, word_width, n_threads)
    return DevicePanel.from_words(p.words, p.bit_length, ids=p.ids, device=device)


def save_panel(panel, path) -> None:
    """``fastid.io.save_panel`` (io.py:130-141): ``#bits=<L>`` then ``<id><TAB><HEX>`` lines, uppercase."""
    digits = panel.word_width // 4
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write(f"#bits={panel.bit_length}\n")
        for ident, row in zip(panel.ids, panel.words):
            if not ident:
                raise PanelFormatError("line 0: empty profile id")
            if "," in ident:
                raise PanelFormatError(f"line 0: id {ident!r} contains a CSV separator")
            fh.write(f"{ident}\t" + "".join(f"{int(w):0{digits}X}" for w in row) + "\n")


__all__ = ["load_panel", "load_panel_device", "parse_panel_text", "save_panel"]
