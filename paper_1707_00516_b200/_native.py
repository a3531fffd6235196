"""Loader and build recipe for the in-tree sm_100a library ``_fastid_b200.so``.

The library is compiled from ``csrc/*.cu`` with nvcc for
``-gencode arch=compute_100a,code=sm_100a`` and bound with ctypes (ctypes
releases the GIL around every call, so pipeline lanes keep running while a
kernel is enqueued).  There is no fallback: if the library is missing,
``lib()`` raises ``DeviceError`` and nothing is computed.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from pathlib import Path

from .errors import CapacityError, CorruptProfileError, DeviceError, PanelFormatError, PanelMismatchError

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
INCLUDE = REPO_DIR / "include"
LIB_PATH = PKG_DIR / "_fastid_b200.so"
SOURCES = ("api.cu", "encode.cu", "popc.cu", "tensor.cu", "merge.cu", "probe.cu", "ingest.cu")
HEADERS = ("common.cuh", "tensor_ptx.cuh")

NVCC_FLAGS = (
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-fvisibility=hidden",
    "--expt-relaxed-constexpr",
)

FASTID_OK, E_INVALID, E_MISMATCH, E_CUDA, E_CAPACITY, E_NOMEM, E_UNSUPPORTED, E_FORMAT, E_CORRUPT = range(9)
FORMULATIONS = {"auto": 0, "popc": 1, "tensor_i8": 2, "tensor_f4": 3}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not LIB_PATH.exists():
        return True
    built = LIB_PATH.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + [CSRC / h for h in HEADERS if (CSRC / h).exists()]
    deps.append(INCLUDE / "fastid_b200.h")
    return any(p.exists() and p.stat().st_mtime > built for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile the library in-tree (nvcc cross-compiles without a GPU)."""
    if not force and not _stale():
        return LIB_PATH
    tmp = LIB_PATH.with_suffix(f".so.tmp{os.getpid()}")
    cmd = [_nvcc(), *NVCC_FLAGS, f"-I{INCLUDE}", "-shared", "-o", str(tmp),
           *[str(CSRC / s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=str(CSRC))
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    """The loaded library; raises DeviceError if it was never built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise DeviceError(
                f"{LIB_PATH.name} is not built; run __graft_entry__.build() "
                "(there is no CPU fallback for the comparison path)")
        L = ctypes.CDLL(str(LIB_PATH))
        vp, i64, i32, u32, sz = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                 ctypes.c_uint32, ctypes.c_size_t)
        sig = {
            "fastid_abi_version": ([], i32),
            "fastid_last_error": ([], ctypes.c_char_p),
            "fastid_row_stride": ([i64], i64),
            "fastid_max_k": ([], i32),
            "fastid_supports": ([i32, i64], i32),
            "fastid_load_words": ([vp, i64, i64, vp, i64, vp], i32),
            "fastid_pack_bits": ([vp, i64, i64, i32, vp, i64, vp], i32),
            "fastid_pack_genotypes": ([vp, i64, i64, i32, vp, i64, vp], i32),
            "fastid_compare_full": ([vp, i64, vp, i64, i64, i64, vp, i64, i32, vp], i32),
            "fastid_topk_workspace": ([i64, i64, i32, i32, ctypes.POINTER(sz)], i32),
            "fastid_compare_topk": ([vp, i64, vp, i64, i64, i64, i32, u32, i64, vp, vp, vp, sz, i32, vp], i32),
            "fastid_topk_partials": ([vp, i64, vp, i64, i64, i64, i32, u32, i64, vp, sz, i32, vp,
                                      ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(sz),
                                      ctypes.POINTER(sz)], i32),
            "fastid_compare_threshold": ([vp, i64, vp, i64, i64, i64, u32, i64, vp, vp, vp, i64, vp, i32, vp], i32),
            "fastid_merge_topk": ([vp, vp, i32, i64, i32, i32, vp, vp, vp], i32),
            "fastid_run_kernel": ([vp, i64, vp, i64, i64, i32, i32, vp, i32], i32),
            "fastid_run_kernel_fd": ([vp, i64, vp, i64, i64, i32, i32, i32, i32], i32),
            "fastid_parse_panel": ([vp, i64, i32, i32, ctypes.POINTER(vp)], i32),
            "fastid_parsed_panel_shape": ([vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64),
                                           ctypes.POINTER(i64)], i32),
            "fastid_parsed_panel_copy": ([vp, vp, vp, vp], i32),
            "fastid_parsed_panel_free": ([vp], None),
            "fastid_db_image_bytes": ([i64, i64, i32], sz),
            "fastid_db_create": ([vp, i64, i64, i64, i32, vp, ctypes.POINTER(vp)], i32),
            "fastid_db_destroy": ([vp], i32),
            "fastid_db_formulation": ([vp], i32),
            "fastid_db_compare_full": ([vp, vp, i64, vp, i64, vp], i32),
            "fastid_db_topk_partials": ([vp, vp, i64, i32, u32, i64, vp, sz, vp, ctypes.POINTER(i32),
                                         ctypes.POINTER(i32), ctypes.POINTER(sz), ctypes.POINTER(sz)], i32),
            "fastid_db_compare_threshold": ([vp, vp, i64, u32, i64, vp, vp, vp, i64, vp, vp], i32),
            "fastid_probe_peak": ([i32, i32, vp, ctypes.POINTER(ctypes.c_double), vp], i32),
            "fastid_probe_tmem_read": ([i32, i32, i32, vp, ctypes.POINTER(ctypes.c_double), vp], i32),
            "fastid_debug_trace": ([vp, i32], i32),
            "fastid_debug_flags": ([i32], i32),
            "fastid_probe_contention": ([i32, i32, vp, vp], i32),
            "fastid_probe_variant": ([i32, i32, i32, vp, vp, i64, ctypes.POINTER(ctypes.c_double), vp], i32),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        if L.fastid_abi_version() != 1:
            raise DeviceError("ABI version mismatch between include/fastid_b200.h and the library")
        _lib = L
        return _lib


def exported_symbols() -> list[str]:
    """Names declared in include/fastid_b200.h (for the export check)."""
    import re

    text = (INCLUDE / "fastid_b200.h").read_text()
    return sorted(set(re.findall(r"\b(fastid_[a-z_0-9]+)\s*\(", text)))


def check(status: int, what: str) -> None:
    """Map a fastid_status to the reference's exception types."""
    if status == FASTID_OK:
        return
    msg = f"{what}: {lib().fastid_last_error().decode(errors='replace')}"
    if status == E_INVALID:
        raise ValueError(msg)
    if status == E_MISMATCH:
        raise PanelMismatchError(msg)
    if status == E_CAPACITY:
        raise CapacityError(msg, required=-1)
    if status == E_FORMAT:
        raise PanelFormatError(msg)
    if status == E_CORRUPT:
        raise CorruptProfileError(msg)
    raise DeviceError(msg)


def supports(formulation: str | int, bit_length: int) -> bool:
    """Whether `formulation` can run panels of `bit_length` loci."""
    return bool(lib().fastid_supports(formulation_code(formulation), int(bit_length)))


def formulation_code(name: str | int) -> int:
    if isinstance(name, int):
        return name
    try:
        return FORMULATIONS[name]
    except KeyError:
        raise ValueError(f"formulation must be one of {sorted(FORMULATIONS)}, got {name!r}") from None
