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
# The bitwise operator before the popcount (enum fastid_operator, carried in
# bits 8-9 of a formulation argument): r AND NOT q (FastID Eq. 1, the
# default), r AND q (shared ones), r XOR q (Hamming distance).
OPERATORS = {"andnot": 0, "and": 0x100, "xor": 0x200}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    return "nvcc"


DIAG_LIB_PATH = PKG_DIR / "_fastid_b200_diag.so"
BUILD_DIR = PKG_DIR / "_build"


def _stale(path: Path) -> bool:
    if not path.exists():
        return True
    built = path.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + [CSRC / h for h in HEADERS if (CSRC / h).exists()]
    deps += [INCLUDE / "fastid_b200.h", INCLUDE / "fastid_b200_diag.h"]
    return any(p.exists() and p.stat().st_mtime > built for p in deps)


def _compile(path: Path, extra: tuple, verbose: bool) -> Path:
    """nvcc every source to an object in parallel, then link the shared library."""
    from concurrent.futures import ThreadPoolExecutor

    objdir = BUILD_DIR / path.stem
    objdir.mkdir(parents=True, exist_ok=True)

    def one(src: str) -> Path:
        obj = objdir / (Path(src).stem + ".o")
        cmd = [_nvcc(), *NVCC_FLAGS, *extra, f"-I{INCLUDE}", "-c", "-o", str(obj), str(CSRC / src)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True, cwd=str(CSRC))
        return obj

    # the tensor kernels take longest: start them first
    order = sorted(SOURCES, key=lambda s: s != "tensor.cu")
    with ThreadPoolExecutor(max_workers=min(len(order), os.cpu_count() or 1)) as pool:
        objs = list(pool.map(one, order))
    tmp = path.with_suffix(f".so.tmp{os.getpid()}")
    cmd = [_nvcc(), *NVCC_FLAGS, "-shared", "-o", str(tmp), *map(str, objs)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=str(CSRC))
    os.replace(tmp, path)
    return path


def build(force: bool = False, verbose: bool = False, diag: bool = False) -> Path:
    """Compile the product library in-tree (nvcc cross-compiles without a GPU).

    ``diag=True`` also builds the experiments library (_fastid_b200_diag.so,
    -DFASTID_EXPERIMENTS) that the timing tools in tools/ load.
    """
    if force or _stale(LIB_PATH):
        _compile(LIB_PATH, (), verbose)
    if diag and (force or _stale(DIAG_LIB_PATH)):
        _compile(DIAG_LIB_PATH, ("-DFASTID_EXPERIMENTS",), verbose)
    return LIB_PATH


def _bind(L: ctypes.CDLL, sig: dict) -> None:
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res


def _signatures() -> dict:
    vp, i64, i32, u32, sz = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint32, ctypes.c_size_t)
    return {
        "fastid_abi_version": ([], i32),
        "fastid_last_error": ([], ctypes.c_char_p),
        "fastid_row_stride": ([i64], i64),
        "fastid_launch_count": ([], ctypes.c_ulonglong),
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
        "fastid_run_topk": ([vp, i64, vp, i64, i64, i32, i32, u32, i64, vp, vp, i64, i32], i32),
        "fastid_parse_panel": ([vp, i64, i32, i32, ctypes.POINTER(vp)], i32),
        "fastid_parsed_panel_shape": ([vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64),
                                       ctypes.POINTER(i64)], i32),
        "fastid_parsed_panel_copy": ([vp, vp, vp, vp], i32),
        "fastid_parsed_panel_free": ([vp], None),
        "fastid_db_image_bytes": ([i64, i64, i32], sz),
        "fastid_db_create": ([vp, i64, i64, i64, i32, vp, ctypes.POINTER(vp)], i32),
        "fastid_db_create_in": ([vp, i64, i64, i64, i32, vp, sz, vp, ctypes.POINTER(vp)], i32),
        "fastid_db_destroy": ([vp], i32),
        "fastid_db_formulation": ([vp], i32),
        "fastid_db_set_option": ([vp, i32, i32], i32),
        "fastid_db_set_operator": ([vp, i32], i32),
        "fastid_db_options": ([vp], i32),
        "fastid_db_compare_full": ([vp, vp, i64, vp, i64, vp], i32),
        "fastid_db_topk_partials": ([vp, vp, i64, i32, u32, i64, vp, sz, vp, ctypes.POINTER(i32),
                                     ctypes.POINTER(i32), ctypes.POINTER(sz), ctypes.POINTER(sz)], i32),
        "fastid_db_compare_threshold": ([vp, vp, i64, u32, i64, vp, vp, vp, i64, vp, vp], i32),
        "fastid_probe_peak": ([i32, i32, vp, ctypes.POINTER(ctypes.c_double), vp], i32),
        "fastid_probe_tmem_read": ([i32, i32, i32, vp, ctypes.POINTER(ctypes.c_double), vp], i32),
        "fastid_probe_contention": ([i32, i32, vp, vp], i32),
        "fastid_probe_variant": ([i32, i32, i32, vp, vp, i64, ctypes.POINTER(ctypes.c_double), vp], i32),
    }


def lib() -> ctypes.CDLL:
    """The loaded library; raises DeviceError if it was never built.

    This is the product library _fastid_b200.so, unless the process set
    FASTID_DIAG=1 before the first call (tools/ only): then it is the
    experiments build _fastid_b200_diag.so, which also exports the timing
    switches of include/fastid_b200_diag.h.
    """
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        diag = os.environ.get("FASTID_DIAG") == "1"
        if diag:
            build(diag=True)
        path = DIAG_LIB_PATH if diag else LIB_PATH
        if not path.exists():
            raise DeviceError(
                f"{path.name} is not built; run __graft_entry__.build() "
                "(there is no CPU fallback for the comparison path)")
        L = ctypes.CDLL(str(path))
        sig = _signatures()
        if diag:
            sig["fastid_debug_trace"] = ([ctypes.c_void_p, ctypes.c_int], ctypes.c_int)
            sig["fastid_debug_flags"] = ([ctypes.c_int], ctypes.c_int)
        _bind(L, sig)
        if L.fastid_abi_version() != 1:
            raise DeviceError("ABI version mismatch between include/fastid_b200.h and the library")
        _lib = L
        return _lib


def diag_lib() -> ctypes.CDLL:
    """The experiments build for the timing tools in tools/: sets FASTID_DIAG=1
    and loads it (every package call in the process then runs on it).  Must be
    called before anything loads the product library."""
    if _lib is not None and os.environ.get("FASTID_DIAG") != "1":
        raise RuntimeError("the product library is already loaded; call diag_lib() first")
    os.environ["FASTID_DIAG"] = "1"
    return lib()


def exported_symbols() -> list[str]:
    """Names declared in include/fastid_b200.h (for the export check)."""
    import re

    text = (INCLUDE / "fastid_b200.h").read_text()
    text = text[text.index("#ifdef __cplusplus"):]  # declarations only (not the header comment)
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


def operator_code(op: str) -> int:
    try:
        return OPERATORS[op]
    except KeyError:
        raise ValueError(f"op must be one of {sorted(OPERATORS)}, got {op!r}") from None


def formulation_code(name: str | int, op: str = "andnot") -> int:
    if isinstance(name, int):
        return name | operator_code(op)
    try:
        return FORMULATIONS[name] | operator_code(op)
    except KeyError:
        raise ValueError(f"formulation must be one of {sorted(FORMULATIONS)}, got {name!r}") from None
