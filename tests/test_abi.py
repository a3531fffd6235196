"""The C-ABI library builds/loads and exports every symbol include/fastid_b200.h
declares (no compute calls: CPU-only)."""

import ctypes
import subprocess

import pytest

from paper_1707_00516_b200 import _native


def test_library_exports_every_declared_symbol():
    names = _native.exported_symbols()
    assert len(names) >= 14
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(names) <= exported
    # nothing but the ABI leaks out of the shared object
    assert {n for n in exported if n.startswith("fastid_")} == set(names)


def test_host_only_entry_points():
    lib = _native.lib()
    assert lib.fastid_abi_version() == 1
    assert lib.fastid_row_stride(1) == 16
    assert lib.fastid_row_stride(128) == 16
    assert lib.fastid_row_stride(129) == 32
    assert lib.fastid_row_stride(1024) == 128
    assert lib.fastid_row_stride(5000) == 640
    assert lib.fastid_row_stride(0) == 0
    assert lib.fastid_max_k() == 32
    assert _native.supports("popc", 40000)
    assert _native.supports("tensor_f4", 1024) and _native.supports("tensor_i8", 1024)
    assert not _native.supports("popc", 0)
    n = ctypes.c_size_t(0)
    assert lib.fastid_topk_workspace(20_000_000, 2048, 16, 0, ctypes.byref(n)) == 0
    assert n.value > 2048 * 16 * 12


def test_status_mapping_without_gpu():
    lib = _native.lib()
    # bad k is rejected on the host before any device work
    n = ctypes.c_size_t(0)
    assert lib.fastid_topk_workspace(10, 10, 0, 0, ctypes.byref(n)) == _native.E_INVALID
    assert b"k must be" in lib.fastid_last_error()
    with pytest.raises(ValueError):
        _native.check(_native.E_INVALID, "probe")
    from paper_1707_00516_b200 import PanelMismatchError, DeviceError

    with pytest.raises(PanelMismatchError):
        _native.check(_native.E_MISMATCH, "probe")
    with pytest.raises(DeviceError):
        _native.check(_native.E_CUDA, "probe")


def test_sass_uses_blackwell_features():
    """The built library contains tcgen05 MMAs (UTC*MMA), TMA (UTMALDG) and TMEM loads (LDTM)."""
    out = subprocess.run(["cuobjdump", "-sass", str(_native.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    sass = out.stdout
    assert "UTCIMMA" in sass or "UTCQMMA" in sass or "UTCOMMA" in sass
    assert "UTMALDG" in sass
    assert "LDTM" in sass
    assert "POPC" in sass


def test_experiment_switches_only_in_the_diag_build():
    """The product library neither declares nor exports the process-global timing
    switches (result-invalidating by design); they live in the experiments build."""
    header = (_native.INCLUDE / "fastid_b200.h").read_text()
    assert "fastid_debug_flags" not in header and "fastid_debug_trace" not in header
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "fastid_debug" not in out
    assert "fastid_db_set_option" in out
    diag = (_native.INCLUDE / "fastid_b200_diag.h").read_text()
    assert "fastid_debug_flags" in diag
    if _native.DIAG_LIB_PATH.exists():
        out = subprocess.run(["nm", "-D", "--defined-only", str(_native.DIAG_LIB_PATH)], capture_output=True,
                             text=True).stdout
        assert "fastid_debug_flags" in out and "fastid_debug_trace" in out
