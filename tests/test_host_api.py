"""Host-side logic: panel validation, errors, layout helpers (CPU only)."""

import numpy as np
import pytest

import paper_1707_00516_b200 as fb
from paper_1707_00516_b200.sharded import shard_range


def test_panel_validation_matches_reference_rules():
    with pytest.raises(fb.CorruptProfileError):
        fb.Panel(("a",), np.array([[1]], dtype=np.uint32), bit_length=8)
    with pytest.raises(ValueError):
        fb.Panel(("a",), np.array([[0, 0]], dtype=np.uint32), bit_length=32)
    with pytest.raises(ValueError):
        fb.Panel(("a",), np.array([[0]], dtype=np.int32), bit_length=32)
    with pytest.raises(ValueError):
        fb.Panel(("a", "b"), np.zeros((1, 1), np.uint64), 64)
    p = fb.Panel(("a",), np.array([[0xF0000000]], dtype=np.uint32), 8)
    assert p.n_profiles == 1 and p.n_words == 1 and p.word_width == 32
    assert not p.words.flags.writeable


def test_relayout_round_trip(rng):
    w = rng.integers(0, 2**63, (7, 3), dtype=np.uint64)
    p = fb.Panel(tuple("abcdefg"), w, 192)
    lay = fb.relayout_queries(p)
    assert lay.words.shape == (3, 7) and lay.n_queries == 7
    back = fb.restore_queries(lay)
    assert np.array_equal(back.words, w) and back.ids == p.ids
    two = fb.Panel(("x", "y"), np.array([[1, 2], [3, 4]], dtype=np.uint32), 64)
    assert fb.relayout_queries(two).words.ravel().tolist() == [1, 3, 2, 4]


def test_tile_config_validation():
    fb.TileConfig(16)
    with pytest.raises(ValueError):
        fb.TileConfig(17)
    with pytest.raises(ValueError):
        fb.TileConfig(64, 0)


def test_row_stride():
    assert fb.row_stride(1) == 16 and fb.row_stride(1024) == 128 and fb.row_stride(5000) == 640
    for L in range(1, 600, 7):
        s = fb.row_stride(L)
        assert s % 16 == 0 and s * 8 >= L and (s - 16) * 8 < L


def test_score_matrix_type():
    m = fb.ScoreMatrix(("r",), ("q0", "q1"), np.array([[1, 2]]))
    assert m.scores.dtype == np.uint32 and m.shape == (1, 2)
    with pytest.raises(ValueError):
        fb.ScoreMatrix(("r",), ("q",), np.zeros((2, 2)))


def test_shard_ranges_partition():
    for n in (0, 1, 7, 20_000_000, 20_000_001):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_device_calls_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    r = fb.Panel(("a",), np.zeros((1, 1), np.uint64), 64)
    with pytest.raises(fb.DeviceError):
        fb.compare_b200(r, r)
    with pytest.raises(fb.DeviceError):
        fb.topk(r, r, 1)


def test_mismatch_checked_before_device():
    a = fb.Panel(("a",), np.zeros((1, 2), np.uint32), 64)
    b = fb.Panel(("b",), np.zeros((1, 2), np.uint32), 40)
    with pytest.raises(fb.PanelMismatchError):
        fb.compare_b200(a, b)
    c = fb.Panel(("c",), np.zeros((1, 1), np.uint64), 64)
    with pytest.raises(fb.PanelMismatchError):
        fb.compare_b200(a, c)
    with pytest.raises(ValueError):
        fb.compare_blocked_b200(a, fb.relayout_queries(a), fb.TileConfig(16), 0)
    # empty panels need no device
    e = fb.Panel((), np.zeros((0, 2), np.uint32), 64)
    assert fb.compare_b200(e, a).shape == (0, 1)


def test_cli_exit_codes(tmp_path):
    """Usage errors exit 2 (argparse), unreadable inputs exit 1 -- cli.py:3-4, 231-241."""
    import pytest
    from paper_1707_00516_b200.__main__ import main

    with pytest.raises(SystemExit) as info:
        main(["compare", "--refs", "a"])
    assert info.value.code == 2
    assert main(["compare", "--refs", str(tmp_path / "nope"), "--queries", "q", "--out", "o"]) == 1


def test_device_panel_validates_words_before_device_work():
    """DevicePanel.from_words (behind KnownDatabase(raw_words, L)) applies the
    reference Panel's rules on the host before touching a device: wrong word
    counts raise ValueError, nonzero padding CorruptProfileError."""
    with pytest.raises(ValueError):
        fb.DevicePanel.from_words(np.zeros((3, 1), np.uint64), 100)  # needs 2 words
    with pytest.raises(ValueError):
        fb.DevicePanel.from_words(np.zeros((3, 3), np.uint32), 64)   # needs 2 words
    bad = np.zeros((2, 2), np.uint64)
    bad[1, 1] = 1  # bit 127 set, L = 100
    with pytest.raises(fb.CorruptProfileError):
        fb.DevicePanel.from_words(bad, 100)
    with pytest.raises(ValueError):
        fb.DevicePanel.from_words(np.zeros((2, 2), np.uint64), 0)


def test_known_database_options_are_named():
    from paper_1707_00516_b200.search import DB_OPTIONS

    assert DB_OPTIONS == {"no_cta_pairs": 1, "no_tma_store": 2, "no_spare_pairs": 4, "narrow_tma_store": 8}


def test_operator_codes_and_validation():
    """op= maps to the C ABI's operator bits (include/fastid_b200.h); unknown
    operators are rejected before any device work, by Python and by the library."""
    from paper_1707_00516_b200 import _native

    assert _native.formulation_code("tensor_f4") == 3
    assert _native.formulation_code("tensor_f4", "and") == 3 | 0x100
    assert _native.formulation_code(1, "xor") == 1 | 0x200
    with pytest.raises(ValueError):
        _native.formulation_code("auto", "nand")
    L = _native.lib()
    assert L.fastid_supports(3 | 0x200, 1024) == 1
    assert L.fastid_supports(0x300, 1024) == 0  # no such operator
    assert L.fastid_db_set_operator(None, 0) == _native.E_INVALID
    a = fb.Panel(("a",), np.zeros((1, 1), np.uint64), 64)
    with pytest.raises(ValueError):
        fb.compare_b200(a, a, op="or")
