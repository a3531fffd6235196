"""Bulk panel ingest (csrc/ingest.cu) against the reference's own load_panel
results (tests/golden/panel_cases.json, made by make_golden.py from
io.load_panel, io.py:45-127): same ids / bit length / words, or the same
exception type and message.  Host code only -- runs without a GPU."""

import json

import numpy as np
import pytest

from conftest import GOLDEN

CASES = json.loads((GOLDEN / "panel_cases.json").read_text())


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
@pytest.mark.parametrize("width", [32, 64])
@pytest.mark.parametrize("threads", [1, 3])
def test_load_panel_matches_reference(tmp_path, case, width, threads):
    import paper_1707_00516_b200 as m
    from paper_1707_00516_b200.ingest import load_panel

    path = tmp_path / "p.panel"
    path.write_bytes(case["text"].encode("utf-8"))
    exp = case["results"][str(width)]
    if "error" in exp:
        err = {"PanelFormatError": m.PanelFormatError, "CorruptProfileError": m.CorruptProfileError}[exp["error"]]
        with pytest.raises(err) as info:
            load_panel(path, width, n_threads=threads)
        assert type(info.value) is err
        assert str(info.value) == exp["message"].replace("<path>", str(path))
        return
    p = load_panel(path, width, n_threads=threads)
    assert p.ids == tuple(exp["ids"]) and p.bit_length == exp["bit_length"]
    words = np.array([[int(w, 16) for w in r] for r in exp["words"]], dtype=p.words.dtype).reshape(p.words.shape)
    assert np.array_equal(p.words, words)


def test_parse_many_threads_large(rng):
    """A larger generated panel parsed with 1 and many threads gives identical words and ids."""
    from paper_1707_00516_b200.ingest import parse_panel_text

    L = 1000
    words = rng.integers(0, 2**64, (20_000, 16), dtype=np.uint64)
    words[:, -1] &= np.uint64(~((1 << 24) - 1) & (2**64 - 1))
    lines = ["#bits=1000"] + [f"p{i}\t" + "".join(f"{int(w):016x}" for w in row)[:250] for i, row in enumerate(words)]
    text = ("\n".join(lines) + "\n").encode()
    a = parse_panel_text(text, 64, 1)
    b = parse_panel_text(text, 64, 8)
    assert a[0] == b[0] and a[2] == b[2] == L and np.array_equal(a[1], b[1])
    assert np.array_equal(a[1], words)
