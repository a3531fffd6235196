"""Out-of-core top-k (fastid_run_topk / topk_streamed): a host-resident known
panel streamed through the device in chunks must give exactly the oracle's
top-k over the whole panel -- chunk boundaries, ragged last chunks, ties that
straddle chunks (lower global index wins), max_score caps, ref_base offsets,
page-locked and pageable host rows, and every formulation."""

import numpy as np
import pytest

import oracle

from conftest import gpu_available, rand_words

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def fb():
    import paper_1707_00516_b200 as m

    return m


def _panels(rng, n_r, n_q, L, width=64, dup_across=True):
    nw = -(-L // width)
    r, _ = rand_words(rng, n_r, nw, width, L)
    q, _ = rand_words(rng, n_q, nw, width, L)
    q[: min(16, n_q)] = r[rng.integers(0, n_r, min(16, n_q))]  # exact copies: score 0
    if dup_across and n_r > 8:
        r[-3:] = r[:3]  # duplicates in the last chunk: ties resolved to the lower index
    m = fb()
    return r, q, m.Panel(tuple(range(n_r)), r, L), m.Panel(tuple(range(n_q)), q, L)


@pytest.mark.parametrize("form", ["tensor_f4", "tensor_i8", "popc"])
@pytest.mark.parametrize("n_r,n_q,L,chunk", [
    (50_000, 300, 1024, 7_777),   # 7 chunks, ragged tail
    (20_000, 64, 5000, 4_096),    # streamed-A (dual-tile) pair kernel per chunk
    (3_001, 129, 777, 1_000),     # u64 words, partial last word, tiny chunks
])
def test_streamed_topk_matches_oracle(rng, form, n_r, n_q, L, chunk):
    m = fb()
    if not m._native.supports(form, L):
        pytest.skip("formulation does not run this length")
    r, q, R, Q = _panels(rng, n_r, n_q, L)
    for k, ms in ((16, None), (1, None), (32, None), (8, L // 3)):
        res = m.topk_streamed(R, Q, k, max_score=ms, formulation=form, chunk_rows=chunk)
        es, ex, _ = oracle.topk(r, q, k, 0xFFFFFFFE if ms is None else ms)
        assert np.array_equal(res.scores, es), (form, n_r, L, k, ms)
        assert np.array_equal(res.index, ex), (form, n_r, L, k, ms)


def test_streamed_equals_resident_and_one_chunk(rng):
    m = fb()
    r, q, R, Q = _panels(rng, 40_000, 256, 1024)
    whole = m.topk(R, Q, 16)
    for chunk in (0, 40_000, 39_999, 192, 193):
        got = m.topk_streamed(R, Q, 16, chunk_rows=chunk)
        assert np.array_equal(got.scores, whole.scores), chunk
        assert np.array_equal(got.index, whole.index), chunk


def test_streamed_ref_base_and_u32_words(rng):
    m = fb()
    n_r, n_q, L = 10_000, 100, 1000
    r, _ = rand_words(rng, n_r, -(-L // 32), 32, L)
    q, _ = rand_words(rng, n_q, -(-L // 32), 32, L)
    q[:10] = r[:10]
    R, Q = m.Panel(tuple(range(n_r)), r, L), m.Panel(tuple(range(n_q)), q, L)
    res = m.topk_streamed(R, Q, 4, chunk_rows=3_000, ref_base=1_000_000)
    es, ex, _ = oracle.topk(r, q, 4, 0xFFFFFFFE)
    assert np.array_equal(res.scores, es)
    assert np.array_equal(res.index, np.where(ex >= 0, ex + 1_000_000, -1))


def test_streamed_page_locked_rows(rng):
    import torch

    m = fb()
    r, q, R, Q = _panels(rng, 30_000, 128, 1024)
    pinned = torch.from_numpy(r.view(np.int64)).pin_memory()
    Rp = m.Panel(tuple(range(r.shape[0])), pinned.numpy().view(np.uint64), 1024)
    got = m.topk_streamed(Rp, Q, 16, chunk_rows=4_000)
    es, ex, _ = oracle.topk(r, q, 16, 0xFFFFFFFE)
    assert np.array_equal(got.scores, es) and np.array_equal(got.index, ex)


def test_streamed_empty_and_errors(rng):
    m = fb()
    r, q, R, Q = _panels(rng, 100, 10, 1024)
    E = m.Panel((), np.zeros((0, 16), np.uint64), 1024)
    res = m.topk_streamed(E, Q, 5)
    assert (res.scores == 0xFFFFFFFF).all() and (res.index == -1).all()
    res = m.topk_streamed(R, m.Panel((), np.zeros((0, 16), np.uint64), 1024), 5)
    assert res.scores.shape == (0, 5)
    with pytest.raises(ValueError):
        m.topk_streamed(R, Q, 0)
    with pytest.raises(ValueError):
        m.topk_streamed(R, Q, 5, chunk_rows=-1)
    with pytest.raises(m.PanelMismatchError):
        m.topk_streamed(R, m.Panel(("x",), np.zeros((1, 8), np.uint64), 512), 5)
