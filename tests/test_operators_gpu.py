"""The bitwise operator before the popcount: AND-NOT (Eq. 1), AND and XOR.

The reference computes AND-NOT only (kernel.py:33-35); AND and
XOR are operator extensions whose oracle is their definition
(oracle.np_scores_op: popcount of the word-wise AND / XOR, PARITY UNPINNED
against the reference).  Every kernel family -- the LOP3+POPC tiles, the
few-unknown scan, the tcgen05 kernels on packed rows, the prepared image with
resident and streamed unknowns, CTA pairs and dual tiles, chunked images and
the host-streamed top-k -- must give the oracle's matrix, top-k lists and
threshold hits bit-exactly for each operator.  Bar: bit-exact.
"""

import numpy as np
import pytest

import oracle

from conftest import gpu_available, rand_words

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

OPS = ["andnot", "and", "xor"]


def fb():
    import paper_1707_00516_b200 as m

    return m


def _case(rng, n_r, n_q, L, dup=20):
    nw = -(-L // 64)
    r, _ = rand_words(rng, n_r, nw, 64, L)
    q, _ = rand_words(rng, n_q, nw, 64, L)
    d = min(dup, n_q)
    q[:d] = r[rng.integers(0, n_r, d)]
    if n_r > 4:
        r[-2:] = r[:2]  # ties across the first and last tiles
    return r, q


def _check_all(m, r, q, L, op, form, k=16):
    exp = oracle.np_scores_op(r, q, op)
    rp = m.Panel(tuple(range(r.shape[0])), r, L)
    qp = m.Panel(tuple(range(q.shape[0])), q, L)
    full = m.compare_b200(rp, qp, formulation=form, op=op).scores
    assert np.array_equal(full, exp), (op, form, "full")
    res = m.topk(rp, qp, k, formulation=form, op=op)
    es, ex, _ = oracle.topk_from_matrix(exp, k)
    assert np.array_equal(res.scores, es) and np.array_equal(res.index, ex), (op, form, "topk")
    thr = int(np.percentile(exp, 2))
    hits = m.threshold_hits(rp, qp, thr, formulation=form, op=op)
    hq, hr, hs = oracle.threshold_from_matrix(exp, thr)
    assert np.array_equal(hits.query, hq) and np.array_equal(hits.ref, hr) and np.array_equal(hits.score, hs), \
        (op, form, "threshold")
    return exp


def test_np_scores_op_andnot_is_eq1(rng):
    r, q = _case(rng, 50, 7, 300)
    assert np.array_equal(oracle.np_scores_op(r, q, "andnot"), oracle.naive(r, q))
    # XOR = popc(r) + popc(q) - 2 popc(r & q): the identity the tensor epilogue uses
    pr = np.bitwise_count(r).sum(axis=1, dtype=np.int64)
    pq = np.bitwise_count(q).sum(axis=1, dtype=np.int64)
    both = oracle.np_scores_op(r, q, "and").astype(np.int64)
    assert np.array_equal(oracle.np_scores_op(r, q, "xor"), pr[:, None] + pq[None, :] - 2 * both)


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("form", ["popc", "tensor_i8", "tensor_f4"])
@pytest.mark.parametrize("L", [300, 1024, 5000])
def test_operator_direct(rng, op, form, L):
    """Unprepared calls: packed rows, each formulation, full / top-k / threshold."""
    m = fb()
    from paper_1707_00516_b200 import _native

    if not _native.supports(form, L):
        pytest.skip("formulation does not run this length")
    r, q = _case(rng, 1500, 140, L)
    _check_all(m, r, q, L, op, form)


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("n_q", [1, 3, 16])
def test_operator_scan(rng, op, n_q):
    """A handful of unknowns: the CUDA-core scan (top-k and threshold)."""
    m = fb()
    L = 1024
    r, q = _case(rng, 20_000, n_q, L, dup=1)
    exp = oracle.np_scores_op(r, q, op)
    rp = m.Panel(tuple(range(r.shape[0])), r, L)
    qp = m.Panel(tuple(range(n_q)), q, L)
    res = m.topk(rp, qp, 16, formulation="popc", op=op)
    es, ex, _ = oracle.topk_from_matrix(exp, 16)
    assert np.array_equal(res.scores, es) and np.array_equal(res.index, ex)
    thr = int(np.percentile(exp, 1))
    hits = m.threshold_hits(rp, qp, thr, formulation="popc", op=op)
    hq, hr, hs = oracle.threshold_from_matrix(exp, thr)
    assert np.array_equal(hits.query, hq) and np.array_equal(hits.ref, hr) and np.array_equal(hits.score, hs)


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("n_r,n_q,L", [(2500, 150, 1024), (22_222, 300, 5000), (30_000, 600, 1024),
                                       (5000, 40, 2048)])
def test_operator_prepared_image(rng, op, n_r, n_q, L):
    """KnownDatabase (prepared mxf4 image: CTA pairs, resident and streamed unknowns,
    dual tiles at L = 5000, spare pairs) with each operator, and the routing of
    small batches to the scan / packed-row kernels."""
    m = fb()
    from paper_1707_00516_b200.search import KnownDatabase

    r, q = _case(rng, n_r, n_q, L)
    exp = oracle.np_scores_op(r, q, op)
    db = KnownDatabase(r, L, op=op, ref_base=7)
    dq = m.DevicePanel.from_words(q, L)
    full = db.full_device(dq).cpu().numpy().view(np.uint32)
    assert np.array_equal(full, exp)
    for k in (16, 5):
        s, x = db.search_words(q, k)
        es, ex, _ = oracle.topk_from_matrix(exp, k)
        assert np.array_equal(s, es) and np.array_equal(x, np.where(ex >= 0, ex + 7, -1)), k
    thr = int(np.percentile(exp, 1))
    hits = db.threshold(m.Panel(tuple(range(n_q)), q, L), thr)
    hq, hr, hs = oracle.threshold_from_matrix(exp, thr)
    assert np.array_equal(hits.query, hq) and np.array_equal(hits.ref, hr + 7) and np.array_equal(hits.score, hs)
    for nq in (1, 4, 100):  # scan and packed-row routes of an "auto" database
        s, x = db.search_words(q[:nq], 8)
        es, ex, _ = oracle.topk_from_matrix(exp[:, :nq], 8)
        assert np.array_equal(s, es) and np.array_equal(x, np.where(ex >= 0, ex + 7, -1)), nq


@pytest.mark.parametrize("op", ["and", "xor"])
def test_operator_chunked_image_and_streamed(rng, op):
    """A chunked image and the host-streamed top-k carry the operator through."""
    m = fb()
    from paper_1707_00516_b200.search import KnownDatabase

    L = 1024
    r, q = _case(rng, 12_000, 300, L)
    exp = oracle.np_scores_op(r, q, op)
    db = KnownDatabase(r, L, op=op, image_chunk_rows=192 * 17)
    db.chunked_min_queries = 1
    s, x = db.search_words(q, 16)
    es, ex, _ = oracle.topk_from_matrix(exp, 16)
    assert np.array_equal(s, es) and np.array_equal(x, ex)
    full = db.full_device(m.DevicePanel.from_words(q, L)).cpu().numpy().view(np.uint32)
    assert np.array_equal(full, exp)
    rp = m.Panel(tuple(range(r.shape[0])), r, L)
    qp = m.Panel(tuple(range(q.shape[0])), q, L)
    res = m.topk_streamed(rp, qp, 16, chunk_rows=5000, op=op)
    assert np.array_equal(res.scores, es) and np.array_equal(res.index, ex)


def test_operator_image_mismatch_raises(rng):
    m = fb()
    from paper_1707_00516_b200.search import KnownDatabase

    r, q = _case(rng, 500, 10, 1024)
    db = KnownDatabase(r, 1024, op="xor")
    dq = m.DevicePanel.from_words(q, 1024)
    with pytest.raises(ValueError):
        m.compare_device(db.panel, dq, image=db.image, op="and")
    with pytest.raises(ValueError):
        m.topk(m.Panel(tuple(range(500)), r, 1024), m.Panel(tuple(range(10)), q, 1024), 4, op="nand")


@pytest.mark.parametrize("form", ["tensor_f4", "tensor_i8"])
def test_db_set_operator_switches_a_prepared_image(rng, form):
    """fastid_db_set_operator on a live handle: the same image serves AND-NOT, XOR
    (the i8 image computes and caches its known-row popcounts on first use) and
    AND, call after call."""
    m = fb()
    from paper_1707_00516_b200 import _native
    from paper_1707_00516_b200.search import KnownDatabase

    L = 1024
    r, q = _case(rng, 7000, 300, L)
    db = KnownDatabase(r, L, formulation=form)
    db.packed_max_queries = db.scan_max_queries = 0  # keep every batch on the image
    for i, op in enumerate(("andnot", "xor", "and", "xor", "andnot")):
        if i % 2:  # the C ABI directly, and through KnownDatabase.set_operator
            _native.check(_native.lib().fastid_db_set_operator(db.image.handle, _native.OPERATORS[op]),
                          "fastid_db_set_operator")
            db.op = db.image.op = op
        else:
            db.set_operator(op)
        exp = oracle.np_scores_op(r, q, op)
        s, x = db.search_words(q, 16)
        es, ex, _ = oracle.topk_from_matrix(exp, 16)
        assert np.array_equal(s, es) and np.array_equal(x, ex), op
        full = db.full_device(m.DevicePanel.from_words(q, L)).cpu().numpy().view(np.uint32)
        assert np.array_equal(full, exp), op


@pytest.mark.parametrize("form", ["tensor_f4", "tensor_i8", "popc"])
def test_operators_longest_profiles_exact(rng, form):
    """L = 2^20 loci with AND and XOR: an all-ones known against an all-zero /
    all-one unknown scores 2^20 / 0 (XOR) and 0 / 2^20 (AND); XOR's signed mxf4
    accumulator spans [-2^20, 2^20] and stays exact in fp32."""
    m = fb()
    from paper_1707_00516_b200.search import KnownDatabase

    L = 1 << 20
    nw = L // 64
    r, _ = rand_words(rng, 24, nw, 64, L)
    q, _ = rand_words(rng, 5, nw, 64, L)
    r[0] = np.uint64(2**64 - 1)
    r[1] = 0
    q[0] = 0
    q[1] = np.uint64(2**64 - 1)
    q[2] = r[3]
    R, Q = m.Panel(tuple(range(24)), r, L), m.Panel(tuple(range(5)), q, L)
    for op in ("and", "xor"):
        exp = oracle.np_scores_op(r, q, op, block=4)
        if op == "xor":
            assert exp[0, 0] == L and exp[0, 1] == 0 and exp[1, 1] == L and exp[3, 2] == 0
        else:
            assert exp[0, 1] == L and exp[0, 0] == 0
        assert np.array_equal(m.compare_b200(R, Q, formulation=form, op=op).scores, exp), (op, "packed full")
        es, ex, _ = oracle.topk_from_matrix(exp, 4)
        res = m.topk(R, Q, 4, formulation=form, op=op)
        assert np.array_equal(res.scores, es) and np.array_equal(res.index, ex), (op, "packed top-k")
        db = KnownDatabase(r, L, formulation=form, op=op)
        full = db.full_device(m.DevicePanel.from_words(q, L)).cpu().numpy().view(np.uint32)
        assert np.array_equal(full, exp), (op, "image full")
        s, x = db.search_words(q, 4)
        assert np.array_equal(s, es) and np.array_equal(x, ex), (op, "image top-k")
