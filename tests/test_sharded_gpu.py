"""The sharded driver with the real device kernels: world size 2, both ranks on
cuda:0, candidates all-gathered over gloo (a one-GPU box has no second device
for NCCL; the NCCL path differs only in the transport).  Each rank's
KnownDatabase (prepared image, CTA-pair kernel) searches its contiguous shard
with global indices; the gathered-and-merged top-k must equal the oracle's
top-k over the whole panel on every rank, including cross-shard ties, and the
gathered threshold hits must equal the oracle's hit list."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, refs, queries, L, k, result_q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1707_00516_b200.search import KnownDatabase
    from paper_1707_00516_b200.sharded import ShardedDatabase, shard_range

    start, stop = shard_range(len(refs), rank, world)
    db = ShardedDatabase(KnownDatabase(refs[start:stop], L, ref_base=start, formulation="tensor_f4"), len(refs))
    s, x = db.search_words(queries, k)
    from paper_1707_00516_b200.panel import Panel

    hits = db.threshold(Panel(tuple(range(len(queries))), queries, L), L // 8)
    # the pipelined serving loop over three batches (global lists per batch)
    many = list(db.search_many([queries, queries[::-1].copy(), queries], k))
    result_q.put((rank, s, x, hits.query, hits.ref, hits.score, many))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_two_ranks_real_kernels(rng):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    from conftest import rand_words

    L, n_r, n_q, k = 1024, 6001, 300, 16
    refs, _ = rand_words(rng, n_r, L // 64, 64, L)
    queries, _ = rand_words(rng, n_q, L // 64, 64, L)
    refs[n_r // 2 + 5] = refs[7]          # identical knowns on both shards: a cross-shard tie
    queries[:50] = refs[rng.integers(0, n_r, 50)]
    queries[50] = refs[7]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, refs, queries, L, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    es, ex, _ = oracle.topk(refs, queries, k)
    hq, hr, hs, _ = oracle.threshold(refs, queries, L // 8)
    assert len(hq) >= 52
    for rank, s, x, tq, tr, ts, many in out:
        assert np.array_equal(s, es) and np.array_equal(x, ex), rank
        assert len(many) == 3
        for (ms, mx), (e_s, e_x) in zip(many, ((es, ex), (es[::-1], ex[::-1]), (es, ex))):
            assert np.array_equal(ms, e_s) and np.array_equal(mx, e_x), rank
        # threshold hits of both shards: count exchange + padded gather, (j, i) order
        assert np.array_equal(tq, hq) and np.array_equal(tr, hr) and np.array_equal(ts, hs), rank
    assert 7 in ex[50] and n_r // 2 + 5 in ex[50]
