"""Multi-rank protocol of the sharded driver on CPU: world_size 2 over gloo.

Each rank owns a contiguous shard of the known panel (shard_range), computes
its local top-k with global indices, and ShardedDatabase.combine all-gathers
the fixed-size candidate lists and merges them.  The device kernels are
replaced by the oracle here (this is test infrastructure); the protocol under
test -- partition, index offsets, gather layout, merge order -- is the one the
NCCL path runs.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleShard:
    """Stands in for KnownDatabase on CPU: local top-k of this rank's rows."""

    def __init__(self, refs, start):
        self.refs = refs
        self.start = start

    def threshold(self, queries, t, capacity=None):
        import oracle
        from paper_1707_00516_b200.panel import ThresholdHits

        q, r, sc, _ = oracle.threshold(self.refs, queries, t)
        return ThresholdHits(q, r + self.start, sc, t)

    def topk_device(self, queries, k, max_score=None, workspace=None, out=None):
        import oracle

        s, x, _ = oracle.topk(self.refs, queries, k, 0xFFFFFFFE if max_score is None else max_score)
        x = np.where(x >= 0, x + self.start, -1)
        return torch.from_numpy(s.view(np.int32).copy()), torch.from_numpy(x)


def _host_merge(s_all, x_all, k):
    import oracle

    s, x = oracle.merge_lists(s_all.numpy().view(np.uint32), x_all.numpy(), k)
    return torch.from_numpy(s.view(np.int32).copy()), torch.from_numpy(x)


def _worker(rank, world, port, n_total, n_q, L, k, result_q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1707_00516_b200.sharded import ShardedDatabase, shard_range

    rng = np.random.default_rng(99)
    refs = rng.integers(0, 2**64, (n_total, L // 64), dtype=np.uint64)
    queries = refs[rng.integers(0, n_total, n_q)].copy()
    queries[:, 0] ^= np.uint64(1)
    refs[n_total // 2 + 1] = refs[3]  # a cross-shard tie
    start, stop = shard_range(n_total, rank, world)
    db = ShardedDatabase(OracleShard(refs[start:stop], start), n_total, merge=_host_merge)
    s, x = db.topk_device(queries, k)
    if rank == 0:
        es, ex, _ = oracle.topk(refs, queries, k)
        result_q.put((np.array_equal(s.numpy().view(np.uint32), es), np.array_equal(x.numpy(), ex)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_topk_matches_single_shard(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 1001, 37, 256, 8, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    ok_s, ok_x = q.get(timeout=5)
    assert ok_s and ok_x


def _threshold_worker(rank, world, port, n_total, n_q, L, result_q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1707_00516_b200.sharded import ShardedDatabase, shard_range

    rng = np.random.default_rng(7)
    refs = rng.integers(0, 2**64, (n_total, L // 64), dtype=np.uint64)
    # copies of rows of the first quarter only: at t = 0 the other ranks have no hits
    queries = refs[rng.integers(0, n_total // 4, n_q)].copy()
    queries[::3, 0] ^= np.uint64(0xFF)
    refs[n_total - 5] = refs[2]  # the same profile in the first and the last shard
    start, stop = shard_range(n_total, rank, world)
    db = ShardedDatabase(OracleShard(refs[start:stop], start), n_total)
    for t in (0, 8, L // 4, 0):
        hits = db.threshold(queries, t)
        if rank == 0:
            eq, er, es, _ = oracle.threshold(refs, queries, t)
            result_q.put((t, np.array_equal(hits.query, eq) and np.array_equal(hits.ref, er)
                          and np.array_equal(hits.score, es), len(hits)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_threshold_matches_single_shard(world):
    """Threshold hits of every rank: count all-gather, padded all-gather, (j, i)
    order -- equal to the single-shard oracle, including a threshold (t = 0) at
    which only the first rank has hits."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_threshold_worker, args=(r, world, port, 997, 29, 256, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    for _ in range(4):
        t, ok, n = q.get(timeout=5)
        assert ok, (t, n)


def test_merge_lists_oracle():
    import oracle

    rng = np.random.default_rng(3)
    full = rng.integers(0, 50, (300, 5)).astype(np.uint32)
    parts_s, parts_x = [], []
    for a, b in ((0, 100), (100, 220), (220, 300)):
        s, x, _ = oracle.topk_from_matrix(full[a:b], 6)
        parts_s.append(s)
        parts_x.append(np.where(x >= 0, x + a, -1))
    s, x = oracle.merge_lists(np.stack(parts_s), np.stack(parts_x), 6)
    es, ex, _ = oracle.topk_from_matrix(full, 6)
    assert np.array_equal(s, es) and np.array_equal(x, ex)
