"""Multi-GPU driver: the known database sharded over ranks, unknowns replicated.

One process per GPU (torch.distributed).  Rank g owns the contiguous known
rows [g*N/G, (g+1)*N/G) -- the same contiguous-range partition the reference
uses for its batches (plan_batches, scheduler.py:108-140) -- and reports
global indices (ref_base = first owned row).  Every (known, unknown) pair is
independent, so the only exchange is the final one the north star names: an
all-gather of each rank's fixed-size top-k candidate lists (N_Q x k x
(4 + 8) bytes per rank, NCCL over NVLink), followed by the same
(score, index) merge kernel the single-GPU path uses.  Threshold hits add a
count exchange, then a gather padded to the largest count
(``gather_hits`` / ``ShardedDatabase.threshold``); the union is ordered by
(unknown, known) like the single-GPU result.

No reference implementation exists for this layer (
PAPER.md:197 lists multi-GPU as future work).
"""

from __future__ import annotations

from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from . import _native

__all__ = ["shard_range", "gather_candidates", "merge_candidates", "gather_hits", "ShardedDatabase"]


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous rows [start, stop) owned by `rank` of `world` (balanced to +-1 row)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if n_total < 0:
        raise ValueError("n_total must be non-negative")
    return n_total * rank // world, n_total * (rank + 1) // world


def gather_candidates(scores: torch.Tensor, index: torch.Tensor, group=None):
    """All-gather fixed-size candidate lists -> ([world, N_Q, k] scores, [world, N_Q, k] index).

    One collective per step: each rank's (score, index) pairs travel as one
    [N_Q, k, 2] int64 block (the u32 score zero-extended), so the exchange costs
    one NCCL launch rather than one per array.
    """
    world = dist.get_world_size(group)
    packed = torch.stack((scores.to(torch.int64) & 0xFFFFFFFF, index.to(torch.int64)), dim=-1)
    p_all = torch.empty((world, *packed.shape), dtype=packed.dtype, device=packed.device)
    if packed.is_cuda and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(p_all, packed, group=group)
    else:
        dist.all_gather(list(p_all.unbind(0)), packed, group=group)
    s_all = p_all[..., 0].to(torch.int32)  # wraps back to the u32 bit pattern
    x_all = p_all[..., 1].contiguous()
    return s_all.to(scores.dtype), x_all.to(index.dtype)


def gather_hits(query: np.ndarray, ref: np.ndarray, score: np.ndarray, group=None, device=None):
    """Variable-size gather of every rank's threshold hits -> the union on every rank,
    ordered by (unknown, known index).

    Step 1 all-gathers the per-rank hit counts; step 2 all-gathers the hit
    triples padded to the largest count (fixed-size collectives, so NCCL's
    all_gather_into_tensor applies); the padding is dropped on receipt.  Rows are
    disjoint between ranks, so no (unknown, known) pair appears twice.
    ``device`` holds the collective buffers (a CUDA device for NCCL, None = CPU).
    """
    world = dist.get_world_size(group)
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device(device) if device is not None else torch.device("cpu")
    n = int(query.shape[0])
    counts = torch.zeros((world, 1), dtype=torch.int64, device=dev)
    mine = torch.tensor([n], dtype=torch.int64, device=dev)
    if nccl:
        dist.all_gather_into_tensor(counts, mine, group=group)
    else:
        dist.all_gather(list(counts.unbind(0)), mine, group=group)
    counts = counts.cpu().numpy()[:, 0]
    m = int(counts.max()) if world else 0
    if m == 0:
        return (np.zeros(0, np.uint32), np.zeros(0, np.int64), np.zeros(0, np.uint32))
    # one (m, 3) int64 block per rank: unknown, known, score
    block = torch.full((m, 3), -1, dtype=torch.int64, device=dev)
    if n:
        block[:n, 0] = torch.from_numpy(query.astype(np.int64))
        block[:n, 1] = torch.from_numpy(ref.astype(np.int64))
        block[:n, 2] = torch.from_numpy(score.astype(np.int64))
    every = torch.empty((world, m, 3), dtype=torch.int64, device=dev)
    if nccl:
        dist.all_gather_into_tensor(every, block, group=group)
    else:
        dist.all_gather(list(every.unbind(0)), block, group=group)
    every = every.cpu().numpy()
    rows = np.concatenate([every[r, : counts[r]] for r in range(world)])
    order = np.lexsort((rows[:, 1], rows[:, 0]))
    rows = rows[order]
    return rows[:, 0].astype(np.uint32), rows[:, 1].astype(np.int64), rows[:, 2].astype(np.uint32)


def merge_candidates(s_all: torch.Tensor, x_all: torch.Tensor, k: int, out=None):
    """Device merge of [lists, N_Q, k_in] sorted candidate lists into the first k per query."""
    n_lists, n_q, k_in = s_all.shape
    if out is None:
        out = (torch.empty((n_q, k), dtype=torch.int32, device=s_all.device),
               torch.empty((n_q, k), dtype=torch.int64, device=s_all.device))
    s, x = out
    if n_q:
        with torch.cuda.device(s_all.device):
            _native.check(_native.lib().fastid_merge_topk(
                s_all.data_ptr(), x_all.data_ptr(), n_lists, n_q, k_in, k, s.data_ptr(), x.data_ptr(),
                torch.cuda.current_stream(s_all.device).cuda_stream), "fastid_merge_topk")
    return s, x


class ShardedDatabase:
    """This rank's shard of a known database plus the cross-rank combine.

    ``local`` is a KnownDatabase (or anything with ``topk_device`` /
    ``search_words``-compatible behaviour) whose ``ref_base`` is the shard's
    first global row.  ``merge`` defaults to the device merge kernel; it is
    injectable so the host-side protocol can be exercised with gloo on CPU.
    """

    def __init__(self, local, n_total: int, group=None, merge: Callable | None = None):
        self.local = local
        self.n_total = int(n_total)
        self.group = group
        self.merge = merge or merge_candidates

    @property
    def world(self) -> int:
        return dist.get_world_size(self.group) if dist.is_initialized() else 1

    def combine(self, s: torch.Tensor, x: torch.Tensor, k: int):
        """Local candidate lists -> global top-k on every rank (one all-gather + merge)."""
        if self.world == 1:
            return s, x
        s_all, x_all = gather_candidates(s, x, self.group)
        return self.merge(s_all, x_all, k)

    def threshold(self, queries, threshold: int, capacity: int | None = None):
        """Every (unknown j, global known i, score) with score <= threshold over the
        whole sharded database, ordered by (j, i), on every rank: the local
        threshold epilogue, then gather_hits."""
        from .panel import ThresholdHits

        hits = self.local.threshold(queries, threshold, capacity)
        if self.world == 1:
            return hits
        dev = getattr(self.local, "device", None)
        if dev is not None and dist.get_backend(self.group) != "nccl":
            dev = None
        q, r, sc = gather_hits(hits.query, hits.ref, hits.score, self.group, dev)
        return ThresholdHits(q, r, sc, int(threshold))

    def topk_device(self, queries, k: int, max_score: int | None = None, workspace=None, out=None):
        s, x = self.local.topk_device(queries, k, max_score, workspace, out)
        return self.combine(s, x, k)

    def search_many(self, batches, k: int = 16, max_score: int | None = None):
        """Pipelined global top-k over a sequence of host query batches (every rank
        passes the same batches): KnownDatabase.search_many with the cross-rank
        gather + merge on the device before each read-back."""
        return self.local.search_many(batches, k, max_score, combine=self.combine)

    def search_words(self, query_words: np.ndarray, k: int = 16, max_score: int | None = None):
        """Host unknowns -> global top-k (host arrays) on every rank."""
        db = self.local
        st = db.stage_queries(query_words, k)
        with torch.cuda.device(db.device):
            s, x = self.topk_device(st.panel, k, max_score, st.workspace, (st.out_s, st.out_x))
        return db.fetch_lists(st, s, x)
