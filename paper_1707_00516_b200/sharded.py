"""Multi-GPU driver: the known database sharded over ranks, unknowns replicated.

One process per GPU (torch.distributed).  Rank g owns the contiguous known
rows [g*N/G, (g+1)*N/G) -- the same contiguous-range partition the reference
uses for its batches (plan_batches, scheduler.py:108-140) -- and reports
global indices (ref_base = first owned row).  Every (known, unknown) pair is
independent, so the only exchange is the final one the north star names: an
all-gather of each rank's fixed-size top-k candidate lists (N_Q x k x
(4 + 8) bytes per rank, NCCL over NVLink), followed by the same
(score, index) merge kernel the single-GPU path uses.  Threshold hits add a
count exchange, then a variable-size gather.

No reference implementation exists for this layer (
PAPER.md:197 lists multi-GPU as future work).
"""

from __future__ import annotations

from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from . import _native

__all__ = ["shard_range", "gather_candidates", "merge_candidates", "ShardedDatabase"]


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous rows [start, stop) owned by `rank` of `world` (balanced to +-1 row)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if n_total < 0:
        raise ValueError("n_total must be non-negative")
    return n_total * rank // world, n_total * (rank + 1) // world


def gather_candidates(scores: torch.Tensor, index: torch.Tensor, group=None):
    """All-gather fixed-size candidate lists -> ([world, N_Q, k] scores, [world, N_Q, k] index)."""
    world = dist.get_world_size(group)
    s_all = torch.empty((world, *scores.shape), dtype=scores.dtype, device=scores.device)
    x_all = torch.empty((world, *index.shape), dtype=index.dtype, device=index.device)
    if scores.is_cuda and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(s_all, scores.contiguous(), group=group)
        dist.all_gather_into_tensor(x_all, index.contiguous(), group=group)
    else:
        dist.all_gather(list(s_all.unbind(0)), scores.contiguous(), group=group)
        dist.all_gather(list(x_all.unbind(0)), index.contiguous(), group=group)
    return s_all, x_all


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

    def topk_device(self, queries, k: int, max_score: int | None = None, workspace=None, out=None):
        s, x = self.local.topk_device(queries, k, max_score, workspace, out)
        return self.combine(s, x, k)

    def search_words(self, query_words: np.ndarray, k: int = 16, max_score: int | None = None):
        """Host unknowns -> global top-k (host arrays) on every rank."""
        db = self.local
        n_q = query_words.shape[0]
        st = db.stager(n_q, k)
        qw = np.ascontiguousarray(query_words)
        st.host_in.numpy()[:] = qw.view(np.uint8).reshape(n_q, -1)
        stream = torch.cuda.current_stream(db.device)
        with torch.cuda.device(db.device):
            st.dev_in.copy_(st.host_in, non_blocking=True)
            _native.check(_native.lib().fastid_load_words(
                st.dev_in.data_ptr(), n_q, st.dev_in.shape[1], st.panel.rows.data_ptr(), st.panel.stride,
                stream.cuda_stream), "fastid_load_words")
            s, x = self.topk_device(st.panel, k, max_score, st.workspace, (st.out_s, st.out_x))
            st.host_s.copy_(s, non_blocking=True)
            st.host_x.copy_(x, non_blocking=True)
            stream.synchronize()
        return st.host_s.numpy().view(np.uint32).copy(), st.host_x.numpy().copy()
