"""Multi-GPU sharded fcLSH: one process per GPU.

Points are sharded across ranks in contiguous id ranges (rank r owns ids
[begin_r, end_r) and builds its own tables over them with the same families
-- families depend only on (d, r, seed), index.cpp:83-88); the query batch is
broadcast from rank 0; every rank answers it against its shard
(query_r_nn over the shard, ids offset by begin_r); rank 0 receives every
rank's (query, id, distance) runs and per-query offsets and the per-query
counters are summed:

* counters are exactly additive across shards -- every posting and every
  id lives in exactly one shard -- so one all-reduce gives the reference's
  single-index collisions / candidates / found;
* shard id ranges increase with the rank, so per query "rank 0's ids, then
  rank 1's, ..." is already the global ascending id order; the device merge
  (fclsh_merge_shards) places every run without a sort.

The exchange (`exchange`) is backend-agnostic torch.distributed (NCCL over
NVLink on GPUs; gloo on CPU for the multi-process tests); the merge and the
per-shard query are the library's CUDA kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import fclsh as F


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced id range of `rank` (the first n % world ranks get one more)."""
    base, rem = divmod(n, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


@dataclass
class Exchanged:
    """Every rank's results, as seen on the destination rank."""
    totals: list           # per-rank triple counts
    offsets: torch.Tensor  # int64 [world, nq+1]
    triples: torch.Tensor  # int32 [world, 3, cap]
    counters: torch.Tensor # int64 [3, nq], summed over ranks


def exchange(triples: torch.Tensor, total: int, offsets: torch.Tensor, counters: torch.Tensor,
             group=None) -> Exchanged:
    """All-gather every rank's triples ([3, >= total] int32, first `total`
    columns valid) and offsets ([nq+1] int64), and all-reduce the counters
    ([3, nq] int64). Triples are padded to the largest total so every rank
    contributes one equally shaped tensor."""
    world = dist.get_world_size(group)
    dev = triples.device
    t = torch.tensor([total], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(sizes, t, group=group)
    totals = [int(s.item()) for s in sizes]
    cap = max(1, max(totals))
    padded = torch.zeros((3, cap), dtype=torch.int32, device=dev)
    if total:
        padded[:, :total] = triples[:, :total]
    trips = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(trips, padded, group=group)
    offs = [torch.empty_like(offsets) for _ in range(world)]
    dist.all_gather(offs, offsets.contiguous(), group=group)
    all_trip = torch.stack(trips)
    all_off = torch.stack(offs)
    summed = counters.clone()
    dist.all_reduce(summed, op=dist.ReduceOp.SUM, group=group)
    return Exchanged(totals, all_off, all_trip, summed)


class ShardedQueryGather:
    """Per-step gather of a shard's device results to a merged device result.

    Used by bench.py under torchrun: after `ix.query_device(...)` on every
    rank, `gather(r)` exchanges over NCCL and (on every rank) merges with the
    device kernel; returns (triples [3, total], offsets [nq+1], counters [3, nq])."""

    def __init__(self, rank: int, world: int, device: torch.device):
        self.rank, self.world, self.device = rank, world, device

    def gather(self, r: F.DeviceQueryResults, stream=None):
        dev = self.device
        nq = r.nq
        trip = torch.empty((3, max(1, r.total)), dtype=torch.int32, device=dev)
        off = torch.empty(nq + 1, dtype=torch.int64, device=dev)
        cnt = torch.empty((3, nq), dtype=torch.int64, device=dev)
        r.copy_to(trip, off, cnt, device=dev.index or 0, stream=stream)
        ex = exchange(trip, r.total, off, cnt)
        total = sum(ex.totals)
        out = torch.empty((3, max(1, total)), dtype=torch.int32, device=dev)
        out_off = torch.empty(nq + 1, dtype=torch.int64, device=dev)
        F.merge_shards(ex.offsets, ex.triples, out, out_off, device=dev.index or 0, stream=stream)
        return out[:, :total], out_off, ex.counters


def broadcast_queries(q: torch.Tensor, src: int = 0) -> torch.Tensor:
    """The query batch travels from `src` to every rank."""
    dist.broadcast(q, src=src)
    return q
