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

The product path is the library's fclsh_cluster (C++ over NCCL,
csrc/cluster_host.cpp): `rank_cluster` forms one rank of it under torchrun,
F.Cluster(devices=[...]) drives several GPUs from one process. `exchange`
restates the same exchange in torch.distributed terms; the multi-process
gloo test (tests/test_cluster_gloo.py) checks on CPU the invariants the
library's merge relies on (shard-additive counters, rank order = id order).
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


def exchange_cluster_id(group=None) -> bytes:
    """Rank 0's NCCL unique id (ncclGetUniqueId, fclsh_cluster_unique_id) on
    every rank, carried by torch.distributed (any backend; gloo is enough).
    A world of one needs no id (the library skips NCCL there)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if world == 1:
        return bytes(F.CLUSTER_ID_BYTES)
    box = [F.cluster_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return box[0]


def rank_cluster(shards_per_rank: int = 1, device: int | None = None, group=None) -> F.Cluster:
    """One rank of a multi-process fclsh_cluster (one process per GPU, e.g.
    under torchrun): rank 0 draws the NCCL id, torch.distributed carries it to
    the other ranks, then every rank joins with ncclCommInitRank inside the
    library."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if device is None:
        device = torch.cuda.current_device()
    uid = exchange_cluster_id(group)
    return F.Cluster(rank=rank, world=world, device=device, uid=uid, shards_per_rank=shards_per_rank)
