"""Multi-process (world_size 2, gloo on CPU) tests of the sharded query
path's host logic (no GPU here):

* the NCCL id exchange of a one-process-per-GPU fclsh_cluster
  (cluster.exchange_cluster_id: rank 0's ncclGetUniqueId reaches every rank);
* the invariants the library's merge (k_merge_sources) relies on -- shard
  ranges, id offsets, shard-additive counters, rank order = id order --
  checked by answering each rank's shard with the CPU oracle and exchanging
  through torch.distributed (cluster.exchange).
The device path itself (fclsh_cluster, 1-8 shards, NCCL forced on at one
rank) is tests/test_cluster_gpu.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from tests.helpers import planted_queries, random_rows

M31 = (1 << 31) - 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dataset():
    rng = np.random.default_rng(77)
    rows = random_rows(rng, 2500, 128)
    q = planted_queries(rng, rows, 128, 60, 6)
    return rows, q


def _worker(rank, world, port, outdir):
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1602_02620_b200 import cluster
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    rows, q = _dataset()
    b, e = cluster.shard_range(rows.shape[0], world, rank)
    orc = O.port()
    ix = orc.index_build(rows[b:e], 128, 4, 11, 22, override=(0, 1), prime=M31)
    counters, offsets, ids = ix.query(q, 4)
    nq = q.shape[0]
    qcol = np.repeat(np.arange(nq), np.diff(offsets).astype(np.int64))
    full = rows[b:e][ids] if ids.size else np.zeros((0, rows.shape[1]), np.uint64)
    qrows = q[qcol] if ids.size else np.zeros((0, rows.shape[1]), np.uint64)
    dists = np.unpackbits((full ^ qrows).view(np.uint8), axis=1).sum(1) if ids.size else np.zeros(0, np.int64)
    trip = torch.tensor(np.stack([qcol, ids.astype(np.int64) + b, dists]).astype(np.int32)) if ids.size \
        else torch.zeros((3, 1), dtype=torch.int32)
    off = torch.tensor(offsets.astype(np.int64))
    cnt = torch.tensor(counters.T.astype(np.int64).copy())
    ex = cluster.exchange(trip, int(ids.size), off, cnt)
    if rank == 0:
        np.savez(os.path.join(outdir, "ex.npz"), totals=np.array(ex.totals), offsets=ex.offsets.numpy(),
                 triples=ex.triples.numpy(), counters=ex.counters.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _id_worker(rank, world, port, outdir):
    import torch.distributed as dist

    from paper_1602_02620_b200 import cluster
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    uid = cluster.exchange_cluster_id()
    with open(os.path.join(outdir, f"id{rank}.bin"), "wb") as f:
        f.write(uid)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_cluster_id_exchange(tmp_path):
    world = 2
    mp.start_processes(_id_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    ids = [open(os.path.join(tmp_path, f"id{r}.bin"), "rb").read() for r in range(world)]
    assert len(ids[0]) == 128 and ids[0] == ids[1] and any(ids[0])


def test_shard_range_partitions():
    from paper_1602_02620_b200.cluster import shard_range
    for n in (1, 7, 100, 1_000_003):
        for world in (1, 2, 3, 8):
            rs = [shard_range(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert max(e - b for b, e in rs) - min(e - b for b, e in rs) <= 1


def test_two_rank_exchange_equals_single_index(tmp_path):
    world = 2
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True, start_method="spawn")
    ex = np.load(os.path.join(tmp_path, "ex.npz"))
    from oracle import oracle as O
    rows, q = _dataset()
    counters, offsets, ids = O.port().index_build(rows, 128, 4, 11, 22, override=(0, 1), prime=M31).query(q, 4)
    # counters are shard-additive
    assert (ex["counters"].T == counters.astype(np.int64)).all()
    # per query, rank 0's run then rank 1's run == the global ascending id list
    nq = q.shape[0]
    merged = []
    for qi in range(nq):
        for r in range(world):
            o = ex["offsets"][r]
            merged.extend(ex["triples"][r, 1, o[qi]:o[qi + 1]].tolist())
    assert merged == ids.astype(np.int64).tolist()
    assert int(ex["totals"].sum()) == ids.size
