"""Sharded path on one GPU: S shard indexes (contiguous id ranges with
id_offset), their device results copied out (fclsh_result_copy_device) and
merged by the device kernel (fclsh_merge_shards) must equal one index over
all points -- triples in (query, id) order, offsets, and the summed
counters. (The NCCL exchange between these steps is covered on CPU by
tests/test_cluster_gloo.py; this box has one GPU.)"""
import numpy as np
import pytest
import torch

from paper_1602_02620_b200 import cluster
from paper_1602_02620_b200 import fclsh as F
from tests.helpers import planted_queries

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shards", [1, 2, 3, 8])
def test_merge_shards_equals_single_index(shards):
    rng = np.random.default_rng(shards)
    n, d, r = 6000, 256, 8
    rows = F.gen_clustered(shards, 40, n, d, 0.01)  # dense neighbourhoods: many results per query
    q = planted_queries(rng, rows, d, 200, 10)
    plan = F.make_plan(d, r, 1.0, n, 5, F.PlanOverride(F.PlanKind.partition, 2))
    full = F.build_index(rows, r, plan, 6, prime=F.M31).query_r_nn(q, r)
    dev = torch.device("cuda:0")
    qd = torch.from_numpy(q.view(np.int64)).to(dev)
    trips, offs, cnts = [], [], []
    idx = []
    for s in range(shards):
        b, e = cluster.shard_range(n, shards, s)
        ix = F.build_index(rows[b:e], r, plan, 6, prime=F.M31, id_offset=b)
        idx.append(ix)
        res = ix.query_device(qd, r)
        t = torch.zeros((3, max(1, res.total)), dtype=torch.int32, device=dev)
        o = torch.zeros(q.shape[0] + 1, dtype=torch.int64, device=dev)
        c = torch.zeros((3, q.shape[0]), dtype=torch.int64, device=dev)
        res.copy_to(t, o, c)
        torch.cuda.synchronize()
        trips.append(t[:, :res.total])
        offs.append(o)
        cnts.append(c)
    cap = max(1, max(t.shape[1] for t in trips))
    all_t = torch.zeros((shards, 3, cap), dtype=torch.int32, device=dev)
    for s, t in enumerate(trips):
        all_t[s, :, :t.shape[1]] = t
    all_o = torch.stack(offs)
    total = sum(t.shape[1] for t in trips)
    out = torch.zeros((3, max(1, total)), dtype=torch.int32, device=dev)
    out_off = torch.zeros(q.shape[0] + 1, dtype=torch.int64, device=dev)
    F.merge_shards(all_o, all_t, out, out_off)
    torch.cuda.synchronize()
    got = out[:, :total].cpu().numpy().T.astype(np.uint32)
    assert (got == full.triples()).all()
    assert (out_off.cpu().numpy() == full.offsets.astype(np.int64)).all()
    summed = torch.stack(cnts).sum(0).cpu().numpy()
    assert (summed[0] == full.collisions).all() and (summed[1] == full.candidates).all()
    assert (summed[2] == full.found).all()
    assert full.found.sum() > 200


# --------------------------------------------------------------- fclsh_cluster

def _cluster_case(seed=3, n=9000, d=256, r=8, nq=300):
    rng = np.random.default_rng(seed)
    rows = F.gen_clustered(seed, 50, n, d, 0.01)
    q = planted_queries(rng, rows, d, nq, 10)
    plan = F.make_plan(d, r, 1.0, n, 5, F.PlanOverride(F.PlanKind.partition, 2))
    return rows, q, plan, r


def _same(res, full):
    assert res.triples().shape == full.triples().shape
    assert (res.triples() == full.triples()).all()
    assert (res.offsets == full.offsets).all()
    assert (res.collisions == full.collisions).all()
    assert (res.candidates == full.candidates).all()
    assert (res.found == full.found).all()


@pytest.mark.parametrize("shards", [1, 2, 3, 8])
def test_cluster_equals_single_index(shards):
    """fclsh_cluster with S shards on this one GPU (the multi-GPU layout,
    shards >= devices): host and device queries equal one index over all points."""
    rows, q, plan, r = _cluster_case(seed=shards)
    full = F.build_index(rows, r, plan, 6, prime=F.M31).query_r_nn(q, r)
    assert full.found.sum() > 300
    cl = F.Cluster([0], shards_per_rank=shards).build(rows, r, plan, 6, prime=F.M31)
    info = cl.info()
    assert info["total_shards"] == shards and info["local_points"] == rows.shape[0]
    assert info["local_entry_count"] == rows.shape[0] * plan.table_count()
    for _ in range(3):  # eager, captured, replayed batches
        _same(cl.query_r_nn(q, r), full)
    qd = torch.from_numpy(q.view(np.int64)).to("cuda:0")
    for _ in range(3):
        dres = cl.query_device(qd, r)
        t = torch.zeros((3, max(1, dres.total)), dtype=torch.int32, device="cuda:0")
        o = torch.zeros(q.shape[0] + 1, dtype=torch.int64, device="cuda:0")
        c = torch.zeros((3, q.shape[0]), dtype=torch.int64, device="cuda:0")
        dres.copy_to(t, o, c)
        torch.cuda.synchronize()
        assert dres.total == full.id.size
        assert (t[:, :dres.total].cpu().numpy().T.astype(np.uint32) == full.triples()).all()
        assert (o.cpu().numpy() == full.offsets.astype(np.int64)).all()
        cc = c.cpu().numpy()
        assert (cc[0] == full.collisions).all() and (cc[1] == full.candidates).all() and (cc[2] == full.found).all()


def test_cluster_smaller_radius_empty_batch_and_offset():
    rows, q, plan, r = _cluster_case(seed=11, n=5000, nq=120)
    ix = F.build_index(rows, r, plan, 6, prime=F.M31, id_offset=1000)
    cl = F.Cluster([0], shards_per_rank=4).build(rows, r, plan, 6, prime=F.M31, id_offset=1000)
    for rad in (r, 5, 0):
        _same(cl.query_r_nn(q, rad), ix.query_r_nn(q, rad))
    empty = cl.query_r_nn(np.zeros((0, q.shape[1]), np.uint64), r)
    assert empty.id.size == 0 and empty.offsets.tolist() == [0]


def test_cluster_rank_mode_world1_and_device_rows():
    """fclsh_cluster_create_rank with world 1 (the torchrun path at N = 1) and rows
    already on the device."""
    rows, q, plan, r = _cluster_case(seed=21, n=6000, nq=150)
    full = F.build_index(rows, r, plan, 6, prime=F.M31).query_r_nn(q, r)
    drows = torch.from_numpy(rows.view(np.int64)).to("cuda:0")
    cl = F.Cluster(rank=0, world=1, device=0, uid=bytes(128), shards_per_rank=2).build(drows, r, plan, 6,
                                                                                      prime=F.M31)
    _same(cl.query_r_nn(q, r), full)


def test_cluster_nccl_single_rank(monkeypatch):
    """The NCCL plumbing (dlopen, ncclCommInitAll, the in-place ncclBroadcast of
    every batch) forced on at one rank."""
    monkeypatch.setenv("FCLSH_CLUSTER_NCCL", "1")
    rows, q, plan, r = _cluster_case(seed=31, n=4000, nq=100)
    full = F.build_index(rows, r, plan, 6, prime=F.M31).query_r_nn(q, r)
    cl = F.Cluster([0], shards_per_rank=2).build(rows, r, plan, 6, prime=F.M31)
    assert cl.info()["uses_nccl"] == 1
    for _ in range(2):
        _same(cl.query_r_nn(q, r), full)


def test_cluster_errors():
    rows, q, plan, r = _cluster_case(seed=41, n=200, nq=5)
    with pytest.raises(F.UsageError, match="appear once"):
        F.Cluster([0, 0])
    with pytest.raises(F.UsageError, match="64 shards"):
        F.Cluster([0], shards_per_rank=65)
    with pytest.raises(F.UsageError, match="does not exist"):
        F.Cluster([F.device_count()])
    cl = F.Cluster([0], shards_per_rank=2)
    with pytest.raises(F.UsageError, match="before build"):
        cl.query_r_nn(q, r)
    with pytest.raises(F.UsageError, match="fewer points than shards"):
        F.Cluster([0], shards_per_rank=8).build(rows[:5], r, plan, 6, prime=F.M31)
    cl.build(rows, r, plan, 6, prime=F.M31)
    with pytest.raises(F.UsageError, match="exceeds the index radius"):
        cl.query_r_nn(q, r + 1)
    with pytest.raises(F.UsageError, match="already built"):
        cl.build(rows, r, plan, 6, prime=F.M31)
