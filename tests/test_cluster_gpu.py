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
