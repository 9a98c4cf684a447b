"""The five BASELINE configs on the GPU.

* Scaled configs 1-4 (same shapes, distributions, plans and P = 2^31-1, fewer
  points so the CPU reference finishes in seconds; cfg1 at its full size):
  ids and every QueryReport counter equal the compiled reference's
  query_r_nn, triples equal scan_truth.
* cfg5: keys of a sample of rows of the real 8M x 1024-bit workload equal
  hash_batch_into, bit for bit (every key: test_cfg5_every_key, -m slow).
* Full-size configs 2-4 through size-independent properties: every planted
  query (k <= r flips) finds its source row, and for a random sample of
  queries the result set equals a CPU linear scan over all n points.
  cfg4 runs sharded 8 ways exactly as on 8 GPUs (shard indexes with id
  offsets, device merge), one shard at a time on this single GPU.
"""
import numpy as np
import pytest
import torch

from paper_1602_02620_b200 import cluster
from paper_1602_02620_b200 import fclsh as F
from paper_1602_02620_b200.configs import CONFIGS, make_data, make_queries

pytestmark = pytest.mark.gpu

M31 = F.M31


def run_and_compare(oracle, cfg, threads=16):
    data = make_data(cfg)
    q = make_queries(cfg, data)
    plan = F.make_plan(cfg.dims, cfg.radius, 1.0, cfg.n, cfg.plan_seed(), cfg.override())
    ix = F.build_index(data, cfg.radius, plan, cfg.index_seed(), prime=M31)
    assert ix.table_count() == cfg.tables
    res = ix.query_r_nn(q, cfg.radius)
    oi = oracle.index_build(data, cfg.dims, cfg.radius, cfg.plan_seed(), cfg.index_seed(),
                            override=(int(cfg.plan_kind), cfg.t), prime=M31, threads=threads)
    counters, offsets, ids = oi.query(q, cfg.radius, threads=threads)
    got = np.stack([res.collisions, res.candidates, res.found], 1)
    bad = np.argwhere((got != counters).any(1)).ravel()
    assert bad.size == 0, f"{cfg.name}: counters differ at {bad[:5].tolist()}"
    assert (res.offsets == offsets).all() and (res.id == ids).all()
    truth = oracle.scan_truth(data, q, cfg.dims, cfg.radius, threads=threads)
    assert (res.triples() == truth).all()
    return res


def test_cfg1_full_size(oracle):
    res = run_and_compare(oracle, CONFIGS[1])
    assert res.found.min() >= 1  # every planted query (k <= 4 = r) finds its source


@pytest.mark.parametrize("cid,n,nq", [(2, 100_000, 400), (3, 200_000, 300), (4, 200_000, 300)])
def test_scaled_configs(oracle, cid, n, nq):
    cfg = CONFIGS[cid].scaled(n, nq)
    res = run_and_compare(oracle, cfg)
    if cfg.data == "bernoulli":
        assert res.found.min() >= 1


def test_cfg5_sample_keys(oracle):
    cfg = CONFIGS[5]
    rows = F.gen_bernoulli(cfg.root(), cfg.n, cfg.dims)
    fam = F.build_covering_family(cfg.dims, cfg.radius, cfg.index_seed(), prime=M31)
    m, s, k = oracle.build_family(cfg.dims, cfg.radius, cfg.index_seed(), prime=M31)
    assert (fam.mapping == m).all() and (fam.seeds == s).all()
    rng = np.random.default_rng(5)
    pick = np.sort(rng.choice(cfg.n, 4096, replace=False))
    L = fam.table_count()
    d = torch.from_numpy(rows.view(np.int64)).cuda()
    keys = torch.empty((1_000_000, L), dtype=torch.int32, device="cuda")
    for c0 in range(0, cfg.n, 1_000_000):
        F.hash_batch_device(fam, d[c0:c0 + 1_000_000], keys, layout=1, key_stride=L)
        torch.cuda.synchronize()
        sel = pick[(pick >= c0) & (pick < c0 + 1_000_000)]
        got = keys[torch.from_numpy(sel - c0).cuda()].cpu().numpy().astype(np.uint64)
        want = oracle.hash_batch(m, s, cfg.dims, cfg.radius, M31, rows[sel], kind=k, threads=16)
        assert (got == want).all(), f"chunk {c0}"


@pytest.mark.slow
def test_cfg5_every_key(oracle):
    """BASELINE cfg5: every one of the 8M x 2047 keys compared bit-exactly."""
    cfg = CONFIGS[5]
    rows = F.gen_bernoulli(cfg.root(), cfg.n, cfg.dims)
    fam = F.build_covering_family(cfg.dims, cfg.radius, cfg.index_seed(), prime=M31)
    L = fam.table_count()
    d = torch.from_numpy(rows.view(np.int64)).cuda()
    keys = torch.empty((1_000_000, L), dtype=torch.int32, device="cuda")
    for c0 in range(0, cfg.n, 1_000_000):
        F.hash_batch_device(fam, d[c0:c0 + 1_000_000], keys, layout=1, key_stride=L)
        got = keys.cpu().numpy()
        for s0 in range(0, 1_000_000, 125_000):
            want = oracle.hash_batch(fam.mapping, fam.seeds, cfg.dims, cfg.radius, M31,
                                     rows[c0 + s0:c0 + s0 + 125_000], kind=int(fam.kind), threads=16)
            assert (got[s0:s0 + 125_000].astype(np.uint64) == want).all(), f"rows {c0 + s0}.."


def _sample_check(oracle, data, q, res_ids_of, dims, radius, sample, threads=16):
    truth = oracle.scan_truth(data, q[sample], dims, radius, threads=threads)
    for j, qi in enumerate(sample):
        want = truth[truth[:, 0] == j][:, 1]
        assert (res_ids_of(qi) == want).all(), f"query {qi}"


@pytest.mark.parametrize("cid", [2, 3])
def test_full_size_properties(oracle, cid):
    cfg = CONFIGS[cid]
    data = make_data(cfg)
    q = make_queries(cfg, data)
    plan = F.make_plan(cfg.dims, cfg.radius, 1.0, cfg.n, cfg.plan_seed(), cfg.override())
    ix = F.build_index(data, cfg.radius, plan, cfg.index_seed(), prime=M31)
    res = ix.query_r_nn(q, cfg.radius)
    assert res.found[:cfg.planted].min() >= 1  # planted queries find their source
    assert (res.collisions >= res.candidates).all() and (res.candidates >= res.found).all()
    assert (res.distance <= cfg.radius).all()
    sample = np.random.default_rng(cid).choice(q.shape[0], 120, replace=False)
    _sample_check(oracle, data, q, res.ids, cfg.dims, cfg.radius, sample)


def test_cfg4_full_size_sharded_8(oracle):
    """cfg4 as specified: 10M clustered points sharded across 8 ranks; each
    shard built and queried in turn on this GPU, results merged on device."""
    cfg = CONFIGS[4]
    data = make_data(cfg)
    q = make_queries(cfg, data)
    nq = q.shape[0]
    plan = F.make_plan(cfg.dims, cfg.radius, 1.0, cfg.n, cfg.plan_seed(), cfg.override())
    dev = torch.device("cuda:0")
    qd = torch.from_numpy(q.view(np.int64)).to(dev)
    world = cfg.shards
    trips, offs, cnt = [], [], torch.zeros((3, nq), dtype=torch.int64, device=dev)
    for r in range(world):
        b, e = cluster.shard_range(cfg.n, world, r)
        ix = F.build_index(data[b:e], cfg.radius, plan, cfg.index_seed(), prime=M31, id_offset=b)
        res = ix.query_device(qd, cfg.radius)
        t = torch.zeros((3, max(1, res.total)), dtype=torch.int32, device=dev)
        o = torch.zeros(nq + 1, dtype=torch.int64, device=dev)
        c = torch.zeros((3, nq), dtype=torch.int64, device=dev)
        res.copy_to(t, o, c)
        torch.cuda.synchronize()
        trips.append(t[:, :res.total].clone())
        offs.append(o)
        cnt += c
        del ix
    cap = max(1, max(t.shape[1] for t in trips))
    all_t = torch.zeros((world, 3, cap), dtype=torch.int32, device=dev)
    for r, t in enumerate(trips):
        all_t[r, :, :t.shape[1]] = t
    total = sum(t.shape[1] for t in trips)
    out = torch.zeros((3, max(1, total)), dtype=torch.int32, device=dev)
    out_off = torch.zeros(nq + 1, dtype=torch.int64, device=dev)
    F.merge_shards(torch.stack(offs), all_t, out, out_off)
    torch.cuda.synchronize()
    trip = out[:, :total].cpu().numpy()
    off = out_off.cpu().numpy()
    counters = cnt.cpu().numpy()
    assert (np.diff(off) == counters[2]).all()
    assert (counters[0] >= counters[1]).all() and (counters[1] >= counters[2]).all()
    assert (trip[2] <= cfg.radius).all()
    for qi in range(nq):  # ids ascending within every query
        ids = trip[1, off[qi]:off[qi + 1]]
        assert (np.diff(ids.astype(np.int64)) > 0).all()
    sample = np.random.default_rng(4).choice(nq, 60, replace=False)
    _sample_check(oracle, data, q, lambda qi: trip[1, off[qi]:off[qi + 1]].astype(np.uint32), cfg.dims,
                  cfg.radius, sample)
