"""K2-K5 parity on the GPU: build_index + query_r_nn through the C-ABI must
return the oracle's ids and QueryReport counters (collisions, candidates,
found) for every query, and the (query, id, distance) triples of
scan_truth (workload.cpp:56-71)."""
import numpy as np
import pytest

from paper_1602_02620_b200 import fclsh as F
from tests.helpers import planted_queries, random_rows

pytestmark = pytest.mark.gpu

M31, M61 = F.M31, F.M61


LAYOUTS = ("buckets", "csr")


def check_against_oracle(oracle, rows, q, d, radius, override, prime, plan_seed=11, index_seed=22, qradius=None,
                         directory_bits=0, layouts=LAYOUTS):
    res = None
    for layout in layouts:
        res = _check_one(oracle, rows, q, d, radius, override, prime, plan_seed, index_seed, qradius, directory_bits,
                         layout)
    return res


def _check_one(oracle, rows, q, d, radius, override, prime, plan_seed, index_seed, qradius, directory_bits, layout):
    qradius = radius if qradius is None else qradius
    force = F.PlanOverride(F.PlanKind(override[0]), override[1])
    plan = F.make_plan(d, radius, 1.0, rows.shape[0], plan_seed, force)
    ix = F.build_index(rows, radius, plan, index_seed, prime=prime, directory_bits=directory_bits, layout=layout)
    assert ix.layout == layout
    assert ix.table_count() == plan.table_count()
    assert ix.entry_count() == plan.table_count() * rows.shape[0]
    res = ix.query_r_nn(q, qradius)
    oi = oracle.index_build(rows, d, radius, plan_seed, index_seed, override=override, prime=prime, threads=4)
    counters, offsets, ids = oi.query(q, qradius, threads=4)
    got_counters = np.stack([res.collisions, res.candidates, res.found], axis=1)
    bad = np.argwhere((got_counters != counters).any(1)).ravel()
    assert bad.size == 0, f"counter mismatch at queries {bad[:8].tolist()}: got {got_counters[bad[:3]].tolist()} " \
                          f"want {counters[bad[:3]].tolist()}"
    assert (res.offsets == offsets).all()
    assert (res.id == ids).all()
    truth = oracle.scan_truth(rows, q, d, qradius, threads=4)
    assert (res.triples() == truth).all()
    return res


@pytest.mark.parametrize("override,radius", [((0, 1), 3), ((0, 1), 4), ((2, 2), 8), ((1, 2), 3), ((2, 3), 9)])
def test_small_indexes_match_oracle(oracle, override, radius):
    rng = np.random.default_rng(radius * 10 + override[0])
    d = 128
    rows = random_rows(rng, 3000, d)
    q = planted_queries(rng, rows, d, 120, radius + 2)
    check_against_oracle(oracle, rows, q, d, radius, override, M31)


def test_query_radius_below_index_radius(oracle):
    rng = np.random.default_rng(3)
    rows = random_rows(rng, 2000, 64)
    q = planted_queries(rng, rows, 64, 50, 6)
    for qr in (0, 1, 3):
        check_against_oracle(oracle, rows, q, 64, 4, (0, 1), M31, qradius=qr)


def test_m61_and_small_prime_indexes(oracle):
    """Wide (key, id) entries for the reference's default field, and a prime
    so small that bucket merges are frequent (counter parity under merges)."""
    rng = np.random.default_rng(61)
    rows = random_rows(rng, 1500, 96)
    q = planted_queries(rng, rows, 96, 60, 5)
    check_against_oracle(oracle, rows, q, 96, 4, (0, 1), M61)
    check_against_oracle(oracle, rows, q, 96, 4, (2, 2), M61)
    check_against_oracle(oracle, rows, q, 96, 3, (0, 1), 101, layouts=("csr",))
    plan = F.make_plan(96, 3, 1.0, 1500, 11, F.PlanOverride(F.PlanKind.identity, 1))
    with pytest.raises(F.UsageError, match="bucket layout"):
        F.build_index(rows, 3, plan, 22, prime=101, layout="buckets")
    assert F.build_index(rows, 3, plan, 22, prime=101).layout == "csr"  # auto falls back


def test_clustered_data_long_cells(oracle):
    """Duplicate-heavy data: long buckets exercise the CTA-wide cell sort."""
    cl = F.gen_clustered(5, 20, 6000, 128, 0.02)
    cl[:500] = cl[0]  # 500 identical rows -> one bucket of >= 500 per table
    q = F.gen_clustered(5, 20, 6100, 128, 0.02)[6000:]
    q[:3] = cl[0]
    res = check_against_oracle(oracle, cl, q, 128, 6, (0, 1), M31)
    assert res.found.max() >= 500


def test_three_query_paths(oracle):
    """One batch that needs all three query kernels: warp per query (sparse),
    CTA per query (more than 32 results; more such queries than the
    persistent grid has CTAs) and the general sort path (more than 2048
    results)."""
    rng = np.random.default_rng(33)
    d, radius = 128, 6
    base = random_rows(rng, 700, d)
    rows = random_rows(rng, 34000, d)
    rows[:28000] = np.repeat(base, 40, axis=0)  # 700 values x 40 copies
    rows[28000:30110] = base[0]  # base[0]: 2150 copies, more results than the CTA kernel holds
    q = np.concatenate([base, random_rows(rng, 200, d), planted_queries(rng, rows[30110:], d, 100, radius)])
    for layout in LAYOUTS:
        force = F.PlanOverride(F.PlanKind.identity, 1)
        plan = F.make_plan(d, radius, 1.0, rows.shape[0], 11, force)
        ix = F.build_index(rows, radius, plan, 22, prime=M31, layout=layout)
        ix.query_r_nn(q, radius)
        paths = ix.path_counts()
        assert paths["dense"] >= 600 and paths["general"] >= 1, paths
    res = check_against_oracle(oracle, rows, q, d, radius, (0, 1), M31)
    assert res.found[0] >= 2150


def test_many_tables_cta_per_query(oracle):
    """More than 600 tables (cfg4 has 1022): every query takes the CTA kernel
    directly; duplicates push one query to the general path."""
    rng = np.random.default_rng(77)
    d, radius = 96, 9
    rows = random_rows(rng, 3000, d)
    rows[100:2300] = rows[0]  # 2201 copies: more results than the CTA kernel holds
    q = np.concatenate([rows[:1], planted_queries(rng, rows[2300:], d, 150, radius)])
    res = check_against_oracle(oracle, rows, q, d, radius, (0, 1), M31)
    assert res.found[0] >= 2201
    plan = F.make_plan(d, radius, 1.0, rows.shape[0], 11, F.PlanOverride(F.PlanKind.identity, 1))
    assert plan.table_count() > 600
    ix = F.build_index(rows, radius, plan, 22, prime=M31)
    ix.query_r_nn(q, radius)
    assert ix.path_counts() == {"dense": q.shape[0], "general": 1}


@pytest.mark.parametrize("layout", LAYOUTS)
def test_many_tables_clustered(oracle, layout):
    """cfg4's shape in small: > 600 tables over clustered rows, every query
    in the CTA kernel (CSR: the flattened probe phase). Most queries have tens
    to hundreds of distinct candidates and more than 32 results (the shared
    result region); queries near a 1500-point cluster read cells of ~1500
    entries."""
    d, radius = 96, 9
    rows = F.gen_clustered(9, 60, 6000, d, 0.04)
    tight = F.gen_clustered(10, 1, 1500, d, 0.01)
    rows[:1500] = tight
    q = np.concatenate([F.gen_clustered(9, 60, 6300, d, 0.04)[6000:], tight[:5]])
    res = _check_one(oracle, rows, q, d, radius, (0, 1), M31, 11, 22, None, 0, layout)
    assert (res.found > 32).sum() >= 20 and res.candidates.max() > 768
    plan = F.make_plan(d, radius, 1.0, rows.shape[0], 11, F.PlanOverride(F.PlanKind.identity, 1))
    ix = F.build_index(rows, radius, plan, 22, prime=M31, layout=layout)
    ix.query_r_nn(q, radius)
    # (buckets: the small CTA shape holds up to 1024 results, so the five
    # queries with ~1500 go on to the general path)
    assert ix.path_counts() == {"dense": q.shape[0], "general": 5 if layout == "buckets" else 0}


def _device_triples(r):
    import torch
    tri = torch.zeros((3, max(r.total, 1)), dtype=torch.int32, device="cuda")
    off = torch.zeros(r.nq + 1, dtype=torch.int64, device="cuda")
    cnt = torch.zeros((3, r.nq), dtype=torch.int64, device="cuda")
    r.copy_to(tri, off, cnt)
    torch.cuda.synchronize()
    return tri[:, :r.total].cpu().numpy(), off.cpu().numpy(), cnt.cpu().numpy()


def test_repeated_device_queries_replay_graph(oracle):
    """The second identical batch is captured into a CUDA graph and later ones
    replay it: results must equal the eager ones, follow new contents of the
    same query buffer, and stay ordered with the caller's side stream."""
    import torch
    rng = np.random.default_rng(5)
    rows = random_rows(rng, 4000, 128)
    qa = planted_queries(rng, rows, 128, 300, 5)
    qb = planted_queries(rng, rows, 128, 300, 5)
    plan = F.make_plan(128, 4, 1.0, 4000, 1, F.PlanOverride(F.PlanKind.identity, 1))
    ix = F.build_index(rows, 4, plan, 2, prime=M31)
    want_a, want_b = ix.query_r_nn(qa, 4), ix.query_r_nn(qb, 4)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        qd = torch.from_numpy(qa.view(np.int64)).cuda()
        for k in range(5):
            if k == 3:  # same buffer, new contents: the replayed graph must read them
                qd.copy_(torch.from_numpy(qb.view(np.int64)))
            want = want_b if k >= 3 else want_a
            tri, off, cnt = _device_triples(ix.query_device(qd, 4, side))
            assert (off == want.offsets.astype(np.int64)).all(), k
            assert (tri[1] == want.id.astype(np.int32)).all(), k
            assert (cnt[2] == want.found.astype(np.int64)).all(), k
            assert set(ix.stage_ms()) == set(F.IndexSet.STAGES)


def test_host_and_device_destinations_interleaved(oracle):
    """Batches with a host result block (fclsh_query) and device-only batches
    alternate, each shape run eagerly, captured and replayed, with the host
    blocks freed in between: the batch prologue rewrites the destination every
    batch and no kernel may act on a previous batch's (freed) block."""
    import torch
    rng = np.random.default_rng(15)
    rows = random_rows(rng, 5000, 128)
    plan = F.make_plan(128, 4, 1.0, 5000, 1, F.PlanOverride(F.PlanKind.identity, 1))
    ix = F.build_index(rows, 4, plan, 2, prime=M31)
    oi = oracle.index_build(rows, 128, 4, 1, 2, override=(0, 1), prime=M31, threads=4)
    for nq in (200, 333, 200, 1000, 333):
        q = planted_queries(rng, rows, 128, nq, 5)
        counters, offsets, ids = oi.query(q, 4, threads=4)
        qd = torch.from_numpy(q.view(np.int64)).cuda()
        for k in range(4):
            if k % 2 == 0:
                res = ix.query_r_nn(q, 4)  # host result block, freed when res is dropped
                assert (res.offsets == offsets).all() and (res.id == ids).all(), (nq, k)
                del res
            else:
                tri, off, cnt = _device_triples(ix.query_device(qd, 4))
                assert (off == offsets.astype(np.int64)).all(), (nq, k)
                assert (tri[1] == ids.astype(np.int32)).all(), (nq, k)
                assert (cnt.T == counters.astype(np.int64)).all(), (nq, k)


def test_directory_extremes(oracle):
    """A 2-cell directory (long scans) and a fine one give the same answers."""
    rng = np.random.default_rng(9)
    rows = random_rows(rng, 2500, 64)
    q = planted_queries(rng, rows, 64, 40, 4)
    for bits in (1, 4, 18):
        check_against_oracle(oracle, rows, q, 64, 3, (0, 1), M31, directory_bits=bits, layouts=("csr",))


def test_edge_queries(oracle):
    rng = np.random.default_rng(17)
    rows = random_rows(rng, 1000, 128)
    plan = F.make_plan(128, 4, 1.0, 1000, 1, F.PlanOverride(F.PlanKind.identity, 1))
    ix = F.build_index(rows, 4, plan, 2, prime=M31)
    empty = ix.query_r_nn(np.zeros((0, 2), np.uint64), 4)
    assert empty.id.size == 0 and empty.offsets.tolist() == [0]
    one = ix.query_r_nn(rows[5:6], 4)
    assert 5 in one.ids(0).tolist()
    with pytest.raises(F.UsageError, match="exceeds the index radius"):
        ix.query_r_nn(rows[:2], 5)
    with pytest.raises(F.UsageError, match="width"):
        ix.query_r_nn(np.zeros((2, 3), np.uint64), 4)
    with pytest.raises(F.UsageError, match="empty dataset"):
        F.build_index(np.zeros((0, 2), np.uint64), 4, plan, 2, prime=M31)
    with pytest.raises(F.UsageError, match="radius does not match"):
        F.build_index(rows, 3, plan, 2, prime=M31)
    with pytest.raises(F.ResourceError):
        F.build_index(rows, 4, plan, 2, prime=M31, table_budget=5)


def test_id_offset_shards_reassemble(oracle):
    """Two shards with id offsets return the single index's answer (counters add)."""
    rng = np.random.default_rng(21)
    rows = random_rows(rng, 4000, 128)
    q = planted_queries(rng, rows, 128, 80, 5)
    plan = F.make_plan(128, 4, 1.0, 4000, 1, F.PlanOverride(F.PlanKind.identity, 1))
    full = F.build_index(rows, 4, plan, 2, prime=M31).query_r_nn(q, 4)
    a = F.build_index(rows[:2500], 4, plan, 2, prime=M31).query_r_nn(q, 4)
    b = F.build_index(rows[2500:], 4, plan, 2, prime=M31, id_offset=2500).query_r_nn(q, 4)
    for k in ("collisions", "candidates", "found"):
        assert (getattr(a, k) + getattr(b, k) == getattr(full, k)).all()
    merged = []
    for qi in range(80):
        merged.extend(a.ids(qi).tolist() + b.ids(qi).tolist())
    assert merged == full.id.tolist()


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("override,radius,budget", [((0, 1), 4, None), ((2, 2), 8, None), ((0, 1), 5, 7),
                                                     ((0, 1), 5, 0), ((1, 2), 3, 40)])
def test_query_c_r_nn_matches_the_reference(layout, override, radius, budget):
    """Strategy 1 (index.cpp:190-235): budgeted walk in table order, closest
    point retrieved (ties: lowest id); duplicates make the budget bite."""
    from oracle import oracle as O
    if not O.reference_available():
        pytest.skip("compiled reference unavailable")
    ref = O.reference()
    rng = np.random.default_rng(radius * 7 + (budget or 0))
    d = 128
    rows = random_rows(rng, 3000, d)
    rows[10:60] = rows[5]  # a 51-copy cluster: long buckets cut by small budgets
    q = np.concatenate([rows[5:6], planted_queries(rng, rows, d, 100, radius + 2), random_rows(rng, 5, d)])
    force = F.PlanOverride(F.PlanKind(override[0]), override[1])
    plan = F.make_plan(d, radius, 1.0, rows.shape[0], 11, force)
    ix = F.build_index(rows, radius, plan, 22, prime=M31, layout=layout)
    counters, bid, bd = ix.query_c_r_nn(q, radius, budget)
    oi = ref.index_build(rows, d, radius, 11, 22, override=override, prime=M31, threads=4)
    want_c, want_b = oi.query_c(q, radius, budget, threads=4)
    assert (counters == want_c).all(), np.argwhere((counters != want_c).any(1))[:5].ravel()
    none = want_b[:, 0] == 0xFFFFFFFF
    assert (bid[none] == -1).all() and (bd[none] == -1).all()
    assert (bid[~none] == want_b[~none, 0]).all() and (bd[~none] == want_b[~none, 1]).all()


@pytest.mark.parametrize("env", [{"FCLSH_FILTER": "0"}, {"FCLSH_FILTER_BPK": "0.75"}, {"FCLSH_FILTER_BPK": "1"},
                                 {"FCLSH_FILTER_BPK": "8", "FCLSH_FILTER_MB": "512"}])
@pytest.mark.parametrize("prime", [M31, M61])
def test_key_filter_sizes_match_oracle(oracle, monkeypatch, env, prime):
    """The L2 key filter of the bucket tables (index.cu, filter_pass) only
    skips bucket reads of keys no posting has: off, near its smallest size
    (many false positives), default and oversized, with 32- and 61-bit keys
    (filter_shift 33 / 3), the ids and every counter equal the reference's.
    Uniform queries (no near neighbour) are mostly filter rejections."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(len(env) * 7 + prime % 13)
    d = 256
    rows = random_rows(rng, 5000, d)
    q = np.concatenate([planted_queries(rng, rows, d, 150, 8), random_rows(rng, 50, d)])
    check_against_oracle(oracle, rows, q, d, 8, (0, 1), prime, layouts=("buckets",))


@pytest.mark.parametrize("d,radius,override", [(256, 8, (0, 1)), (128, 4, (0, 1)), (512, 12, (2, 2))])
def test_pinned_rows_hashed_in_place(oracle, d, radius, override):
    """fclsh_query with rows in pinned host memory hashes them in place (the
    hash kernel reads them over PCIe and writes the device copy the verify
    reads; other hash kernels copy first): results and counters equal the
    pageable-rows call and the reference, batch after batch (graph replay)."""
    import torch
    rng = np.random.default_rng(d + radius)
    rows = random_rows(rng, 4000, d)
    q = planted_queries(rng, rows, d, 300, radius + 2)
    force = F.PlanOverride(F.PlanKind(override[0]), override[1])
    plan = F.make_plan(d, radius, 1.0, rows.shape[0], 11, force)
    ix = F.build_index(rows, radius, plan, 22, prime=M31)
    pinned = torch.from_numpy(q.view(np.int64)).pin_memory().numpy().view(np.uint64)
    want = ix.query_r_nn(q, radius)
    oi = oracle.index_build(rows, d, radius, 11, 22, override=override, prime=M31, threads=4)
    counters, offsets, ids = oi.query(q, radius, threads=4)
    assert (want.id == ids).all() and (want.offsets == offsets).all()
    for _ in range(3):
        got = ix.query_r_nn(pinned, radius)
        assert (got.triples() == want.triples()).all()
        assert (np.stack([got.collisions, got.candidates, got.found], 1) == counters).all()


@pytest.mark.parametrize("budget", [20000, 10**12])
@pytest.mark.parametrize("dup", [60, 6000])
def test_query_c_r_nn_any_budget_and_long_cut_buckets(budget, dup):
    """Budgets past the shared id set (> 12288) and buckets longer than the
    shared cut buffer (> 4096 postings: `dup` copies of one row) run from a
    global-memory set; the reference takes any std::optional<uint64_t> budget
    (index.hpp:90-93). Also: the shard's id offset is applied to the best id."""
    from oracle import oracle as O
    if not O.reference_available():
        pytest.skip("compiled reference unavailable")
    ref = O.reference()
    rng = np.random.default_rng(dup + budget % 97)
    d, radius = 128, 5
    rows = random_rows(rng, 9000, d)
    rows[10:10 + dup] = rows[5]
    q = np.concatenate([rows[5:6], planted_queries(rng, rows, d, 60, radius + 2)])
    plan = F.make_plan(d, radius, 1.0, rows.shape[0], 11, F.PlanOverride(F.PlanKind.identity, 1))
    oi = ref.index_build(rows, d, radius, 11, 22, override=(0, 1), prime=M31, threads=4)
    for b in (budget, 4100, 13000):
        want_c, want_b = oi.query_c(q, radius, b, threads=4)
        for layout in LAYOUTS:
            ix = F.build_index(rows, radius, plan, 22, prime=M31, layout=layout, id_offset=777)
            counters, bid, bd = ix.query_c_r_nn(q, radius, b)
            assert (counters == want_c).all(), (b, layout)
            none = want_b[:, 0] == 0xFFFFFFFF
            assert (bid[none] == -1).all()
            assert (bid[~none] == want_b[~none, 0].astype(np.int64) + 777).all()
            assert (bd[~none] == want_b[~none, 1]).all()


@pytest.mark.parametrize("prime", [(1 << 62) + 135, (1 << 40) - 87, 2147483659])
def test_home_bucket_spread_for_primes_below_a_power_of_two(oracle, prime):
    """Home buckets and filter bits come from the key's fraction of [0, P)
    (key * floor(2^64 / P)), so a prime just above a power of two (kbits = 63
    for 2^62 + 135) still spreads keys over every bucket; results equal the
    reference either way."""
    rng = np.random.default_rng(prime % 1000)
    d = 128
    rows = random_rows(rng, 4000, d)
    q = planted_queries(rng, rows, d, 120, 6)
    check_against_oracle(oracle, rows, q, d, 4, (0, 1), prime, layouts=("buckets", "csr"))


@pytest.mark.parametrize("extra", [-1, 0, 1, 15, 16, 17, 700])
def test_query_handout_around_the_first_wave(oracle, extra):
    """The warp kernel's first wave takes queries 0 .. warps-1 by warp index and
    hands the rest out from 16 counters (CTA b draws from counter b mod 16):
    batches just below, at and past the first wave's size (every counter
    empty, one query, each counter's first, a second round) answer every
    query exactly once. cfg3's shape (d = 512, two 256-bit parts, per-part
    radius 6: the fused hash, 5 CTAs/SM of 8 warps on this GPU)."""
    import torch
    rng = np.random.default_rng(1000 + extra)
    d, r = 512, 12
    rows = random_rows(rng, 20000, d)
    wave = 5 * 8 * torch.cuda.get_device_properties(0).multi_processor_count
    nq = wave + extra
    q = planted_queries(rng, rows, d, nq, r)
    res = check_against_oracle(oracle, rows, q, d, r, (2, 2), M31, layouts=("buckets",))
    assert res.found.sum() >= nq  # every planted query finds its source row
