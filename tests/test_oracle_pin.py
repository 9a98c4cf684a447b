"""Pins the CPU oracles before anything is checked against them.

* The plain-C restatement (oracle/fclsh_oracle.c) must equal the compiled
  reference (oracle/_ref, built from /root/reference's own sources) on RNG
  draws, families, plans, hashes, index queries and the linear scan.
* Both must reproduce the golden values of the reference's own unit tests
  (restated here with file:line; doctest itself is absent from the mount).
"""
import numpy as np
import pytest

from tests.helpers import flip, from_string, planted_queries, random_rows

P101 = 101
M31 = (1 << 31) - 1
M61 = (1 << 61) - 1


def oracles():
    from oracle import oracle as O
    out = [O.port()]
    if O.reference_available():
        out.append(O.reference())
    return out


@pytest.fixture(params=["port", "reference"])
def orc(request):
    from oracle import oracle as O
    if request.param == "reference":
        if not O.reference_available():
            pytest.skip("oracle/_ref not built")
        return O.reference()
    return O.port()


# ----------------------------------------------------------- test_hadamard.cpp

def test_fht_mod_goldens(orc):  # test_hadamard.cpp:93-106
    assert list(orc.fht_mod([1, 2, 3, 4], 5)) == [0, 3, 1, 0]
    assert list(orc.fht_mod([1, 1, 1, 1], 3)) == [1, 0, 0, 0]
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as e:
        orc.fht_mod([1, 2], 4)
    assert e.value.code == 2
    with pytest.raises(OracleError):
        orc.fht_mod([1, 2, 3], 5)


def test_batch_kernel_goldens(orc):  # test_hadamard.cpp:131-150
    assert list(orc.batch_hash_kernel([0, 0, 1, 1], 2, P101)) == [0, 1, 2, 1]
    assert list(orc.batch_hash_kernel([0] * 8, 0, 97)) == [0] * 8
    t = orc.batch_hash_kernel([1] * 8, 8, 97)
    assert t[0] == 0 and all(x == 4 for x in t[1:])


def test_batch_kernel_equals_codeword_dot_products(orc):  # test_hadamard.cpp:152-172
    rng = np.random.default_rng(24)
    for p in (5, 97, M61):
        for m in range(1, 7):
            n = 1 << m
            s = [int(rng.integers(0, min(p, 2**62))) % p for _ in range(n)]
            l1 = sum(s) % p
            direct = [sum(s[i] for i in range(n) if bin(v & i).count("1") & 1) % p for v in range(n)]
            assert list(orc.batch_hash_kernel(s, l1, p)) == direct


# ----------------------------------------------------------- test_covering.cpp

def _hash_one(orc, mapping, seeds, dims, radius, prime, s):
    return orc.hash_batch(np.array(mapping, np.uint32), np.array(seeds, np.uint64), dims, radius, prime,
                          from_string(s).reshape(1, -1), kind=0)[0]


def test_worked_small_family(orc):  # test_covering.cpp:37-78
    m, s = [3, 4, 5, 1], [2, 3, 5, 7]
    hx = _hash_one(orc, m, s, 4, 2, P101, "0011")
    hq = _hash_one(orc, m, s, 4, 2, P101, "1010")
    hz = _hash_one(orc, m, s, 4, 2, P101, "1001")
    assert [v for v in range(1, 8) if hx[v - 1] == hq[v - 1]] == [4]
    assert hx[3] == 5
    assert [v for v in range(1, 8) if hq[v - 1] == hz[v - 1]] == [2]


def test_worked_identity_family(orc):  # test_covering.cpp:80-112
    m, s = list(range(8)), [1, 2, 3, 4, 5, 6, 7, 8]
    hx = orc.hash_batch(np.array(m, np.uint32), np.array(s, np.uint64), 8, 2, P101,
                        from_string("00110011").reshape(1, -1), kind=1)[0]
    hq = orc.hash_batch(np.array(m, np.uint32), np.array(s, np.uint64), 8, 2, P101,
                        from_string("00111010").reshape(1, -1), kind=1)[0]
    hy = orc.hash_batch(np.array(m, np.uint32), np.array(s, np.uint64), 8, 2, P101,
                        from_string("00110001").reshape(1, -1), kind=1)[0]
    assert [v for v in range(1, 8) if hx[v - 1] == hq[v - 1]] == [3]
    assert hx[2] == 10
    assert not any(hy[v] == hq[v] for v in range(7))


def test_radius_one_unit_seeds(orc):  # test_covering.cpp:114-124
    h = orc.hash_batch(np.arange(4, dtype=np.uint32), np.ones(4, np.uint64), 4, 1, P101,
                       from_string("0011").reshape(1, -1), kind=1)[0]
    assert list(h) == [1, 2, 1]


def test_zero_vector_hashes_to_zero(orc):  # test_covering.cpp:126-134
    for r in (1, 2, 3):
        m, s, k = orc.build_family(100, r, 99 + r)
        h = orc.hash_batch(m, s, 100, r, M61, np.zeros((1, 2), np.uint64), kind=k)
        assert not h.any()


def test_family_reproducibility(orc):  # test_covering.cpp:180-191
    a = orc.build_family(200, 3, 424242)
    b = orc.build_family(200, 3, 424242)
    c = orc.build_family(200, 3, 424243)
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
    assert (a[0] != c[0]).any() or (a[1] != c[1]).any()


def test_family_validation(orc):  # test_covering.cpp:193-216
    from oracle.oracle import OracleError
    for args, code in [((0, 2, 1), 2), ((10, 0, 1), 2), ((10, 21, 1), 4)]:
        with pytest.raises(OracleError) as e:
            orc.build_family(*args)
        assert e.value.code == code
    with pytest.raises(OracleError):
        orc.build_family(10, 2, 1, prime=4)


def test_zero_column_handling(orc):  # test_covering.cpp:166-178
    m, _, _ = orc.build_family(500, 2, 7)
    assert (m >= 1).all()
    m0, _, _ = orc.build_family(500, 2, 7, include_zero=True)
    assert (m0 == 0).any()


# ------------------------------------------------------- port == reference

def test_port_equals_reference_rng(reference, port):
    for s in (0, 1, 12345, 2**63 + 7, 2**64 - 1):
        assert (reference.rng_draw(s, 2000) == port.rng_draw(s, 2000)).all()
        for lab in ("family", "mapping", "seeds", "plan-permutation", "run"):
            assert reference.stream(s, lab) == port.stream(s, lab)
            assert reference.stream(s, lab, 5) == port.stream(s, lab, 5)


def test_port_equals_reference_families_and_hashes(reference, port):
    rng = np.random.default_rng(2026)
    for trial in range(120):  # acceptance.cpp:152-181 style mix
        r = int(rng.integers(1, 8))
        order = 1 << (r + 1)
        general = trial % 2 == 0
        d = int(order + 1 + rng.integers(0, 300)) if general else int(2 + rng.integers(0, order - 1))
        prime = [M61, M31, 101, 97][trial % 4]
        iz = bool(rng.integers(0, 2))
        a = reference.build_family(d, r, 1000 + trial, prime=prime, include_zero=iz)
        b = port.build_family(d, r, 1000 + trial, prime=prime, include_zero=iz)
        assert (a[0] == b[0]).all() and (a[1] == b[1]).all() and a[2] == b[2] == (0 if general else 1)
        rows = random_rows(rng, 4, d)
        ka = reference.hash_batch(a[0], a[1], d, r, prime, rows, kind=a[2])
        kb = port.hash_batch(b[0], b[1], d, r, prime, rows)
        kc = port.hash_batch(b[0], b[1], d, r, prime, rows, reference_path=True)
        assert (ka == kb).all() and (kb == kc).all()


def test_port_equals_reference_plans(reference, port):
    cases = [(64, 2, 1.0, 1 << 16, None), (64, 2, 1.0, 1 << 16, None, 1000), (64, 4, 4.0, 1 << 16, None),
             (64, 5, 1.0, 1 << 14, None), (64, 16, 1.0, 1 << 14, None), (4, 3, 1.0, 16, None),
             (10, 6, 1.0, 16, (2, 3)), (512, 12, 1.0, 4_000_000, (2, 2)), (256, 16, 1.0, 10_000_000, (2, 2)),
             (64, 2, 4.0, 1 << 10, (1, 3)), (64, 2, 1.0, 1 << 16, (1, 1))]
    for cs in cases:
        d, r, c, n, ov = cs[:5]
        budget = cs[5] if len(cs) > 5 else 1 << 21
        a = reference.make_plan(d, r, c, n, 9, override=ov, budget=budget)
        b = port.make_plan(d, r, c, n, 9, override=ov, budget=budget)
        assert (a.kind, a.t, a.per_part_radius) == (b.kind, b.t, b.per_part_radius)
        assert (a.perm == b.perm).all() and (a.parts == b.parts).all()


def test_plan_goldens(orc):  # test_transform.cpp:15-66
    p = orc.make_plan(64, 2, 1.0, 1 << 16, 1)
    assert (p.kind, p.t, p.per_part_radius) == (1, 8, 16)
    p = orc.make_plan(64, 2, 1.0, 1 << 16, 1, budget=1000)
    assert (p.kind, p.t, p.per_part_radius) == (1, 4, 8)
    p = orc.make_plan(64, 4, 4.0, 1 << 16, 1)
    assert (p.kind, p.t, p.per_part_radius) == (0, 1, 4)
    p = orc.make_plan(64, 5, 1.0, 1 << 14, 1)
    assert (p.kind, p.t, p.per_part_radius) == (1, 2, 10)
    p = orc.make_plan(64, 16, 1.0, 1 << 14, 1)
    assert (p.kind, p.t, p.per_part_radius) == (2, 2, 8) and len(p.perm) == 64 and len(p.parts) == 2
    p = orc.make_plan(4, 3, 1.0, 16, 1)
    assert (p.kind, p.t) == (0, 1)


def test_partition_widths_and_bijection(orc):  # test_transform.cpp:103-120
    p = orc.make_plan(10, 6, 1.0, 16, 3, override=(2, 3))
    assert [int(e - b) for b, e in p.parts] == [3, 3, 4]
    assert sorted(p.perm.tolist()) == list(range(10))


def test_exhaustive_pigeonhole(orc):  # test_transform.cpp:214-236
    for r in (4, 6):
        for t in (2, 3):
            p = orc.make_plan(16, r, 1.0, 1 << 8, 20, override=(2, t))
            share = r // t
            z = np.arange(1 << 16, dtype=np.uint32)
            bits = ((z[:, None] >> np.arange(16, dtype=np.uint32)) & 1).astype(np.uint8)
            keep = bits.sum(1) <= r
            bits = bits[keep]
            light = np.zeros(bits.shape[0], bool)
            for b, e in p.parts:
                light |= bits[:, p.perm[b:e]].sum(1) <= share
            assert light.all()


def test_port_equals_reference_index_queries(reference, port):
    rng = np.random.default_rng(5)
    n, d = 3000, 128
    rows = random_rows(rng, n, d)
    q = planted_queries(rng, rows, d, 150, 9)
    for ov, rad in [((0, 1), 4), ((2, 2), 8), ((1, 2), 3)]:
        ir = reference.index_build(rows, d, rad, 11, 22, override=ov, prime=M31, threads=1)
        ip = port.index_build(rows, d, rad, 11, 22, override=ov, prime=M31, threads=4)
        a = ir.query(q, rad)
        b = ip.query(q, rad, threads=3)
        for x, y in zip(a, b):
            assert (x == y).all()
        truth = port.scan_truth(rows, q, d, rad, threads=2)
        assert (truth[:, 1] == a[2]).all()
        assert (reference.scan_truth(rows, q, d, rad, threads=3) == truth).all()


def test_parallel_reference_build_equals_build_index(reference):
    """ref_index_build(threads>1) must be the same IndexSet as build_index itself."""
    rng = np.random.default_rng(8)
    rows = random_rows(rng, 2000, 64)
    q = planted_queries(rng, rows, 64, 60, 5)
    a = reference.index_build(rows, 64, 8, 3, 4, override=(2, 2), prime=M61, threads=1).query(q, 8)
    b = reference.index_build(rows, 64, 8, 3, 4, override=(2, 2), prime=M61, threads=5).query(q, 8)
    for x, y in zip(a, b):
        assert (x == y).all()


def test_index_matches_brute_force_every_plan(orc):  # test_index.cpp:132-176
    rng = np.random.default_rng(330)
    d = 64
    rows = random_rows(rng, 1500, d)
    q = planted_queries(rng, rows, d, 8, 8)
    for ov, rad in [((0, 1), 3), ((1, 2), 3), ((2, 2), 8)]:
        ix = orc.index_build(rows, d, rad, 331, 332, override=ov)
        counters, offsets, ids = ix.query(q, rad)
        truth = orc.scan_truth(rows, q, d, rad)
        assert (ids == truth[:, 1]).all()
        assert (counters[:, 2] == np.diff(offsets)).all()
        assert (counters[:, 0] >= counters[:, 1]).all() and (counters[:, 1] >= counters[:, 2]).all()


def test_golden_fixtures(orc):
    """Vectors produced by the compiled reference (tests/golden/make_golden.py)."""
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "golden.json")
    g = json.load(open(path))
    for fam in g["families"]:
        m, s, k = orc.build_family(fam["dims"], fam["radius"], fam["seed"], prime=fam["prime"],
                                   include_zero=fam["include_zero"])
        assert m.tolist() == fam["mapping"] and [int(x) for x in s] == fam["seeds"] and k == fam["kind"]
        rows = np.array(fam["rows"], np.uint64).reshape(len(fam["keys"]), -1)
        keys = orc.hash_batch(m, s, fam["dims"], fam["radius"], fam["prime"], rows, kind=k)
        assert [[int(x) for x in r] for r in keys] == fam["keys"]
    for ix in g["indexes"]:
        rows = np.array(ix["rows"], np.uint64).reshape(ix["n"], -1)
        q = np.array(ix["queries"], np.uint64).reshape(len(ix["counters"]), -1)
        h = orc.index_build(rows, ix["dims"], ix["radius"], ix["plan_seed"], ix["index_seed"],
                            override=tuple(ix["override"]), prime=ix["prime"])
        counters, offsets, ids = h.query(q, ix["radius"])
        assert counters.tolist() == ix["counters"]
        assert offsets.tolist() == ix["offsets"] and ids.tolist() == ix["ids"]


def test_workload_generators_oracle_equals_product():
    """oracle/workloads.py (liboracle.so's orc_gen_*) produces the product's
    BASELINE inputs byte for byte, seed chain included, so the reference arm
    and the CPU baselines of bench.py never load libfclsh_b200.so; slices
    [row0, row0 + n) continue one global stream (the ranks of a cluster)."""
    from oracle.workloads import OracleBackend, load_configs
    from paper_1602_02620_b200 import configs as P
    S = load_configs()
    ob = OracleBackend()
    for cid in (1, 2, 3, 4):
        cfg = P.CONFIGS[cid].scaled(3000 if cid != 4 else 5000, queries=50)
        scfg = S.CONFIGS[cid].scaled(3000 if cid != 4 else 5000, queries=50)
        assert cfg.plan_seed() == scfg.plan_seed(ob) and cfg.index_seed() == scfg.index_seed(ob)
        a = P.make_data(cfg, 3)
        b = S.make_data(scfg, 5, backend=ob)
        assert (a == b).all()
        assert (P.make_queries(cfg, a, 2) == S.make_queries(scfg, b, 7, backend=ob)).all()
        tail = S.make_data(scfg, 4, backend=ob, row0=1000, n=1500)
        assert (tail == a[1000:2500]).all()
        assert (P.make_data(cfg, 1, row0=1000, n=1500) == tail).all()
    u = P.CONFIGS[2].scaled(2000)  # with the uniform queries
    d = P.make_data(u)
    assert (P.make_queries(u, d) == S.make_queries(S.CONFIGS[2].scaled(2000), d, backend=ob)).all()
