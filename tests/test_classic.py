"""The classic bit-sampling baseline (classic.hpp / classic.cpp, the
paper's comparison method; Method::classic in build_index, index.cpp:65-76)
on the device: choose_k and the family (host) and hash_tables_into (device
kernel k_hash_classic) equal the compiled reference's, and a classic index
answers query_r_nn with the reference's ids and counters."""
import numpy as np
import pytest

from paper_1602_02620_b200 import fclsh as F
from tests.helpers import planted_queries, random_rows

M31 = F.M31


@pytest.fixture(scope="module")
def ref():
    from oracle import oracle as O
    if not O.reference_available():
        pytest.skip("compiled reference unavailable")
    return O.reference()


@pytest.mark.parametrize("dims,radius,tables,delta", [(128, 4, 31, 0.1), (256, 8, 511, 0.1), (64, 3, 15, 0.5),
                                                      (1024, 10, 2047, 0.01), (100, 99, 7, 0.3), (32, 1, 1, 0.9)])
def test_choose_k_equals_reference(ref, dims, radius, tables, delta):
    assert F.choose_k(dims, radius, tables, delta) == ref.choose_k(dims, radius, tables, delta)


@pytest.mark.parametrize("dims,k,tables,prime", [(128, 83, 31, M31), (256, 40, 511, F.M61), (70, 3, 5, 101)])
def test_bit_sample_family_equals_reference(ref, dims, k, tables, prime):
    f = F.build_bit_sample_family(dims, k, tables, 1234, prime)
    pos, seeds = ref.bitsample_family(dims, k, tables, 1234, prime)
    assert (f.positions == pos).all() and (f.seeds == seeds).all()
    assert f.positions.max() < dims and f.seeds.max() < prime


def test_classic_errors_mirror_reference():
    with pytest.raises(F.UsageError, match="choose_k: radius must be in"):
        F.choose_k(64, 64, 3, 0.1)
    with pytest.raises(F.UsageError, match="choose_k: delta must be in"):
        F.choose_k(64, 3, 3, 1.0)
    with pytest.raises(F.UsageError, match="k must be >= 1"):
        F.build_bit_sample_family(64, 0, 3, 1, M31)
    with pytest.raises(F.UsageError, match="prime must be odd"):
        F.build_bit_sample_family(64, 3, 3, 1, 100)


@pytest.mark.gpu
@pytest.mark.parametrize("dims,k,tables,prime", [(128, 83, 31, M31), (256, 40, 511, F.M61), (100, 400, 7, 101),
                                                 (1024, 9, 2047, M31)])
def test_hash_tables_equals_reference(ref, dims, k, tables, prime):
    rng = np.random.default_rng(dims + k)
    rows = random_rows(rng, 3000, dims)
    f = F.build_bit_sample_family(dims, k, tables, 77, prime)
    got = F.hash_tables(f, rows)
    want = ref.hash_tables(dims, k, tables, f.positions, f.seeds, prime, rows, threads=8)
    assert (got == want).all()


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["buckets", "csr"])
@pytest.mark.parametrize("d,radius,prime,k_override,tables_override,delta",
                         [(128, 4, M31, 0, 0, 0.1), (256, 8, F.M61, 0, 0, 0.1), (128, 6, M31, 20, 64, 0.1),
                          (96, 3, M31, 0, 200, 0.3)])
def test_classic_index_equals_reference(ref, layout, d, radius, prime, k_override, tables_override, delta):
    rng = np.random.default_rng(d * radius + k_override)
    rows = random_rows(rng, 4000, d)
    rows[100:140] = rows[7]  # duplicates: long buckets
    q = np.concatenate([rows[7:8], planted_queries(rng, rows, d, 200, radius + 2), random_rows(rng, 10, d)])
    plan = F.make_plan(d, radius, 1.0, rows.shape[0], 11, F.PlanOverride(F.PlanKind.identity, 1))
    ix = F.build_index(rows, radius, plan, 22, prime=prime, layout=layout, method="classic", delta=delta,
                       k_override=k_override or None, tables_override=tables_override or None)
    assert ix.method == "classic"
    oi = ref.index_build_classic(rows, d, radius, 11, 22, prime=prime, delta=delta, k_override=k_override,
                                 tables_override=tables_override)
    assert ix.table_count() == oi.table_count
    res = ix.query_r_nn(q, radius)
    counters, offsets, ids = oi.query(q, radius, threads=4)
    assert (np.stack([res.collisions, res.candidates, res.found], 1) == counters).all()
    assert (res.offsets == offsets).all() and (res.id == ids).all()
    fam = ix.bit_sample_family()
    k = F.choose_k(d, radius, ix.table_count(), delta) if not k_override else k_override
    assert ix.classic_k == k and fam.positions.size == k * ix.table_count()
    # the same classic index sharded three ways (fclsh_cluster): same families, same results
    cl = F.Cluster([0], 3).build(rows, radius, plan, 22, prime=prime, layout=layout, method="classic", delta=delta,
                                 k_override=k_override or None, tables_override=tables_override or None)
    cres = cl.query_r_nn(q, radius)
    assert (cres.triples() == res.triples()).all() and (cres.collisions == res.collisions).all()
    assert (cres.candidates == res.candidates).all()


@pytest.mark.gpu
def test_classic_index_rejects_non_identity_plans():
    rows = random_rows(np.random.default_rng(3), 100, 64)
    plan = F.make_plan(64, 4, 1.0, 100, 1, F.PlanOverride(F.PlanKind.partition, 2))
    with pytest.raises(F.UsageError, match="classic baseline expects the identity plan"):
        F.build_index(rows, 4, plan, 2, prime=M31, method="classic")
