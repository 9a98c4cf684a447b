"""GPU linear scan against the reference's scan_truth
(workload.cpp:56-71) and distance_histogram (workload.cpp:133-151), and the
FCL1 -> pinned host -> device upload path."""
import numpy as np
import pytest

from paper_1602_02620_b200 import fclsh as F
from tests.helpers import planted_queries, random_rows

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).cuda()


@pytest.mark.parametrize("dims,radius", [(64, 3), (100, 6), (256, 8), (600, 40), (1024, 12)])
def test_scan_truth_matches_the_reference(oracle, dims, radius):
    rng = np.random.default_rng(dims)
    rows = random_rows(rng, 3000, dims)
    q = np.concatenate([planted_queries(rng, rows, dims, 90, radius + 3), random_rows(rng, 10, dims)])
    got = F.LinearScan().triples(_dev(rows), _dev(q), dims, radius)
    want = oracle.scan_truth(rows, q, dims, radius, threads=8)
    assert got.shape == want.shape and (got == want).all()


def test_scan_truth_edges(oracle):
    rng = np.random.default_rng(1)
    rows = random_rows(rng, 500, 128)
    sc = F.LinearScan()
    empty = sc.scan_truth(_dev(rows), _dev(np.zeros((0, 2), np.uint64)), 128, 5)
    assert empty.nq == 0 and empty.total == 0
    # radius 0: exact duplicates only; radius = dims: every pair
    q = rows[:7].copy()
    assert (sc.triples(_dev(rows), _dev(q), 128, 0) == oracle.scan_truth(rows, q, 128, 0)).all()
    all_pairs = sc.triples(_dev(rows), _dev(q), 128, 128)
    assert all_pairs.shape[0] == 7 * 500 and (all_pairs == oracle.scan_truth(rows, q, 128, 128)).all()
    with pytest.raises(F.UsageError):
        sc.scan_truth(_dev(rows), _dev(q), 0, 1)


def test_scan_agrees_with_the_index(oracle):
    """The exhaustive scan and the fcLSH index return the same triples (100 % recall)."""
    rng = np.random.default_rng(7)
    rows = random_rows(rng, 20000, 256)
    q = planted_queries(rng, rows, 256, 500, 8)
    plan = F.make_plan(256, 8, 1.0, 20000, 3, F.PlanOverride(F.PlanKind.identity, 1))
    res = F.build_index(rows, 8, plan, 4, prime=F.M31).query_r_nn(q, 8)
    assert (F.LinearScan().triples(_dev(rows), _dev(q), 256, 8) == res.triples()).all()


@pytest.mark.parametrize("sample", [0, 7])
def test_distance_histogram_matches_the_reference(sample):
    from oracle import oracle as O
    if not O.reference_available():
        pytest.skip("compiled reference unavailable")
    ref = O.reference()
    rng = np.random.default_rng(5 + sample)
    rows = random_rows(rng, 700, 96)
    q = random_rows(rng, 40, 96)
    got = F.LinearScan().distance_histogram(_dev(rows), _dev(q), 96, sample_per_query=sample, seed=99)
    want = ref.distance_histogram(rows, q, 96, sample_per_query=sample, seed=99)
    assert (got == want).all()
    assert got.sum() == 40 * (700 if sample == 0 else sample)


def test_dataset_upload(tmp_path):
    import torch
    rows = random_rows(np.random.default_rng(2), 3000, 320)
    path = tmp_path / "d.bin"
    F.save_dataset(path, rows, 320)
    ds = F.load_dataset(path)
    dev = ds.upload(0)
    torch.cuda.synchronize()
    assert (dev.cpu().numpy().view(np.uint64) == rows).all()
