"""run_experiment over the engine against the reference's
run_experiment (bench.cpp:64-158): every column but the stage times equal."""
import numpy as np
import pytest

from paper_1602_02620_b200 import fclsh as F
from paper_1602_02620_b200.experiment import ExperimentConfig, GroundTruth, run_experiment
from tests.helpers import planted_queries, random_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    from oracle import oracle as O
    if not O.reference_available():
        pytest.skip("compiled reference unavailable")
    return O.reference()


CASES = [
    ("fclsh", 64, 3, (0, 1), F.M31, 2, True),
    ("fclsh", 128, 6, (2, 2), F.M61, 2, False),
    ("bclsh", 96, 4, (0, 1), F.M31, 1, True),
    ("fclsh", 100, 5, None, F.M61, 3, True),
    ("linear", 128, 5, None, F.M31, 1, True),
    ("classic", 64, 3, (0, 1), F.M31, 2, True),
    ("classic", 128, 6, (2, 2), F.M61, 1, False),
]


@pytest.mark.parametrize("method,dims,radius,override,prime,repeats,fresh", CASES)
def test_metrics_match_the_reference(ref, method, dims, radius, override, prime, repeats, fresh):
    rng = np.random.default_rng(dims + radius)
    rows = random_rows(rng, 2500, dims)
    q = np.concatenate([planted_queries(rng, rows, dims, 60, radius + 2), random_rows(rng, 5, dims)])
    truth = ref.scan_truth(rows, q, dims, radius + 1, threads=8)  # a truth radius above the query radius
    ov = None if override is None else F.PlanOverride(F.PlanKind(override[0]), override[1])
    cfg = ExperimentConfig(method=method, radius=radius, plan_override=ov, seed=11, repeats=repeats,
                           fresh_seeds=fresh, prime=prime)
    got = run_experiment(rows, q, dims, GroundTruth(radius + 1, truth), cfg)
    want = ref.run_experiment(rows, q, dims, truth, radius + 1, method, radius, override=override, seed=11,
                              repeats=repeats, fresh_seeds=fresh, prime=prime)
    g = np.array([[r.query_id, r.radius, r.collisions, r.candidates, r.found, r.true_near, r.precision, r.recall]
                  for r in got])
    assert (g == want[:, :8]).all(), np.argwhere(g != want[:, :8])[:5]


def test_experiment_errors():
    rows = random_rows(np.random.default_rng(1), 100, 64)
    t = GroundTruth(3)
    with pytest.raises(F.DataError, match="below the query radius"):
        run_experiment(rows, rows[:3], 64, t, ExperimentConfig(radius=4))
    with pytest.raises(F.UsageError, match="repeats"):
        run_experiment(rows, rows[:3], 64, t, ExperimentConfig(radius=2, repeats=0))
    with pytest.raises(F.UsageError, match="not part of the GPU engine"):
        run_experiment(rows, rows[:3], 64, t, ExperimentConfig(method="mih", radius=2))
    with pytest.raises(F.UsageError, match="unknown method"):
        run_experiment(rows, rows[:3], 64, t, ExperimentConfig(method="foo", radius=2))
