"""CPU-only checks of the product library (no kernel launches):
the C-ABI loads and exports every symbol include/fclsh_gpu.h declares, and
its host logic -- Rng streams, covering-family construction, plans,
validation / error codes, workload generators -- equals the oracle."""
import re

import numpy as np
import pytest

from paper_1602_02620_b200 import _native as N
from paper_1602_02620_b200 import fclsh as F

M31, M61 = F.M31, F.M61


def declared_functions():
    src = open(N.HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(fclsh_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    names = declared_functions()
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(N.SIGNATURES), "ctypes table out of sync with the header"
    assert b"sm_100a" in lib.fclsh_version()


def test_device_count_without_gpu_is_zero_or_more():
    assert F.device_count() >= 0


def test_rng_streams_equal_oracle(oracle):
    for s in (0, 5, 2**64 - 1, 0x1602_02620):
        for lab in ("family", "plan", "run", "index", "plan-permutation"):
            assert F.rng_stream(s, lab) == oracle.stream(s, lab)
            assert F.rng_stream(s, lab, 3) == oracle.stream(s, lab, 3)


@pytest.mark.parametrize("prime", [M31, M61, 101, 97, 5])
def test_families_equal_oracle(oracle, prime):
    rng = np.random.default_rng(prime % 1000)
    for trial in range(60):
        r = int(rng.integers(1, 11))
        order = 1 << (r + 1)
        d = int(rng.integers(1, 3 * order))
        iz = bool(trial % 3 == 0)
        seed = int(rng.integers(0, 2**63))
        m, s, k = oracle.build_family(d, r, seed, prime=prime, include_zero=iz)
        f = F.build_covering_family(d, r, seed, prime=prime, include_zero_column=iz)
        assert f.kind == k and f.dims == d and f.radius == r and f.prime == prime
        assert (f.mapping == m).all() and (f.seeds == s).all()


def test_family_errors_mirror_reference():
    with pytest.raises(F.UsageError, match="dims must be positive"):
        F.build_covering_family(0, 2, 1)
    with pytest.raises(F.UsageError, match="radius must be >= 1"):
        F.build_covering_family(10, 0, 1)
    with pytest.raises(F.ResourceError):
        F.build_covering_family(10, 21, 1)
    with pytest.raises(F.UsageError, match="prime"):
        F.build_covering_family(10, 2, 1, prime=4)
    with pytest.raises(F.UsageError, match="specific construction"):
        F.build_covering_family(100, 2, 1, kind=F.ConstructionKind.specific)
    with pytest.raises(F.UsageError, match="general construction"):
        F.build_covering_family(4, 2, 1, kind=F.ConstructionKind.general)
    # make_covering_family validation (test_covering.cpp:204-215)
    with pytest.raises(F.UsageError):
        F.make_covering_family(4, 2, F.ConstructionKind.general, [3, 4, 5], [2, 3, 5, 7], 101)
    with pytest.raises(F.UsageError, match="out of range"):
        F.make_covering_family(4, 2, F.ConstructionKind.general, [3, 4, 5, 9], [2, 3, 5, 7], 101)
    with pytest.raises(F.UsageError, match="injective"):
        F.make_covering_family(4, 2, F.ConstructionKind.specific, [1, 1, 2, 3], [2, 3, 5, 7], 101)
    with pytest.raises(F.UsageError, match="seed out of field"):
        F.make_covering_family(4, 2, F.ConstructionKind.general, [3, 4, 5, 1], [2, 3, 5, 101], 101)
    f = F.make_covering_family(4, 2, F.ConstructionKind.general, [3, 4, 5, 1], [2, 3, 5, 7], 101)
    assert f.table_count() == 7 and f.code_order() == 8


def test_plans_equal_oracle(oracle):
    cases = [(64, 2, 1.0, 1 << 16, None, 1 << 21), (64, 2, 1.0, 1 << 16, None, 1000),
             (64, 4, 4.0, 1 << 16, None, 1 << 21), (64, 5, 1.0, 1 << 14, None, 1 << 21),
             (64, 16, 1.0, 1 << 14, None, 1 << 21), (4, 3, 1.0, 16, None, 1 << 21),
             (10, 6, 1.0, 16, (2, 3), 1 << 21), (512, 12, 1.0, 4_000_000, (2, 2), 1 << 21),
             (256, 16, 1.0, 10_000_000, (2, 2), 1 << 21), (64, 2, 4.0, 1 << 10, (1, 3), 1 << 21),
             (101, 7, 1.5, 5000, (2, 3), 1 << 21)]
    for d, r, c, n, ov, budget in cases:
        o = oracle.make_plan(d, r, c, n, 33, override=ov, budget=budget)
        force = None if ov is None else F.PlanOverride(F.PlanKind(ov[0]), ov[1])
        p = F.make_plan(d, r, c, n, 33, force, budget)
        assert (int(p.kind), p.t, p.per_part_radius) == (o.kind, o.t, o.per_part_radius)
        if p.kind == F.PlanKind.partition:
            assert (p.permutation == o.perm).all()
            assert p.parts == [tuple(int(x) for x in pr) for pr in o.parts]


def test_plan_errors_mirror_reference():
    with pytest.raises(F.UsageError, match="radius must be below dims"):
        F.make_plan(64, 64, 1.0, 1024, 1)
    with pytest.raises(F.UsageError, match="approximation factor"):
        F.make_plan(64, 2, 0.5, 1024, 1)
    with pytest.raises(F.UsageError, match="two data points"):
        F.make_plan(64, 2, 1.0, 1, 1)
    with pytest.raises(F.UsageError, match="identity override"):
        F.make_plan(64, 2, 1.0, 1024, 1, F.PlanOverride(F.PlanKind.identity, 2))
    with pytest.raises(F.UsageError, match="override factor"):
        F.make_plan(64, 2, 1.0, 1024, 1, F.PlanOverride(F.PlanKind.replicate, 0))
    with pytest.raises(F.UsageError, match="cannot cut radius"):
        F.make_plan(64, 4, 1.0, 1024, 1, F.PlanOverride(F.PlanKind.partition, 5))
    with pytest.raises(F.ResourceError):
        F.make_plan(64, 21, 1.0, 1 << 21, 1, F.PlanOverride(F.PlanKind.identity, 1))


def test_generators_deterministic_and_shaped():
    a = F.gen_bernoulli(7, 5000, 200, threads=1)
    b = F.gen_bernoulli(7, 5000, 200, threads=7)
    assert (a == b).all()
    assert not (a[:, -1] >> np.uint64(8)).any()  # padding bits zero (200 % 64 = 8)
    ones = np.unpackbits(a.view(np.uint8), axis=1).sum() / (5000 * 200)
    assert abs(ones - 0.5) < 0.01
    c1 = F.gen_clustered(3, 10, 4000, 128, 0.05, threads=1)
    c2 = F.gen_clustered(3, 10, 4000, 128, 0.05, threads=5)
    assert (c1 == c2).all()
    q, src = F.gen_planted(9, a, 200, 300, 6)
    d = np.unpackbits((q ^ a[src]).view(np.uint8), axis=1).sum(1)
    assert d.max() <= 6 and (d == 0).any() and (d == 6).any()


def test_configs_seed_chain():
    from paper_1602_02620_b200.configs import CONFIGS
    cfg = CONFIGS[2]
    run = F.rng_stream(cfg.root(), "run", 0)
    assert cfg.plan_seed() == F.rng_stream(run, "plan")
    assert cfg.index_seed() == F.rng_stream(run, "index")
    assert CONFIGS[3].tables == 254 and CONFIGS[4].tables == 1022 and CONFIGS[5].tables == 2047
