"""K1 parity on the GPU: every key bit-exact against the oracle's
hash_batch_into (covering.cpp:169-182), through the C-ABI."""
import numpy as np
import pytest

from paper_1602_02620_b200 import fclsh as F
from tests.helpers import from_string, random_rows

pytestmark = pytest.mark.gpu

M31, M61 = F.M31, F.M61


def test_worked_small_family():  # test_covering.cpp:37-78, P = 101 (generic path)
    f = F.make_covering_family(4, 2, F.ConstructionKind.general, [3, 4, 5, 1], [2, 3, 5, 7], 101)
    rows = np.stack([from_string("0011"), from_string("1010"), from_string("1001")])
    hx, hq, hz = F.hash_batch(f, rows)
    assert [v for v in range(1, 8) if hx[v - 1] == hq[v - 1]] == [4]
    assert hx[3] == 5
    assert [v for v in range(1, 8) if hq[v - 1] == hz[v - 1]] == [2]


def test_worked_identity_family():  # test_covering.cpp:80-112
    f = F.make_covering_family(8, 2, F.ConstructionKind.specific, list(range(8)), [1, 2, 3, 4, 5, 6, 7, 8], 101)
    hx, hq, hy = F.hash_batch(f, np.stack([from_string(s) for s in ("00110011", "00111010", "00110001")]))
    assert [v for v in range(1, 8) if hx[v - 1] == hq[v - 1]] == [3]
    assert hx[2] == 10
    assert not (hy == hq).any()


def test_radius_one_unit_seeds():  # test_covering.cpp:114-124
    f = F.make_covering_family(4, 1, F.ConstructionKind.specific, [0, 1, 2, 3], [1, 1, 1, 1], 101)
    assert list(F.hash_batch(f, from_string("0011").reshape(1, -1))[0]) == [1, 2, 1]


def test_worked_families_in_m31_fast_path(oracle):
    """The same worked families in the 2^31-1 field exercise the fast kernel."""
    for d, r, kind, m, s in [(4, 2, F.ConstructionKind.general, [3, 4, 5, 1], [2, 3, 5, 7]),
                             (8, 2, F.ConstructionKind.specific, list(range(8)), [1, 2, 3, 4, 5, 6, 7, 8]),
                             (4, 1, F.ConstructionKind.specific, [0, 1, 2, 3], [M31 - 1] * 4)]:
        f = F.make_covering_family(d, r, kind, m, s, M31)
        rows = random_rows(np.random.default_rng(d), 300, d)
        want = oracle.hash_batch(np.array(m, np.uint32), np.array(s, np.uint64), d, r, M31, rows, kind=int(kind))
        assert (F.hash_batch(f, rows).astype(np.uint64) == want).all()


def test_zero_and_full_rows():
    for r in (1, 2, 3, 5, 9):
        f = F.build_covering_family(100, r, 99 + r, prime=M31)
        zero = np.zeros((3, 2), np.uint64)
        assert not F.hash_batch(f, zero).any()


@pytest.mark.parametrize("radius", list(range(1, 11)))
@pytest.mark.parametrize("kind", ["specific", "general", "general0"])
def test_fast_path_random_families(oracle, radius, kind):
    """Every code order of the fast kernel (N = 4 .. 2048), both constructions,
    with and without the zero column, ragged n (not a multiple of the tile)."""
    order = 1 << (radius + 1)
    rng = np.random.default_rng(radius * 7 + len(kind))
    for trial in range(2):
        if kind == "specific":
            d = int(rng.integers(max(1, order // 2), order + 1))
        else:
            d = int(order + 1 + rng.integers(0, 3 * order))
        m, s, k = oracle.build_family(d, radius, 1000 * radius + trial, prime=M31, include_zero=(kind == "general0"))
        f = F.build_covering_family(d, radius, 1000 * radius + trial, prime=M31,
                                    include_zero_column=(kind == "general0"))
        n = int(rng.integers(1, 700))
        rows = random_rows(rng, n, d)
        rows[0] = 0
        if n > 2:
            rows[1] = ~np.uint64(0)
            if d % 64:
                rows[1, -1] &= np.uint64((1 << (d % 64)) - 1)
        want = oracle.hash_batch(m, s, d, radius, M31, rows, kind=k, threads=4)
        got = F.hash_batch(f, rows)
        bad = np.argwhere(got.astype(np.uint64) != want)
        assert bad.size == 0, f"d={d} r={radius} kind={kind}: {len(bad)} mismatches, first {bad[:5].tolist()}"


@pytest.mark.parametrize("prime", [M61, 101, (1 << 40) - 87, 2**62 + 135])
def test_generic_path_random_families(oracle, prime):
    rng = np.random.default_rng(prime % 977)
    for radius in (1, 3, 6, 9):
        d = int(rng.integers(2, 600))
        m, s, k = oracle.build_family(d, radius, radius, prime=prime)
        f = F.build_covering_family(d, radius, radius, prime=prime)
        rows = random_rows(rng, 37, d)
        want = oracle.hash_batch(m, s, d, radius, prime, rows, kind=k)
        got = F.hash_batch(f, rows, key_bytes=8)
        assert (got == want).all(), (d, radius, prime)


def test_device_layouts_match_host(oracle):
    """fclsh_hash_batch on device tensors: table-major and point-major layouts,
    4- and 8-byte keys, a padded stride."""
    import torch
    rng = np.random.default_rng(4)
    d, r = 300, 7
    f = F.build_covering_family(d, r, 5, prime=M31)
    rows = random_rows(rng, 1001, d)
    want = oracle.hash_batch(f.mapping, f.seeds, d, r, M31, rows, kind=int(f.kind))
    L = f.table_count()
    dr = torch.from_numpy(rows.view(np.int64)).cuda()
    kt = torch.zeros((L, 1004), dtype=torch.int32, device="cuda")
    F.hash_batch_device(f, dr, kt, layout=0, key_stride=1004)
    kp = torch.zeros((1001, L), dtype=torch.int64, device="cuda")
    F.hash_batch_device(f, dr, kp, layout=1)
    torch.cuda.synchronize()
    assert (kt.cpu().numpy()[:, :1001].T.astype(np.uint64) == want).all()
    assert (kp.cpu().numpy().astype(np.uint64) == want).all()


def test_hash_errors():
    f = F.build_covering_family(64, 3, 1, prime=M61)
    with pytest.raises(F.UsageError, match="width"):
        F.hash_batch(f, np.zeros((2, 2), np.uint64))
    with pytest.raises(F.UsageError, match="4-byte keys"):
        F.hash_batch(f, np.zeros((2, 1), np.uint64), key_bytes=4)


def test_partition_parts_fold_the_permutation(oracle):
    """Index families of a partition plan hash the permuted part views
    (split_vector, transform.cpp:123-135) -- checked through a built index."""
    rng = np.random.default_rng(12)
    d, r = 512, 12
    rows = random_rows(rng, 900, d)
    plan = F.make_plan(d, r, 1.0, 900, 3, F.PlanOverride(F.PlanKind.partition, 2))
    ix = F.build_index(rows, r, plan, 4, prime=M31)
    oi = oracle.index_build(rows, d, r, 3, 4, override=(2, 2), prime=M31)
    for p in range(2):
        fam = ix.family(p)
        m, s, rr, k = oi.family(p)
        assert (fam.mapping == m).all() and (fam.seeds == s).all() and fam.radius == rr == 6


_VARIANT_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from oracle import oracle as O
from paper_1602_02620_b200 import fclsh as F
from tests.helpers import random_rows
orc = O.best()
rng = np.random.default_rng(5)
for radius, d in [(2, 7), (5, 64), (6, 100), (8, 512), (9, 1000), (10, 1024), (10, 2048)]:
    m, s, k = orc.build_family(d, radius, 77 + radius, prime=F.M31)
    f = F.build_covering_family(d, radius, 77 + radius, prime=F.M31)
    rows = random_rows(rng, 333, d)
    rows[0] = 0
    rows[1] = ~np.uint64(0)
    if d % 64:
        rows[1, -1] &= np.uint64((1 << (d % 64)) - 1)
    want = orc.hash_batch(m, s, d, radius, F.M31, rows, kind=k, threads=4)
    for kb in (4, 8):
        got = F.hash_batch(f, rows, key_bytes=kb)
        assert (got.astype(np.uint64) == want).all(), (radius, d, kb)
print("variant ok")
"""


@pytest.mark.parametrize("env", [{}, {"FCLSH_HASH_F64_PM": "1"}, {"FCLSH_HASH_INT": "1"}, {"FCLSH_HASH_PK32": "1"}],
                         ids=["default", "f64_pm", "int_planes", "pk32"])
def test_hash_kernel_variants(env):
    """The 2^31-1 kernels the launcher falls back to (family table too large
    for the 12-warp layout, A/B knobs) hold the same keys as the default one:
    each variant in its own process (the knobs are read once), 4- and 8-byte
    keys, against hash_batch_into (covering.cpp:169-182)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT, root], env=e, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "variant ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
