"""The header-only C++ adapter (include/fclsh_gpu.hpp) compiles against the
C-ABI with a plain g++ and behaves like the reference API: host-only parts on
CPU, the full build + query on the GPU."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1602_02620_b200", "lib")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "cpp_drop_in")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "cpp_drop_in.cpp"), "-L", LIB, "-lfclsh_b200",
                    f"-Wl,-rpath,{LIB}", "-o", out], check=True)
    return out


def test_cpp_adapter_host_only(binary, oracle):
    r = subprocess.run([binary, "--host-only"], capture_output=True, text=True, check=True)
    lines = r.stdout.splitlines()
    assert lines[0].startswith("family tables=31")
    assert "usage error ok: plan: radius must be >= 1" in r.stdout
    run = oracle.stream(42, "run", 0)
    m, s, _ = oracle.build_family(128, 4, oracle.stream(oracle.stream(run, "index"), "family", 0), prime=(1 << 31) - 1)
    assert f"mapping0={m[0]} seed0={s[0]}" in lines[0]


def _read_dump(path, nq):
    with open(path) as f:
        lines = f.read().split("\n")
    out, k = [], 0
    for _ in range(2):
        total = int(lines[k])
        k += 1
        per = np.array([[int(x) for x in lines[k + i].split()] for i in range(nq)], np.uint64)
        k += nq
        pairs = np.array([[int(x) for x in lines[k + i].split()] for i in range(total)], np.uint64).reshape(-1, 2)
        k += total
        out.append((per, pairs))
    return out


@pytest.mark.gpu
def test_cpp_adapter_on_gpu(binary, tmp_path, oracle):
    """The C++ caller's index and 4-shard cluster results equal the
    reference's query_r_nn (ids, counters) and scan_truth (distances)."""
    from oracle.workloads import OracleBackend
    path = str(tmp_path / "dump.txt")
    r = subprocess.run([binary, "--dump", path], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "index tables=31" in r.stdout
    n, d, nq, radius = 20000, 128, 200, 4
    rows = OracleBackend().gen_bernoulli(42, n, d, 4)
    q = rows[np.arange(nq) * 100].copy()
    for i in range(nq):
        for b in range(i % 6):
            q[i, b // 64] ^= np.uint64(1 << (b % 64))
    run = oracle.stream(42, "run", 0)
    oi = oracle.index_build(rows, d, radius, oracle.stream(run, "plan"), oracle.stream(run, "index"),
                            override=(0, 1), prime=(1 << 31) - 1, threads=4)
    counters, offsets, ids = oi.query(q, radius, threads=4)
    truth = oracle.scan_truth(rows, q, d, radius, threads=4)
    for per, pairs in _read_dump(path, nq):
        assert (per[:, 0] == offsets[1:]).all()
        assert (per[:, 1:] == counters).all()
        assert (pairs[:, 0] == ids).all()
        assert (pairs[:, 1] == truth[:, 2]).all()
