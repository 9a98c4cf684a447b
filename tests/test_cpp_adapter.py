"""The header-only C++ adapter (include/fclsh_gpu.hpp) compiles against the
C-ABI with a plain g++ and behaves like the reference API: host-only parts on
CPU, the full build + query on the GPU."""
import os
import subprocess

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


@pytest.mark.gpu
def test_cpp_adapter_on_gpu(binary):
    r = subprocess.run([binary], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "index tables=31" in r.stdout
