"""TEST / BENCH INFRASTRUCTURE ONLY -- the BASELINE inputs without the product.

A backend for paper_1602_02620_b200/configs.py (make_data / make_queries /
the seed chain) built on the plain-C oracle (oracle/lib/liboracle.so:
orc_gen_*, orc_rng_stream), byte-identical to the product's fclsh_gen_*
(pinned by tests/test_oracle_pin.py). bench.py's reference arm and CPU
legs use it so that the reference's timed path never maps libfclsh_b200.so.

configs.py is loaded from its file here (not as part of the product
package, whose __init__ would import the product's Python modules).
"""
from __future__ import annotations

import ctypes as C
import importlib.util
import os
import sys

import numpy as np

from . import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
CONFIGS_PY = os.path.join(os.path.dirname(HERE), "paper_1602_02620_b200", "configs.py")

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)


def load_configs():
    """paper_1602_02620_b200/configs.py as a standalone module (its product
    backend is only imported lazily, and never by the oracle backend)."""
    name = "fclsh_bench_configs"
    if name in sys.modules:
        return sys.modules[name]
    spec = importlib.util.spec_from_file_location(name, CONFIGS_PY)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod  # (dataclasses resolve their module through sys.modules)
    spec.loader.exec_module(mod)
    return mod


class OracleBackend:
    """Seed chain + generators of configs.py on liboracle.so."""

    def __init__(self):
        self.orc = O.port()
        L = self.orc.lib
        L.orc_gen_bernoulli.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u64p, C.c_int]
        L.orc_gen_bernoulli.restype = None
        L.orc_gen_clustered.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                        u64p, C.c_int]
        L.orc_gen_clustered.restype = None
        L.orc_gen_planted.argtypes = [C.c_uint64, u64p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, u64p, u32p]
        L.orc_gen_planted.restype = None
        self.L = L

    def rng_stream(self, seed, label, index=None):
        return self.orc.stream(seed, label, index)

    def gen_bernoulli(self, seed, n, dims, threads=8, row0=0):
        out = np.zeros((n, (dims + 63) // 64), np.uint64)
        self.L.orc_gen_bernoulli(seed, row0, n, dims, out.ctypes.data_as(u64p), threads)
        return out

    def gen_clustered(self, seed, centres, n, dims, flip_p, threads=8, row0=0):
        out = np.zeros((n, (dims + 63) // 64), np.uint64)
        self.L.orc_gen_clustered(seed, centres, row0, n, dims, float(flip_p), out.ctypes.data_as(u64p), threads)
        return out

    def gen_planted(self, seed, data, dims, nq, kmax):
        d = np.ascontiguousarray(data, dtype=np.uint64)
        out = np.zeros((nq, (dims + 63) // 64), np.uint64)
        src = np.zeros(nq, np.uint32)
        self.L.orc_gen_planted(seed, d.ctypes.data_as(u64p), d.shape[0], dims, nq, kmax, out.ctypes.data_as(u64p),
                               src.ctypes.data_as(u32p))
        return out, src
