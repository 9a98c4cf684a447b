"""TEST INFRASTRUCTURE ONLY -- ctypes access to the two CPU oracles.

* ``port()``      -> oracle/lib/liboracle.so, the plain-C restatement
                     (oracle/fclsh_oracle.c).
* ``reference()`` -> oracle/_ref/libfclsh_ref.so, the reference library
                     compiled from its own sources (oracle/Makefile) behind
                     oracle/ref_shim.cpp.

Both expose the same functions (prefix ``orc_`` / ``ref_``); this module
wraps them behind one class so a test can run the same check against either.
Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs import this.
The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "lib", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfclsh_ref.so")

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
i64p = C.POINTER(C.c_int64)


def _p(a, t):
    return a.ctypes.data_as(t)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


@dataclass
class Plan:
    kind: int  # 0 identity, 1 replicate, 2 partition
    t: int
    per_part_radius: int
    perm: np.ndarray  # uint32 [dims] (partition only)
    parts: np.ndarray  # uint64 [t, 2] (partition only)


class Oracle:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        self.kind = "reference" if prefix == "ref_" else "port"
        self.lib = C.CDLL(path)
        self.p = prefix
        L = self.lib
        f = lambda name: getattr(L, prefix + name)  # noqa: E731
        self._last_error = f("last_error")
        self._last_error.restype = C.c_char_p
        self._free = f("free")
        self._free.argtypes = [C.c_void_p]
        self._stream = f("rng_stream")
        self._stream.restype = C.c_uint64
        self._stream.argtypes = [C.c_uint64, C.c_char_p]
        self._stream_idx = f("rng_stream_idx")
        self._stream_idx.restype = C.c_uint64
        self._stream_idx.argtypes = [C.c_uint64, C.c_char_p, C.c_uint64]
        self._draw = f("rng_draw")
        self._draw.argtypes = [C.c_uint64, C.c_uint64, u64p]
        self._fht_mod = f("fht_mod")
        self._fht_mod.argtypes = [u64p, C.c_uint64, C.c_uint64]
        self._bhk = f("batch_hash_kernel")
        self._bhk.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint64]
        self._build_family = f("build_family")
        self._build_family.argtypes = [C.c_uint64, C.c_uint32, C.c_int, C.c_uint64, C.c_uint64,
                                       C.c_int, u32p, u64p, C.POINTER(C.c_int)]
        self._make_plan = f("make_plan")
        self._make_plan.argtypes = [C.c_uint64, C.c_uint32, C.c_double, C.c_uint64, C.c_uint64,
                                    C.c_int, C.c_int, C.c_uint32, C.c_uint64, C.POINTER(C.c_int),
                                    u32p, u32p, u32p, u64p]
        self._index_destroy = f("index_destroy")
        self._index_destroy.argtypes = [C.c_void_p]
        self._index_family = f("index_family")
        self._index_family.argtypes = [C.c_void_p, C.c_uint32, u32p, u64p, u64p, u32p,
                                       C.POINTER(C.c_int)]
        self._table_count = f("index_table_count")
        self._table_count.restype = C.c_uint64
        self._table_count.argtypes = [C.c_void_p]
        self._index_query = f("index_query")
        self._index_query.argtypes = [C.c_void_p, u64p, C.c_uint64, C.c_uint32, C.c_int, u64p,
                                      u64p, C.POINTER(u32p)] + ([C.POINTER(C.c_double)] if prefix == "ref_" else [])
        self._scan = f("scan_truth")
        self._scan.argtypes = [u64p, C.c_uint64, u64p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_int,
                               C.POINTER(u32p), u64p]
        if prefix == "ref_":
            self._hash = f("hash_batch")
            self._hash.argtypes = [C.c_uint64, C.c_uint32, C.c_int, u32p, u64p, C.c_uint64, u64p,
                                   C.c_uint64, u64p, C.c_int, C.c_int, C.POINTER(C.c_double)]
            self._index_build = f("index_build")
            self._index_build.restype = C.c_void_p
            self._index_build.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64,
                                          C.c_int, C.c_int, C.c_uint32, C.c_double, C.c_uint64,
                                          C.c_uint64, C.c_int, C.c_uint64, C.c_int,
                                          C.POINTER(C.c_double), C.POINTER(C.c_int)]
            self._ds_save = f("dataset_save")
            self._ds_save.argtypes = [C.c_char_p, u64p, C.c_uint64, C.c_uint64, C.c_int]
            self._ds_load = f("dataset_load")
            self._ds_load.argtypes = [C.c_char_p, u64p, u64p, C.POINTER(u64p)]
            self._index_query_c = f("index_query_c")
            self._index_query_c.argtypes = [C.c_void_p, u64p, C.c_uint64, C.c_uint32, C.c_int64, C.c_int, u64p,
                                            u32p]
            self._run_exp = f("run_experiment")
            self._run_exp.argtypes = [u64p, C.c_uint64, u64p, C.c_uint64, C.c_uint64, u32p, C.c_uint64, C.c_uint32,
                                      C.c_char_p, C.c_uint32, C.c_double, C.c_int, C.c_uint32, C.c_uint64,
                                      C.c_uint32, C.c_int, C.c_uint64, C.POINTER(C.c_double),
                                      C.POINTER(C.c_char_p)]
            self._choose_k = f("choose_k")
            self._choose_k.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_double, u32p]
            self._bsf = f("bitsample_family")
            self._bsf.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, u32p, u64p]
            self._hash_tables = f("hash_tables")
            self._hash_tables.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, u32p, u64p, C.c_uint64, u64p,
                                          C.c_uint64, u64p, C.c_int]
            self._build_classic = f("index_build_classic")
            self._build_classic.restype = C.c_void_p
            self._build_classic.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, C.c_double,
                                            C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_uint32,
                                            C.c_uint64, C.POINTER(C.c_int)]
            self._hist = f("distance_histogram")
            self._hist.argtypes = [u64p, C.c_uint64, u64p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        else:
            self._hash = f("hash_batch")
            self._hash.argtypes = [u32p, u64p, C.c_uint64, C.c_uint32, C.c_uint64, u64p,
                                   C.c_uint64, u64p, C.c_int]
            self._hash_ref = f("hash_reference")
            self._hash_ref.argtypes = [u32p, u64p, C.c_uint64, C.c_uint32, C.c_uint64, u64p,
                                       C.c_uint64, u64p]
            self._index_build = f("index_build")
            self._index_build.restype = C.c_void_p
            self._index_build.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64,
                                          C.c_int, C.c_int, C.c_uint32, C.c_double, C.c_uint64,
                                          C.c_uint64, C.c_int, C.c_uint64, C.c_int,
                                          C.POINTER(C.c_int)]
            self._apply = f("apply_plan")
            self._apply.argtypes = [C.c_int, C.c_uint64, C.c_uint32, u32p, u64p, C.c_uint32, u64p,
                                    C.c_uint64, u64p]

    # ------------------------------------------------------------------ utils
    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._last_error().decode())

    def stream(self, seed: int, label: str, idx: int | None = None) -> int:
        if idx is None:
            return int(self._stream(seed, label.encode()))
        return int(self._stream_idx(seed, label.encode(), idx))

    def rng_draw(self, seed: int, count: int) -> np.ndarray:
        out = np.zeros(count, np.uint64)
        self._draw(seed, count, _p(out, u64p))
        return out

    def fht_mod(self, v, p):
        a = np.ascontiguousarray(np.asarray(v, dtype=np.uint64)).copy()
        self._check(self._fht_mod(_p(a, u64p), a.size, p))
        return a

    def batch_hash_kernel(self, t, l1, p):
        a = np.ascontiguousarray(np.asarray(t, dtype=np.uint64)).copy()
        self._check(self._bhk(_p(a, u64p), a.size, l1, p))
        return a

    # ----------------------------------------------------------------- family
    def build_family(self, dims, radius, seed, prime=(1 << 61) - 1, kind=-1, include_zero=False):
        mapping = np.zeros(dims, np.uint32)
        seeds = np.zeros(dims, np.uint64)
        k = C.c_int(0)
        self._check(self._build_family(dims, radius, kind, seed, prime, int(include_zero),
                                       _p(mapping, u32p), _p(seeds, u64p), C.byref(k)))
        return mapping, seeds, k.value

    def hash_batch(self, mapping, seeds, dims, radius, prime, rows, kind=None, threads=1,
                   reference_path=False):
        """Keys of every row, point-major uint64 [n, L]."""
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        n = rows.shape[0]
        L = (1 << (radius + 1)) - 1
        out = np.zeros((n, L), np.uint64)
        mapping = np.ascontiguousarray(mapping, np.uint32)
        seeds = np.ascontiguousarray(seeds, np.uint64)
        if self.p == "ref_":
            if kind is None:
                kind = 1 if dims <= (1 << (radius + 1)) else 0
            el = C.c_double(0)
            self._check(self._hash(dims, radius, kind, _p(mapping, u32p), _p(seeds, u64p), prime,
                                   _p(rows, u64p), n, _p(out, u64p), threads, int(reference_path),
                                   C.byref(el)))
            self.last_elapsed = el.value
        elif reference_path:
            self._check(self._hash_ref(_p(mapping, u32p), _p(seeds, u64p), dims, radius, prime,
                                       _p(rows, u64p), n, _p(out, u64p)))
        else:
            self._check(self._hash(_p(mapping, u32p), _p(seeds, u64p), dims, radius, prime,
                                   _p(rows, u64p), n, _p(out, u64p), threads))
        return out

    # ------------------------------------------------------------------- plan
    def make_plan(self, dims, radius, c, n, seed, override=None, budget=1 << 21) -> Plan:
        kind = C.c_int(0)
        t = C.c_uint32(0)
        ppr = C.c_uint32(0)
        perm = np.zeros(max(dims, 1), np.uint32)
        parts = np.zeros(2 * (radius + 1), np.uint64)
        ok, ot = (override if override is not None else (0, 1))
        self._check(self._make_plan(dims, radius, c, n, seed, int(override is not None), ok, ot,
                                    budget, C.byref(kind), C.byref(t), C.byref(ppr),
                                    _p(perm, u32p), _p(parts, u64p)))
        k = kind.value
        return Plan(k, t.value, ppr.value, perm[:dims] if k == 2 else np.zeros(0, np.uint32),
                    parts[: 2 * t.value].reshape(-1, 2) if k == 2 else np.zeros((0, 2), np.uint64))

    # ------------------------------------------------------------------ index
    def index_build(self, rows, dims, radius, plan_seed, index_seed, override=None, c=1.0,
                    prime=(1 << 61) - 1, include_zero=False, budget=1 << 21, threads=1):
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        n = rows.shape[0]
        code = C.c_int(0)
        ok, ot = (override if override is not None else (0, 1))
        if self.p == "ref_":
            el = C.c_double(0)
            h = self._index_build(_p(rows, u64p), n, dims, radius, plan_seed,
                                  int(override is not None), ok, ot, c, index_seed, prime,
                                  int(include_zero), budget, threads, C.byref(el), C.byref(code))
            self.last_elapsed = el.value
        else:
            h = self._index_build(_p(rows, u64p), n, dims, radius, plan_seed,
                                  int(override is not None), ok, ot, c, index_seed, prime,
                                  int(include_zero), budget, threads, C.byref(code))
        self._check(code.value)
        return OracleIndex(self, h, dims)

    # ----------------------------------------- classic (compiled reference only)
    def choose_k(self, dims, radius, tables, delta):
        out = C.c_uint32(0)
        self._check(self._choose_k(dims, radius, tables, float(delta), C.byref(out)))
        return int(out.value)

    def bitsample_family(self, dims, k, tables, seed, prime=(1 << 61) - 1):
        pos = np.zeros(tables * k, np.uint32)
        seeds = np.zeros(tables * k, np.uint64)
        self._check(self._bsf(dims, k, tables, seed, prime, _p(pos, u32p), _p(seeds, u64p)))
        return pos, seeds

    def hash_tables(self, dims, k, tables, positions, seeds, prime, rows, threads=1):
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        out = np.zeros((rows.shape[0], tables), np.uint64)
        self._check(self._hash_tables(dims, k, tables, _p(np.ascontiguousarray(positions, np.uint32), u32p),
                                      _p(np.ascontiguousarray(seeds, np.uint64), u64p), prime, _p(rows, u64p),
                                      rows.shape[0], _p(out, u64p), threads))
        return out

    def index_build_classic(self, rows, dims, radius, plan_seed, index_seed, prime=(1 << 61) - 1, c=1.0,
                            budget=1 << 21, delta=0.1, k_override=0, tables_override=0):
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        code = C.c_int(0)
        h = self._build_classic(_p(rows, u64p), rows.shape[0], dims, radius, plan_seed, c, index_seed, prime, budget,
                                delta, k_override, tables_override, C.byref(code))
        self._check(code.value)
        return OracleIndex(self, h, dims)

    def scan_truth(self, rows, qrows, dims, radius, threads=1) -> np.ndarray:
        """(query, point, distance) uint32 triples sorted by (query, point)."""
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        qrows = np.ascontiguousarray(qrows, dtype=np.uint64)
        ptr = u32p()
        cnt = C.c_uint64(0)
        self._check(self._scan(_p(rows, u64p), rows.shape[0], _p(qrows, u64p), qrows.shape[0],
                               dims, radius, threads, C.byref(ptr), C.byref(cnt)))
        n = cnt.value
        out = np.ctypeslib.as_array(ptr, shape=(max(n, 1) * 3,))[: 3 * n].copy().reshape(n, 3)
        self._free(ptr)
        return out


    # dataset containers and the distance histogram: the compiled reference only
    def dataset_save(self, path, rows, dims, text=False):
        """save_dataset / save_dataset_text (dataset.cpp:82-98)."""
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        self._check(self._ds_save(str(path).encode(), _p(rows, u64p), rows.shape[0], dims, int(text)))

    def dataset_load(self, path):
        """load_dataset (dataset.cpp:101-111) -> (rows [n, W] uint64, dims)."""
        n, d, ptr = C.c_uint64(0), C.c_uint64(0), u64p()
        self._check(self._ds_load(str(path).encode(), C.byref(n), C.byref(d), C.byref(ptr)))
        W = (d.value + 63) // 64
        out = np.ctypeslib.as_array(ptr, shape=(max(1, n.value * W),))[: n.value * W].copy().reshape(n.value, W)
        self._free(ptr)
        return out, d.value

    def run_experiment(self, rows, qrows, dims, truth, truth_radius, method, radius, c=1.0, override=None,
                       seed=0, repeats=1, fresh_seeds=True, prime=(1 << 61) - 1):
        """run_experiment (bench.cpp:64-158) -> rows [nq, 12] doubles: query_id, radius, collisions,
        candidates, found, true_near, precision, recall, time_s1_us, time_s2_us, time_s3_us, 0."""
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        qrows = np.ascontiguousarray(qrows, dtype=np.uint64)
        truth = np.ascontiguousarray(truth, dtype=np.uint32).reshape(-1, 3)
        out = np.zeros((qrows.shape[0], 12), np.float64)
        csv = C.c_char_p()
        kind, t = (-1, 0) if override is None else override
        self._check(self._run_exp(_p(rows, u64p), rows.shape[0], _p(qrows, u64p), qrows.shape[0], dims,
                                  _p(truth, u32p), truth.shape[0], truth_radius, method.encode(), radius, c,
                                  kind, t, seed, repeats, int(fresh_seeds), prime,
                                  out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(csv)))
        return out

    def distance_histogram(self, rows, qrows, dims, sample_per_query=0, seed=0):
        """distance_histogram (workload.cpp:133-151): counts[dims + 1]."""
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        qrows = np.ascontiguousarray(qrows, dtype=np.uint64)
        counts = np.zeros(dims + 1, np.uint64)
        self._check(self._hist(_p(rows, u64p), rows.shape[0], _p(qrows, u64p), qrows.shape[0], dims,
                               sample_per_query, seed, _p(counts, u64p)))
        return counts


class OracleIndex:
    def __init__(self, orc: Oracle, handle, dims):
        self.o = orc
        self.h = handle
        self.dims = dims

    def __del__(self):
        if getattr(self, "h", None):
            self.o._index_destroy(self.h)
            self.h = None

    @property
    def table_count(self):
        return int(self.o._table_count(self.h))

    def family(self, p):
        dims = C.c_uint64(0)
        r = C.c_uint32(0)
        k = C.c_int(0)
        self.o._check(self.o._index_family(self.h, p, None, None, C.byref(dims), C.byref(r), C.byref(k)))
        mapping = np.zeros(dims.value, np.uint32)
        seeds = np.zeros(dims.value, np.uint64)
        self.o._check(self.o._index_family(self.h, p, _p(mapping, u32p), _p(seeds, u64p),
                                           C.byref(dims), C.byref(r), C.byref(k)))
        return mapping, seeds, int(r.value), int(k.value)

    def query(self, qrows, radius, threads=1):
        """query_r_nn per row -> (counters [nq,3], offsets [nq+1], ids)."""
        qrows = np.ascontiguousarray(qrows, dtype=np.uint64)
        nq = qrows.shape[0]
        counters = np.zeros((nq, 3), np.uint64)
        offsets = np.zeros(nq + 1, np.uint64)
        ptr = u32p()
        args = [self.h, _p(qrows, u64p), nq, radius, threads, _p(counters, u64p),
                _p(offsets, u64p), C.byref(ptr)]
        if self.o.p == "ref_":
            el = C.c_double(0)
            args.append(C.byref(el))
            self.o._check(self.o._index_query(*args))
            self.last_elapsed = el.value
        else:
            self.o._check(self.o._index_query(*args))
        total = int(offsets[-1])
        ids = np.ctypeslib.as_array(ptr, shape=(max(total, 1),))[:total].copy()
        self.o._free(ptr)
        return counters, offsets, ids

    def query_c(self, qrows, radius, budget=None, threads=1):
        """query_c_r_nn per row (compiled reference only) -> (counters [nq, 3], best [nq, 2] id/distance,
        UINT32_MAX when nothing was retrieved)."""
        qrows = np.ascontiguousarray(qrows, dtype=np.uint64)
        nq = qrows.shape[0]
        counters = np.zeros((nq, 3), np.uint64)
        best = np.zeros((nq, 2), np.uint32)
        self.o._check(self.o._index_query_c(self.h, _p(qrows, u64p), nq, radius, -1 if budget is None else budget,
                                            threads, _p(counters, u64p), _p(best, u32p)))
        return counters, best


_cache: dict = {}


def port() -> Oracle:
    if "port" not in _cache:
        _cache["port"] = Oracle(PORT_SO, "orc_")
    return _cache["port"]


def reference() -> Oracle:
    if "ref" not in _cache:
        _cache["ref"] = Oracle(REF_SO, "ref_")
    return _cache["ref"]


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def best() -> Oracle:
    """The compiled reference when it was built (it travels with the snapshot),
    else the C restatement."""
    return reference() if reference_available() else port()
