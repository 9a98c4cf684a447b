"""Reference-shaped Python API over the C-ABI (include/fclsh_gpu.h).

Names, argument meaning and error classes follow the reference library
(/root/reference/proj/include/fclsh/*.hpp) so that parity tests read like its
own tests:

    build_covering_family / make_covering_family   covering.hpp:55-66
    hash_batch  (hash_batch_into for many rows)    covering.hpp:83-84
    make_plan / PlanOverride / PlanKind            transform.hpp:24-59
    build_index / IndexSet.query_r_nn              index.hpp:70-79
    UsageError / DataError / ResourceError         errors.hpp:8-29

An ``Rng&`` argument of the reference is passed as the Rng's seed (its
sub-streams depend on the seed only, rng.cpp:31-37). Rows are numpy uint64
arrays [n, ceil(d/64)] (BitVector word layout) or, for the device entry
points, CUDA tensors of dtype int64/uint64 with the same layout.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import _native as N

M61 = (1 << 61) - 1  # kMersenne61, modmath.hpp:10
M31 = (1 << 31) - 1
DEFAULT_TABLE_BUDGET = 1 << 21  # transform.hpp:52


class FclshError(RuntimeError):
    code = 1


class UsageError(FclshError):
    code = 2


class DataError(FclshError):
    code = 3


class ResourceError(FclshError):
    code = 4


class CudaRuntimeError(FclshError):
    code = 5


_ERRORS = {2: UsageError, 3: DataError, 4: ResourceError, 5: CudaRuntimeError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = N.lib().fclsh_last_error().decode()
        raise _ERRORS.get(rc, FclshError)(msg)


def _release(obj, destroy: str) -> None:
    """__del__ helper: frees the handle; a no-op once interpreter shutdown has
    torn the module globals down."""
    h = getattr(obj, "_h", None)
    if h is None or not h.value or N is None:
        return
    try:
        getattr(N.lib(), destroy)(h)
    except (AttributeError, TypeError):  # pragma: no cover - shutdown order
        return
    obj._h = None


class _ResultBlock:
    """Owns one fclsh_result (a pinned block); frees it when collected."""

    def __init__(self, rp):
        self._rp = rp

    def __del__(self, _lib=N.lib):
        try:
            _lib().fclsh_result_free(self._rp)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def words_for(dims: int) -> int:
    return (dims + 63) // 64


def rng_stream(seed: int, label: str, index: int | None = None) -> int:
    """Seed of Rng(seed).stream(label[, index]) (rng.cpp:31-37)."""
    L = N.lib()
    if index is None:
        return int(L.fclsh_rng_stream(seed, label.encode()))
    return int(L.fclsh_rng_stream_index(seed, label.encode(), index))


def device_count() -> int:
    c = C.c_int(0)
    _check(N.lib().fclsh_device_count(C.byref(c)))
    return c.value


class ConstructionKind(enum.IntEnum):  # covering.hpp:21
    general = 0
    specific = 1


class PlanKind(enum.IntEnum):  # transform.hpp:24
    identity = 0
    replicate = 1
    partition = 2


@dataclass
class PlanOverride:  # transform.hpp:46-50
    kind: PlanKind
    t: int = 1


_CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: torch's default stream, passed so the C side joins it


def _stream_ptr(stream):
    """cudaStream_t for the C-ABI. A torch stream (None = torch's current one)
    is passed as itself; torch's default stream (handle 0) as cudaStreamLegacy,
    because NULL means the library's own stream, which is not ordered with the
    caller's work. A plain int is passed through unchanged."""
    if isinstance(stream, int):
        return C.c_void_p(stream)
    if stream is None:
        try:
            import torch
            stream = torch.cuda.current_stream()
        except Exception:  # pragma: no cover - torch is always present in this image
            return C.c_void_p(0)
    return C.c_void_p(stream.cuda_stream or _CUDA_STREAM_LEGACY)


class CoveringFamily:
    """CoveringFamily (covering.hpp:34-43), host-built, device-uploaded lazily."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        info = N.FamilyInfo()
        _check(N.lib().fclsh_family_info_get(self._h, C.byref(info)))
        self.dims = int(info.dims)
        self.radius = int(info.radius)
        self.kind = ConstructionKind(info.kind)
        self.prime = int(info.prime)
        self._mapping = None
        self._seeds = None

    def __del__(self, _free=_release):  # bound at definition: module globals may be gone at exit
        _free(self, "fclsh_family_destroy")

    def code_order(self) -> int:
        return 1 << (self.radius + 1)

    def table_count(self) -> int:
        return self.code_order() - 1

    def _export(self):
        m = np.zeros(self.dims, np.uint32)
        s = np.zeros(self.dims, np.uint64)
        _check(N.lib().fclsh_family_export(self._h, _ptr(m, N.u32p), _ptr(s, N.u64p)))
        self._mapping, self._seeds = m, s

    @property
    def mapping(self) -> np.ndarray:
        if self._mapping is None:
            self._export()
        return self._mapping

    @property
    def seeds(self) -> np.ndarray:
        if self._seeds is None:
            self._export()
        return self._seeds


def build_covering_family(dims: int, radius: int, rng_seed: int, kind: ConstructionKind | None = None,
                          prime: int = M61, include_zero_column: bool = False) -> CoveringFamily:
    """build_covering_family (covering.cpp:40-80); kind None derives it from the widths."""
    h = C.c_void_p()
    k = -1 if kind is None else int(kind)
    _check(N.lib().fclsh_family_build(dims, radius, k, rng_seed, prime, int(include_zero_column), C.byref(h)))
    return CoveringFamily(h)


def make_covering_family(dims: int, radius: int, kind: ConstructionKind, mapping, seeds,
                         prime: int = M61) -> CoveringFamily:
    """make_covering_family (covering.cpp:84-111)."""
    m = np.ascontiguousarray(mapping, dtype=np.uint32)
    s = _u64(seeds)
    if m.size != dims or s.size != dims:
        raise UsageError("covering family: mapping/seeds must have one entry per dimension")
    h = C.c_void_p()
    _check(N.lib().fclsh_family_make(dims, radius, int(kind), _ptr(m, N.u32p), _ptr(s, N.u64p), prime,
                                     C.byref(h)))
    return CoveringFamily(h)


def hash_batch(family: CoveringFamily, rows, device: int = 0, key_bytes: int | None = None) -> np.ndarray:
    """hash_batch_into for every row: keys [n, L] (point-major), via the GPU.

    key_bytes defaults to 4 when the prime fits 32 bits (uint32 result), else 8.
    """
    r = _u64(rows)
    if r.ndim == 1:
        r = r.reshape(1, -1)
    n, w = r.shape
    kb = key_bytes or (4 if family.prime < (1 << 32) else 8)
    out = np.zeros((n, family.table_count()), np.uint32 if kb == 4 else np.uint64)
    _check(N.lib().fclsh_hash_batch_host(family._h, _ptr(r, N.u64p), n, w, out.ctypes.data_as(C.c_void_p), kb,
                                         device))
    return out


def hash_batch_device(family: CoveringFamily, rows, keys, *, layout: int = 0, key_stride: int | None = None,
                      device: int | None = None, stream=None) -> None:
    """Device-buffer hash: rows / keys are CUDA tensors (rows int64/uint64 [n, W];
    keys int32/uint32 or int64/uint64). layout 0 = table-major, 1 = point-major."""
    n = rows.shape[0]
    kb = keys.element_size()
    stride = key_stride if key_stride is not None else (n if layout == 0 else family.table_count())
    dev = rows.device.index if device is None else device
    _check(N.lib().fclsh_hash_batch(family._h, C.c_void_p(rows.data_ptr()), n, rows.shape[1],
                                    C.c_void_p(keys.data_ptr()), kb, stride, layout, dev or 0, _stream_ptr(stream)))


# ----------------------------------------------------------- classic family

@dataclass
class BitSampleFamily:  # classic.hpp:15-27
    dims: int
    k: int
    tables: int
    prime: int
    positions: np.ndarray  # uint32 [tables * k]
    seeds: np.ndarray      # uint64 [tables * k]

    def table_count(self) -> int:
        return self.tables


def choose_k(dims: int, radius: int, tables: int, delta: float) -> int:
    """choose_k (classic.cpp:10-23)."""
    out = C.c_uint32(0)
    _check(N.lib().fclsh_choose_k(dims, radius, tables, float(delta), C.byref(out)))
    return int(out.value)


def build_bit_sample_family(dims: int, k: int, tables: int, rng_seed: int, prime: int = M61) -> BitSampleFamily:
    """build_bit_sample_family (classic.cpp:25-46)."""
    pos = np.zeros(max(1, tables * k), np.uint32)
    seeds = np.zeros(max(1, tables * k), np.uint64)
    _check(N.lib().fclsh_bitsample_family_build(dims, k, tables, rng_seed, prime, _ptr(pos, N.u32p),
                                                _ptr(seeds, N.u64p)))
    return BitSampleFamily(dims, k, tables, prime, pos[:tables * k], seeds[:tables * k])


def hash_tables(family: BitSampleFamily, rows, device: int = 0) -> np.ndarray:
    """hash_tables_into (classic.cpp:48-63) for every row, on the device -> uint64 [n, tables]."""
    r = _u64(rows)
    if r.ndim == 1:
        r = r.reshape(1, -1)
    n = r.shape[0]
    if n and r.shape[1] != words_for(family.dims):
        raise UsageError("hash: vector width does not match the family")
    out = np.zeros((n, family.tables), np.uint64)
    pos = np.ascontiguousarray(family.positions, np.uint32)
    sd = np.ascontiguousarray(family.seeds, np.uint64)
    _check(N.lib().fclsh_hash_tables_batch(family.dims, family.k, family.tables, _ptr(pos, N.u32p),
                                           _ptr(sd, N.u64p), family.prime, _ptr(r, N.u64p), n, _ptr(out, N.u64p),
                                           device))
    return out


class PreprocessPlan:
    """PreprocessPlan (transform.hpp:26-44)."""

    def __init__(self, handle):
        self._h = handle
        info = N.PlanInfo()
        _check(N.lib().fclsh_plan_info_get(self._h, C.byref(info)))
        self.kind = PlanKind(info.kind)
        self.dims = int(info.dims)
        self.radius = int(info.radius)
        self.t = int(info.t)
        self.per_part_radius = int(info.per_part_radius)
        self._part_count = int(info.part_count)
        self._table_count = int(info.table_count)
        perm = np.zeros(max(self.dims, 1), np.uint32)
        parts = np.zeros(2 * max(self.t, 1), np.uint64)
        _check(N.lib().fclsh_plan_export(self._h, _ptr(perm, N.u32p), _ptr(parts, N.u64p)))
        if self.kind == PlanKind.partition:
            self.permutation = perm[: self.dims]
            self.parts = [(int(parts[2 * i]), int(parts[2 * i + 1])) for i in range(self.t)]
        else:
            self.permutation = np.zeros(0, np.uint32)
            self.parts = []

    def __del__(self, _free=_release):  # bound at definition: module globals may be gone at exit
        _free(self, "fclsh_plan_destroy")

    def part_count(self) -> int:
        return self._part_count

    def part_dims(self, p: int) -> int:
        if self.kind == PlanKind.partition:
            b, e = self.parts[p]
            return e - b
        return self.dims * self.t if self.kind == PlanKind.replicate else self.dims

    def table_count(self) -> int:  # plan_table_count (transform.cpp:155-158)
        return self._table_count


def make_plan(dims: int, radius: int, c: float, n: int, rng_seed: int, force: PlanOverride | None = None,
              table_budget: int = DEFAULT_TABLE_BUDGET) -> PreprocessPlan:
    """make_plan (transform.cpp:32-113)."""
    h = C.c_void_p()
    fp = None
    if force is not None:
        fp = C.byref(N.PlanOverride(int(force.kind), int(force.t)))
    _check(N.lib().fclsh_plan_make(dims, radius, float(c), n, rng_seed, fp, table_budget, C.byref(h)))
    return PreprocessPlan(h)


@dataclass
class QueryResults:
    """query_r_nn over a batch: per-query ids (ascending) + QueryReport counters."""
    query: np.ndarray       # uint32 [total]
    id: np.ndarray          # uint32 [total]
    distance: np.ndarray    # uint32 [total]
    offsets: np.ndarray     # uint64 [nq+1]
    collisions: np.ndarray  # uint64 [nq]
    candidates: np.ndarray  # uint64 [nq]
    found: np.ndarray       # uint64 [nq]
    time_s1_ms: float = 0.0
    time_s2_ms: float = 0.0
    time_s3_ms: float = 0.0

    def ids(self, q: int) -> np.ndarray:
        return self.id[int(self.offsets[q]): int(self.offsets[q + 1])]

    def triples(self) -> np.ndarray:
        return np.stack([self.query, self.id, self.distance], axis=1)


@dataclass
class DeviceQueryResults:
    nq: int
    total: int
    d_query: int
    d_id: int
    d_distance: int
    d_offsets: int
    d_collisions: int
    d_candidates: int
    d_found: int
    raw: object = None  # the C struct (for fclsh_result_copy_device)

    def copy_to(self, triples=None, offsets=None, counters=None, device: int = 0, stream=None) -> None:
        """Copy into caller CUDA tensors: triples int32 [3, cap], offsets int64 [nq+1],
        counters int64 [3, nq] (collisions, candidates, found)."""
        cap = triples.shape[1] if triples is not None else 0
        _check(N.lib().fclsh_result_copy_device(
            C.byref(self.raw), C.c_void_p(triples.data_ptr() if triples is not None else 0), cap,
            C.c_void_p(offsets.data_ptr() if offsets is not None else 0),
            C.c_void_p(counters.data_ptr() if counters is not None else 0), device, _stream_ptr(stream)))


def merge_shards(offsets_all, triples_all, out_triples, out_offsets, device: int = 0, stream=None) -> None:
    """fclsh_merge_shards over CUDA tensors: offsets_all int64 [world, nq+1],
    triples_all int32 [world, 3, cap] -> out_triples int32 [3, out_cap],
    out_offsets int64 [nq+1] (rank runs in rank order = (query, id) order)."""
    world, nq1 = offsets_all.shape
    _check(N.lib().fclsh_merge_shards(world, nq1 - 1, C.c_void_p(offsets_all.data_ptr()),
                                      C.c_void_p(triples_all.data_ptr()), triples_all.shape[2],
                                      C.c_void_p(out_triples.data_ptr()), out_triples.shape[1],
                                      C.c_void_p(out_offsets.data_ptr()), device, _stream_ptr(stream)))


def _results_from(rp, nq: int) -> "QueryResults":
    """QueryResults viewing the pinned block behind an fclsh_result (freed
    with fclsh_result_free once the last view is gone)."""
    owner = _ResultBlock(rp)
    r = rp.contents
    tot = int(r.total)

    def arr(p, cnt, ct, dt):
        if cnt == 0:
            return np.zeros(0, dt)
        buf = (ct * cnt).from_address(C.cast(p, C.c_void_p).value)
        buf._owner = owner
        return np.frombuffer(buf, dtype=dt)

    return QueryResults(arr(r.query, tot, C.c_uint32, np.uint32), arr(r.id, tot, C.c_uint32, np.uint32),
                        arr(r.distance, tot, C.c_uint32, np.uint32),
                        arr(r.offsets, nq + 1, C.c_uint64, np.uint64),
                        arr(r.collisions, nq, C.c_uint64, np.uint64),
                        arr(r.candidates, nq, C.c_uint64, np.uint64), arr(r.found, nq, C.c_uint64, np.uint64),
                        float(r.time_hash_ms), float(r.time_probe_ms), float(r.time_verify_ms))


class IndexSet:
    """IndexSet (index.hpp:42-52) resident on one GPU."""

    def __init__(self, handle, plan: PreprocessPlan):
        self._h = handle
        self.plan = plan
        info = N.IndexInfo()
        _check(N.lib().fclsh_index_info_get(self._h, C.byref(info)))
        self.n = int(info.n)
        self.dims = int(info.dims)
        self.radius = int(info.radius)
        self._tables = int(info.table_count)
        self._entries = int(info.entry_count)
        self.directory_bits = int(info.directory_bits)
        self.device_bytes = int(info.device_bytes)
        self.build_ms = float(info.build_ms)
        self.layout = {1: "csr", 2: "buckets"}.get(int(info.layout), "?")
        self.buckets_per_table = int(info.buckets_per_table)
        self.method = {0: "covering", 2: "classic"}.get(int(info.method), "?")
        self.classic_k = int(info.classic_k)

    def bit_sample_family(self) -> BitSampleFamily:
        """A classic index's family (positions / seeds [tables * k])."""
        k, T = self.classic_k, self._tables
        pos = np.zeros(max(1, T * k), np.uint32)
        seeds = np.zeros(max(1, T * k), np.uint64)
        _check(N.lib().fclsh_index_bitsample_family(self._h, _ptr(pos, N.u32p), _ptr(seeds, N.u64p)))
        return BitSampleFamily(self.dims, k, T, self._prime, pos[:T * k], seeds[:T * k])

    def __del__(self, _free=_release):  # bound at definition: module globals may be gone at exit
        _free(self, "fclsh_index_destroy")

    def table_count(self) -> int:
        return self._tables

    def entry_count(self) -> int:
        return self._entries

    def family(self, part: int) -> CoveringFamily:
        h = C.c_void_p()
        _check(N.lib().fclsh_index_family(self._h, part, C.byref(h)))
        return CoveringFamily(h)

    def query_r_nn(self, q_rows, radius: int) -> QueryResults:
        """query_r_nn (index.cpp:157-188) for every row of q_rows (host)."""
        q = _u64(q_rows)
        if q.ndim == 1:
            q = q.reshape(1, -1)
        nq = q.shape[0]
        if nq and q.shape[1] != words_for(self.dims):
            raise UsageError("query width does not match the index")
        rp = C.POINTER(N.Result)()
        _check(N.lib().fclsh_query(self._h, _ptr(q, N.u64p), nq, radius, C.byref(rp)))
        return _results_from(rp, nq)

    STAGES = ("hash", "fused", "dense", "found_scan", "compact", "overflow")

    def stage_ms(self) -> dict:
        """Device time per stage of the last query (CUDA events)."""
        buf = (C.c_double * 8)()
        k = N.lib().fclsh_query_stage_ms(self._h, buf, 8)
        if k < 0:
            _check(-k)
        return {name: float(buf[i]) for i, name in enumerate(self.STAGES[:k])}

    def query_c_r_nn(self, q_rows, radius: int, posting_budget: int | None = None):
        """query_c_r_nn (index.cpp:190-235) per row -> (counters [nq, 3] collisions/candidates/found,
        best_id [nq], best_distance [nq]); -1 where nothing was retrieved."""
        q = _u64(q_rows)
        if q.ndim == 1:
            q = q.reshape(1, -1)
        nq = q.shape[0]
        if nq and q.shape[1] != words_for(self.dims):
            raise UsageError("query width does not match the index")
        counters = np.zeros((nq, 3), np.uint64)
        best = np.zeros((nq, 2), np.uint32)
        _check(N.lib().fclsh_query_c_r_nn(self._h, _ptr(q, N.u64p), nq, radius,
                                          -1 if posting_budget is None else posting_budget,
                                          _ptr(counters, N.u64p), _ptr(best, N.u32p)))
        none = best[:, 0] == 0xFFFFFFFF
        bid = np.where(none, -1, best[:, 0].astype(np.int64))
        bd = np.where(none, -1, best[:, 1].astype(np.int64))
        return counters, bid, bd

    def stage_timing(self, enable: bool = True) -> None:
        """Per-stage CUDA events on the next batches (off by default: ~4 us each)."""
        _check(N.lib().fclsh_query_stage_timing(self._h, int(bool(enable))))

    def batch_ms(self) -> float:
        """Device time of the last batch (hash .. compaction)."""
        ms = C.c_double(0)
        _check(N.lib().fclsh_query_batch_ms(self._h, C.byref(ms)))
        return float(ms.value)

    def path_counts(self) -> dict:
        """Queries of the last batch served by the dense (CTA) kernel and by the general path."""
        dense, general = C.c_uint64(0), C.c_uint64(0)
        _check(N.lib().fclsh_query_path_counts(self._h, C.byref(dense), C.byref(general)))
        return {"dense": int(dense.value), "general": int(general.value)}

    def query_device(self, q_rows, radius: int, stream=None) -> DeviceQueryResults:
        """Device rows in (CUDA tensor), device results out (index-owned buffers)."""
        out = N.DeviceResult()
        _check(N.lib().fclsh_query_device(self._h, C.c_void_p(q_rows.data_ptr()), q_rows.shape[0], radius,
                                          _stream_ptr(stream), C.byref(out)))
        return DeviceQueryResults(int(out.nq), int(out.total), out.d_query or 0, out.d_id or 0,
                                  out.d_distance or 0, out.d_offsets or 0, out.d_collisions or 0,
                                  out.d_candidates or 0, out.d_found or 0, out)


METHODS = {"covering": 0, "covering_batch": 0, "covering_reference": 0, "classic": 2}


def build_index(data_rows, radius: int, plan: PreprocessPlan, rng_seed: int, *, prime: int = M61,
                include_zero_column: bool = False, table_budget: int = DEFAULT_TABLE_BUDGET, device: int = 0,
                id_offset: int = 0, directory_bits: int = 0, dims: int | None = None,
                layout: str = "auto", method: str = "covering", delta: float = 0.1,
                k_override: int | None = None, tables_override: int | None = None) -> IndexSet:
    """build_index(data, method, radius, plan, Rng(rng_seed), IndexOptions{...})
    (index.cpp:49-119). data_rows: numpy uint64 [n, W] or a CUDA tensor.
    layout: "auto" | "csr" | "buckets" (device table layout; same results).
    method: "covering" (covering_batch; covering_reference builds the same
    buckets) or "classic" (bit sampling, identity plan; delta / k_override /
    tables_override as IndexOptions, index.hpp:29-32)."""
    if method not in METHODS:
        raise UsageError(f"unknown method '{method}'")
    opt = N.IndexOptions()
    N.lib().fclsh_index_options_default(C.byref(opt))
    opt.method = METHODS[method]
    opt.delta = float(delta)
    opt.k_override = k_override or 0
    opt.tables_override = tables_override or 0
    opt.prime = prime
    opt.include_zero_column = int(include_zero_column)
    opt.table_budget = table_budget
    opt.device = device
    opt.id_offset = id_offset
    opt.directory_bits = directory_bits
    opt.layout = {"auto": 0, "csr": 1, "buckets": 2}[layout]
    d = plan.dims if dims is None else dims
    h = C.c_void_p()
    if hasattr(data_rows, "data_ptr"):  # torch tensor on the device
        n = data_rows.shape[0] if data_rows.ndim == 2 else 0
        ptr = C.c_void_p(data_rows.data_ptr())
        on_dev = 1 if data_rows.is_cuda else 0
        if not data_rows.is_cuda:
            data_rows = data_rows.contiguous()
        _check(N.lib().fclsh_index_build(ptr, on_dev, n, d, radius, plan._h, rng_seed, C.byref(opt), C.byref(h)))
    else:
        r = _u64(data_rows)
        n = r.shape[0] if r.ndim == 2 else 0
        if n and r.shape[1] != words_for(d):
            raise UsageError("index: dataset width does not match the plan")
        _check(N.lib().fclsh_index_build(r.ctypes.data_as(C.c_void_p), 0, n, d, radius, plan._h, rng_seed,
                                         C.byref(opt), C.byref(h)))
    ix = IndexSet(h, plan)
    ix._prime = prime
    return ix


def launch_count() -> int:
    return int(N.lib().fclsh_launch_count())


def launch_count_reset() -> None:
    N.lib().fclsh_launch_count_reset()


# ------------------------------------------------------------------ cluster

CLUSTER_ID_BYTES = 128


def cluster_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0 of a multi-process cluster sends it to the others)."""
    buf = C.create_string_buffer(CLUSTER_ID_BYTES)
    _check(N.lib().fclsh_cluster_unique_id(buf))
    return buf.raw


class Cluster:
    """Point-sharded index over the GPUs of one box (fclsh_cluster_*).

    Cluster(devices=[0, 1, ...], shards_per_rank=k): this process drives every
    GPU. Cluster(rank=r, world=w, device=d, uid=...): one process per GPU
    (uid from cluster_unique_id() on rank 0). build / query_r_nn are
    collective: every process calls them. query_r_nn returns the merged result
    on rank 0 and None elsewhere."""

    def __init__(self, devices=None, shards_per_rank: int = 1, *, rank: int | None = None, world: int = 1,
                 device: int = 0, uid: bytes | None = None):
        h = C.c_void_p()
        if rank is None:
            devs = list(devices) if devices is not None else [0]
            arr = (C.c_int * len(devs))(*devs)
            _check(N.lib().fclsh_cluster_create(arr, len(devs), shards_per_rank, C.byref(h)))
        else:
            _check(N.lib().fclsh_cluster_create_rank(uid, world, rank, device, shards_per_rank, C.byref(h)))
        self._h = h
        self.plan = None

    def __del__(self, _free=_release):
        _free(self, "fclsh_cluster_destroy")

    def info(self) -> dict:
        i = N.ClusterInfo()
        _check(N.lib().fclsh_cluster_info_get(self._h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in N.ClusterInfo._fields_}

    @property
    def is_root(self) -> bool:
        return self.info()["rank"] == 0

    def build(self, data_rows, radius: int, plan: PreprocessPlan, rng_seed: int, *, n: int | None = None,
              local_rows: bool = False, prime: int = M61, include_zero_column: bool = False,
              table_budget: int = DEFAULT_TABLE_BUDGET, id_offset: int = 0, directory_bits: int = 0,
              layout: str = "auto", method: str = "covering", delta: float = 0.1, k_override: int | None = None,
              tables_override: int | None = None) -> "Cluster":
        """build_index over the sharded points. data_rows: all n points (numpy
        or a CUDA tensor), or with local_rows=True only this process's range
        (n = the global count)."""
        opt = N.IndexOptions()
        N.lib().fclsh_index_options_default(C.byref(opt))
        opt.prime = prime
        opt.include_zero_column = int(include_zero_column)
        opt.table_budget = table_budget
        opt.id_offset = id_offset
        opt.directory_bits = directory_bits
        opt.layout = {"auto": 0, "csr": 1, "buckets": 2}[layout]
        if method not in METHODS:
            raise UsageError(f"unknown method '{method}'")
        opt.method = METHODS[method]
        opt.delta = float(delta)
        opt.k_override = k_override or 0
        opt.tables_override = tables_override or 0
        if hasattr(data_rows, "data_ptr"):
            ptr, on_dev, rows_n = C.c_void_p(data_rows.data_ptr()), int(data_rows.is_cuda), data_rows.shape[0]
        else:
            data_rows = _u64(data_rows)
            if data_rows.ndim != 2 or data_rows.shape[1] != words_for(plan.dims):
                raise UsageError("index: dataset width does not match the plan")
            ptr, on_dev, rows_n = data_rows.ctypes.data_as(C.c_void_p), 0, data_rows.shape[0]
        total = rows_n if n is None else n
        _check(N.lib().fclsh_cluster_build(self._h, ptr, on_dev, 1 if local_rows else 0, total, plan.dims, radius,
                                           plan._h, rng_seed, C.byref(opt)))
        self.plan = plan
        self._keep = data_rows  # (the library copied the rows; kept only for symmetry with IndexSet)
        return self

    def query_r_nn(self, q_rows, radius: int, nq: int | None = None):
        """query_r_nn over every shard (host rows in on rank 0, where the merged
        result comes back; other ranks pass None and the batch size `nq` and
        get None)."""
        if q_rows is None:
            nq = nq or 0
            ptr = N.u64p()
        else:
            q = _u64(q_rows)
            if q.ndim == 1:
                q = q.reshape(1, -1)
            nq = q.shape[0]
            ptr = _ptr(q, N.u64p)
        rp = C.POINTER(N.Result)()
        _check(N.lib().fclsh_cluster_query(self._h, ptr, nq, radius, C.byref(rp)))
        if not rp:
            return None
        return _results_from(rp, nq)

    def stage_timing(self, enable: bool = True) -> None:
        """Per-stage CUDA events in every local shard (off by default)."""
        _check(N.lib().fclsh_cluster_stage_timing(self._h, int(bool(enable))))

    def stage_ms(self, shard: int = 0) -> dict:
        """Stage times (ms) of the last batch on local shard `shard`."""
        buf = (C.c_double * 8)()
        k = N.lib().fclsh_cluster_stage_ms(self._h, shard, buf, 8)
        if k < 0:
            _check(-k)
        return {name: float(buf[i]) for i, name in enumerate(IndexSet.STAGES[:k])}

    def path_counts(self, shard: int = 0) -> dict:
        dense, general = C.c_uint64(0), C.c_uint64(0)
        rc = N.lib().fclsh_cluster_path_counts(self._h, shard, C.byref(dense), C.byref(general))
        if rc < 0:
            _check(-rc)
        return {"dense": int(dense.value), "general": int(general.value)}

    def query_device(self, q_rows, radius: int, stream=None, nq: int | None = None):
        """Device rows in (CUDA tensor on rank 0's GPU), device results on rank 0
        (DeviceQueryResults; nq == 0 and null pointers on other ranks)."""
        out = N.DeviceResult()
        ptr = C.c_void_p(q_rows.data_ptr()) if q_rows is not None else C.c_void_p(0)
        count = q_rows.shape[0] if q_rows is not None else (nq or 0)
        _check(N.lib().fclsh_cluster_query_device(self._h, ptr, count, radius, _stream_ptr(stream), C.byref(out)))
        return DeviceQueryResults(int(out.nq), int(out.total), out.d_query or 0, out.d_id or 0,
                                  out.d_distance or 0, out.d_offsets or 0, out.d_collisions or 0,
                                  out.d_candidates or 0, out.d_found or 0, out)


# ------------------------------------------------------------------ workloads

def gen_bernoulli(seed: int, n: int, dims: int, threads: int = 8, row0: int = 0) -> np.ndarray:
    """Rows [row0, row0 + n) of the seeded Bernoulli(0.5) stream."""
    out = np.zeros((n, words_for(dims)), np.uint64)
    _check(N.lib().fclsh_gen_bernoulli(seed, row0, n, dims, _ptr(out, N.u64p), threads))
    return out


def gen_clustered(seed: int, centres: int, n: int, dims: int, flip_p: float, threads: int = 8,
                  row0: int = 0) -> np.ndarray:
    """Rows [row0, row0 + n) of the seeded clustered stream."""
    out = np.zeros((n, words_for(dims)), np.uint64)
    _check(N.lib().fclsh_gen_clustered(seed, centres, row0, n, dims, float(flip_p), _ptr(out, N.u64p), threads))
    return out


def gen_planted(seed: int, data: np.ndarray, dims: int, nq: int, kmax: int):
    d = _u64(data)
    out = np.zeros((nq, words_for(dims)), np.uint64)
    src = np.zeros(nq, np.uint32)
    _check(N.lib().fclsh_gen_planted(seed, _ptr(d, N.u64p), d.shape[0], dims, nq, kmax, _ptr(out, N.u64p),
                                     _ptr(src, N.u32p)))
    return out, src


# ----------------------------------------------------------------- datasets

DATASET_FCL1 = 1
DATASET_TEXT = 2


class Dataset:
    """load_dataset (dataset.cpp:101-111): rows [n, ceil(dims/64)] uint64 in
    the engine's row layout, held in pinned host memory when a GPU is usable."""

    def __init__(self, handle):
        self._h = handle
        n, d, fmt, rows = C.c_uint64(0), C.c_uint64(0), C.c_int32(0), N.u64p()
        _check(N.lib().fclsh_dataset_info_get(self._h, C.byref(n), C.byref(d), C.byref(fmt), C.byref(rows)))
        self.n, self.dims, self.format = int(n.value), int(d.value), int(fmt.value)
        W = words_for(self.dims)
        if self.n:
            buf = (C.c_uint64 * (self.n * W)).from_address(C.cast(rows, C.c_void_p).value)
            buf._owner = self  # the handle outlives every view of its rows
            self.rows = np.frombuffer(buf, dtype=np.uint64).reshape(self.n, W)
        else:
            self.rows = np.zeros((0, W), np.uint64)

    def __del__(self, _free=_release):
        _free(self, "fclsh_dataset_destroy")

    def __len__(self) -> int:
        return self.n

    def upload(self, device: int = 0, stream=None):
        """The rows as a CUDA int64 tensor [n, W] (pinned host -> device copy)."""
        import torch
        out = torch.empty((self.n, words_for(self.dims)), dtype=torch.int64, device=f"cuda:{device}")
        _check(N.lib().fclsh_dataset_upload(self._h, C.c_void_p(out.data_ptr()), device, _stream_ptr(stream)))
        return out


def load_dataset(path: str) -> Dataset:
    """load_dataset (dataset.hpp:30): FCL1 (magic sniffed) or text."""
    h = C.c_void_p()
    _check(N.lib().fclsh_dataset_load(str(path).encode(), C.byref(h)))
    return Dataset(h)


def save_dataset(path: str, rows, dims: int, text: bool = False) -> None:
    """save_dataset / save_dataset_text (dataset.hpp:22-27) of rows [n, ceil(dims/64)]."""
    r = _u64(rows)
    if r.ndim == 1:
        r = r.reshape(-1, words_for(dims))
    _check(N.lib().fclsh_dataset_save(str(path).encode(), _ptr(r, N.u64p), r.shape[0], dims,
                                      DATASET_TEXT if text else DATASET_FCL1))


# -------------------------------------------------------------- linear scan

class LinearScan:
    """scan_truth (workload.cpp:56-71) and distance_histogram
    (workload.cpp:133-151) on device rows (CUDA int64/uint64 tensors [n, W])."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(N.lib().fclsh_scan_create(device, C.byref(h)))
        self._h = h
        self.device = device

    def __del__(self, _free=_release):
        _free(self, "fclsh_scan_destroy")

    def scan_truth(self, rows, q_rows, dims: int, radius: int, stream=None) -> DeviceQueryResults:
        out = N.DeviceResult()
        _check(N.lib().fclsh_scan_truth(self._h, C.c_void_p(rows.data_ptr()), rows.shape[0],
                                        C.c_void_p(q_rows.data_ptr()), q_rows.shape[0], dims, radius,
                                        _stream_ptr(stream), C.byref(out)))
        return DeviceQueryResults(int(out.nq), int(out.total), out.d_query or 0, out.d_id or 0,
                                  out.d_distance or 0, out.d_offsets or 0, 0, 0, 0, raw=out)

    def triples(self, rows, q_rows, dims: int, radius: int) -> np.ndarray:
        """(query, point, distance) uint32 triples ordered by (query, point), on the host."""
        import torch
        r = self.scan_truth(rows, q_rows, dims, radius)
        tri = torch.zeros((3, max(r.total, 1)), dtype=torch.int32, device=f"cuda:{self.device}")
        r.copy_to(tri, None, None, device=self.device)
        torch.cuda.synchronize(self.device)
        return tri[:, :r.total].cpu().numpy().view(np.uint32).T.copy()

    def distance_histogram(self, rows, q_rows, dims: int, sample_per_query: int = 0, seed: int = 0,
                           stream=None) -> np.ndarray:
        counts = np.zeros(dims + 1, np.uint64)
        _check(N.lib().fclsh_distance_histogram(self._h, C.c_void_p(rows.data_ptr()), rows.shape[0],
                                                C.c_void_p(q_rows.data_ptr()), q_rows.shape[0], dims,
                                                sample_per_query, seed, _stream_ptr(stream), _ptr(counts, N.u64p)))
        return counts
