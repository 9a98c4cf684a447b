"""ctypes binding of libfclsh_b200.so (the C-ABI in include/fclsh_gpu.h).

The shared library is built in-tree (``make -C paper_1602_02620_b200``, or
``__graft_entry__.build()``) and loaded from ``paper_1602_02620_b200/lib``.
There is no fallback: if the library is missing every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FCLSH_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("FCLSH_LIB") or os.path.join(HERE, "lib", "libfclsh_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "fclsh_gpu.h")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class FamilyInfo(C.Structure):
    _fields_ = [("dims", C.c_uint64), ("radius", C.c_uint32), ("kind", C.c_int32),
                ("prime", C.c_uint64), ("tables", C.c_uint64)]


class PlanOverride(C.Structure):
    _fields_ = [("kind", C.c_int32), ("t", C.c_uint32)]


class PlanInfo(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dims", C.c_uint64), ("radius", C.c_uint32), ("t", C.c_uint32),
                ("per_part_radius", C.c_uint32), ("part_count", C.c_uint32), ("table_count", C.c_uint64)]


class IndexOptions(C.Structure):
    _fields_ = [("prime", C.c_uint64), ("include_zero_column", C.c_int32), ("table_budget", C.c_uint64),
                ("device", C.c_int32), ("id_offset", C.c_uint64), ("directory_bits", C.c_int32),
                ("layout", C.c_int32), ("method", C.c_int32), ("delta", C.c_double), ("k_override", C.c_uint32),
                ("tables_override", C.c_uint64)]


class IndexInfo(C.Structure):
    _fields_ = [("n", C.c_uint64), ("dims", C.c_uint64), ("radius", C.c_uint32), ("table_count", C.c_uint64),
                ("entry_count", C.c_uint64), ("directory_bits", C.c_uint32), ("device_bytes", C.c_uint64),
                ("build_ms", C.c_double), ("layout", C.c_int32), ("buckets_per_table", C.c_uint64),
                ("method", C.c_int32), ("classic_k", C.c_uint32)]


class Result(C.Structure):
    _fields_ = [("nq", C.c_uint64), ("total", C.c_uint64), ("query", u32p), ("id", u32p), ("distance", u32p),
                ("offsets", u64p), ("collisions", u64p), ("candidates", u64p), ("found", u64p),
                ("time_hash_ms", C.c_double), ("time_probe_ms", C.c_double), ("time_verify_ms", C.c_double)]


class DeviceResult(C.Structure):
    _fields_ = [("nq", C.c_uint64), ("total", C.c_uint64), ("d_query", vp), ("d_id", vp), ("d_distance", vp),
                ("d_offsets", vp), ("d_collisions", vp), ("d_candidates", vp), ("d_found", vp)]


class ClusterInfo(C.Structure):
    _fields_ = [("world", C.c_uint32), ("rank", C.c_uint32), ("local_ranks", C.c_uint32),
                ("shards_per_rank", C.c_uint32), ("total_shards", C.c_uint32), ("device", C.c_int32),
                ("uses_nccl", C.c_int32), ("n", C.c_uint64), ("dims", C.c_uint64), ("radius", C.c_uint32),
                ("table_count", C.c_uint64), ("local_points", C.c_uint64), ("local_entry_count", C.c_uint64),
                ("local_device_bytes", C.c_uint64), ("local_bucket_shards", C.c_uint32), ("build_ms", C.c_double)]


# name -> (restype, argtypes)
SIGNATURES = {
    "fclsh_version": (C.c_char_p, []),
    "fclsh_last_error": (C.c_char_p, []),
    "fclsh_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "fclsh_rng_stream": (C.c_uint64, [C.c_uint64, C.c_char_p]),
    "fclsh_rng_stream_index": (C.c_uint64, [C.c_uint64, C.c_char_p, C.c_uint64]),
    "fclsh_family_build": (C.c_int, [C.c_uint64, C.c_uint32, C.c_int32, C.c_uint64, C.c_uint64, C.c_int,
                                     C.POINTER(vp)]),
    "fclsh_family_make": (C.c_int, [C.c_uint64, C.c_uint32, C.c_int32, u32p, u64p, C.c_uint64, C.POINTER(vp)]),
    "fclsh_family_info_get": (C.c_int, [vp, C.POINTER(FamilyInfo)]),
    "fclsh_family_export": (C.c_int, [vp, u32p, u64p]),
    "fclsh_family_destroy": (None, [vp]),
    "fclsh_hash_batch": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, vp, C.c_uint32, C.c_uint64, C.c_int32, C.c_int,
                                   vp]),
    "fclsh_hash_batch_host": (C.c_int, [vp, u64p, C.c_uint64, C.c_uint32, vp, C.c_uint32, C.c_int]),
    "fclsh_plan_make": (C.c_int, [C.c_uint64, C.c_uint32, C.c_double, C.c_uint64, C.c_uint64,
                                  C.POINTER(PlanOverride), C.c_uint64, C.POINTER(vp)]),
    "fclsh_plan_info_get": (C.c_int, [vp, C.POINTER(PlanInfo)]),
    "fclsh_plan_export": (C.c_int, [vp, u32p, u64p]),
    "fclsh_plan_destroy": (None, [vp]),
    "fclsh_index_options_default": (None, [C.POINTER(IndexOptions)]),
    "fclsh_index_build": (C.c_int, [vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, vp, C.c_uint64,
                                    C.POINTER(IndexOptions), C.POINTER(vp)]),
    "fclsh_index_info_get": (C.c_int, [vp, C.POINTER(IndexInfo)]),
    "fclsh_index_family": (C.c_int, [vp, C.c_uint32, C.POINTER(vp)]),
    "fclsh_index_destroy": (None, [vp]),
    "fclsh_index_bitsample_family": (C.c_int, [vp, u32p, u64p]),
    "fclsh_choose_k": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_double, u32p]),
    "fclsh_bitsample_family_build": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, u32p,
                                               u64p]),
    "fclsh_hash_tables_batch": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint64, u32p, u64p, C.c_uint64, u64p,
                                          C.c_uint64, u64p, C.c_int]),
    "fclsh_query": (C.c_int, [vp, u64p, C.c_uint64, C.c_uint32, C.POINTER(C.POINTER(Result))]),
    "fclsh_result_free": (None, [C.POINTER(Result)]),
    "fclsh_query_c_r_nn": (C.c_int, [vp, u64p, C.c_uint64, C.c_uint32, C.c_int64, u64p, u32p]),
    "fclsh_query_device": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, vp, C.POINTER(DeviceResult)]),
    "fclsh_query_stage_ms": (C.c_int, [vp, C.POINTER(C.c_double), C.c_int]),
    "fclsh_query_path_counts": (C.c_int, [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "fclsh_query_stage_timing": (C.c_int, [vp, C.c_int]),
    "fclsh_query_batch_ms": (C.c_int, [vp, C.POINTER(C.c_double)]),
    "fclsh_result_copy_device": (C.c_int, [C.POINTER(DeviceResult), vp, C.c_uint64, vp, vp, C.c_int, vp]),
    "fclsh_merge_shards": (C.c_int, [C.c_uint32, C.c_uint64, vp, vp, C.c_uint64, vp, C.c_uint64, vp, C.c_int, vp]),
    "fclsh_dataset_load": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "fclsh_dataset_info_get": (C.c_int, [vp, u64p, u64p, C.POINTER(C.c_int32), C.POINTER(u64p)]),
    "fclsh_dataset_upload": (C.c_int, [vp, vp, C.c_int, vp]),
    "fclsh_dataset_destroy": (None, [vp]),
    "fclsh_dataset_save": (C.c_int, [C.c_char_p, u64p, C.c_uint64, C.c_uint64, C.c_int32]),
    "fclsh_scan_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "fclsh_scan_destroy": (None, [vp]),
    "fclsh_scan_truth": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, C.c_uint64, C.c_uint32, vp,
                                   C.POINTER(DeviceResult)]),
    "fclsh_distance_histogram": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                           vp, u64p]),
    "fclsh_cluster_unique_id": (C.c_int, [C.c_char_p]),
    "fclsh_cluster_create": (C.c_int, [C.POINTER(C.c_int), C.c_uint32, C.c_uint32, C.POINTER(vp)]),
    "fclsh_cluster_create_rank": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint32, C.c_int, C.c_uint32,
                                            C.POINTER(vp)]),
    "fclsh_cluster_build": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, vp, C.c_uint64,
                                      C.POINTER(IndexOptions)]),
    "fclsh_cluster_info_get": (C.c_int, [vp, C.POINTER(ClusterInfo)]),
    "fclsh_cluster_query": (C.c_int, [vp, u64p, C.c_uint64, C.c_uint32, C.POINTER(C.POINTER(Result))]),
    "fclsh_cluster_query_device": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, vp, C.POINTER(DeviceResult)]),
    "fclsh_cluster_stage_timing": (C.c_int, [vp, C.c_int]),
    "fclsh_cluster_stage_ms": (C.c_int, [vp, C.c_uint32, C.POINTER(C.c_double), C.c_int]),
    "fclsh_cluster_path_counts": (C.c_int, [vp, C.c_uint32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "fclsh_cluster_destroy": (None, [vp]),
    "fclsh_launch_count": (C.c_uint64, []),
    "fclsh_launch_count_reset": (None, []),
    "fclsh_gen_bernoulli": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u64p, C.c_int]),
    "fclsh_gen_clustered": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, u64p,
                                      C.c_int]),
    "fclsh_gen_planted": (C.c_int, [C.c_uint64, u64p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, u64p, u32p]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded library (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libfclsh_b200.so not found at {LIB_PATH}; build it with "
                "`make -C paper_1602_02620_b200` or __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
