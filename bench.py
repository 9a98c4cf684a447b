#!/usr/bin/env python
"""fcLSH B200 bench -- one JSON line on rank 0.

Headline workload (the largest single-GPU BASELINE config, configs[2],
"cfg3"): n = 4,000,000 points of d = 512 i.i.d. Bernoulli(0.5) bits, r = 12
through the pigeonhole partition (t = 2 blocks of 256 bits, per-block radius
6, 2 x 127 tables), exact verify on all 512 bits, P = 2^31 - 1 (32-bit keys);
10,000 planted queries. A step is one query_r_nn pass over the whole batch
(hash -> probe -> dedup -> verify -> (query, id, distance) triples in
(query, id) order + per-query counters). `value` = queries/s with the query
rows already in HBM; `e2e` = the same through the host C-ABI call
fclsh_cluster_query (host rows in, host result block out, every copy inside
the timed region). Everything runs through fclsh_cluster, the multi-GPU
path: at N = 1 it is one shard on one GPU.

Also on the line: cfg1 / cfg2 / cfg4 with the same step definition (value,
e2e, roofline, CPU baseline, parity), the cfg5 hash microbenchmark (8M x
1024-bit rows, r = 10, 2047 keys per row in 1M-row chunks) with the CPU
hash_batch_into baseline at 1 and all host threads, and the device / CPU
index build times.

Scaling: cfg1-3 and cfg5 are weak (every GPU holds the config's n points of
one global dataset of N x n points; queries broadcast), cfg4 is strong (the
10M points in one shard per GPU: at N = 8 the BASELINE's 8-way sharding).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU)
  python bench.py --gpus N ...                        (one process, N GPUs)
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
RANDOM_READ_CEILING = 41.5e9  # random 32-B reads/s, tools/rand_bench.cu (profiles/r01/rand_bench.txt)
METRIC = "queries/sec at 100% recall (result set == oracle)"
HEADLINE = 3
M31 = (1 << 31) - 1


def measured_traffic(prefix: str, config: str | None = None):
    """DRAM bytes per launch (read + write) of a kernel from the newest
    committed ncu --set full capture (profiles/rNN/traffic.json), or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "traffic.json")), reverse=True):
        try:
            for k, v in json.load(open(path)).items():
                if k.startswith(prefix) and (config is None or v.get("config") == config):
                    return int(v["dram_read_bytes"] + v["dram_write_bytes"]), os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None, None


def hbm_peak():
    try:
        p = json.load(open(PEAKS_PATH))
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed regions (the
    same fields as the nvidia-smi clocks line of the profiling recipe), via
    NVML polled every ~1 ms from a thread: the timed regions here are
    milliseconds long, too short for nvidia-smi's 200-ms loop. Reentrant:
    `with sampler:` around each timed region accumulates samples."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, device: int):
        self.device = device
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, const in self.REASONS.items():
                    if r & getattr(nv, const):
                        self.reasons.add(name)
            except Exception:
                return
            time.sleep(0.001)

    def __enter__(self):
        if self.nv is not None:
            self._stop.clear()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._t is not None:
            self._stop.set()
            self._t.join()
            self._t = None

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "NVML, 1 ms polling during the timed regions"}


# --------------------------------------------------------------------- context

class Ctx:
    """Where this process sits: `G` GPUs in all, either one process per GPU
    (torchrun: WORLD_SIZE = G) or one process driving all G (--gpus G)."""

    def __init__(self, args):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.torchrun = self.world > 1
        self.G = self.world if self.torchrun else args.gpus
        if self.torchrun:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            # the data path is the library's own NCCL communicator; this group
            # only carries the NCCL id, barriers and the max-over-ranks timing
            dist.init_process_group("gloo")
            self.dist = dist
        self.devices = [self.local] if self.torchrun else list(range(self.G))
        if self.G > 1:  # NCCL's own log names every rank it connects (the library's communicator)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
        self.root = self.rank == 0

    def check_gpus(self, args):
        if self.torchrun and args.gpus != self.world:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={self.world}")
        import torch
        have = torch.cuda.device_count()
        need = (self.local + 1) if self.torchrun else self.G
        if have < need:
            raise SystemExit(f"bench.py: --gpus {args.gpus} needs {need} visible GPU(s), found {have}")

    def barrier(self):
        if self.torchrun:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if not self.torchrun:
            return x
        import torch
        t = torch.tensor([float(x)], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.torchrun:
            self.dist.destroy_process_group()


def host_threads():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


# ------------------------------------------------------------- reference arm

def run_reference_arm(args, ctx):
    """--impl reference: the reference's own CPU query_r_nn (oracle/_ref: the
    reference sources compiled unmodified; else the C restatement, labelled
    "port") on all host threads, on the headline config's full query batch per
    step. Inputs come from the oracle's generators (byte-identical to the
    product's): this process never maps libfclsh_b200.so."""
    if not ctx.root:
        return
    from oracle import oracle as O
    from oracle.workloads import OracleBackend, load_configs
    C = load_configs()
    ob = OracleBackend()
    cfg = C.CONFIGS[HEADLINE]
    if args.ref_scale:  # (tests: the same path on a small slice)
        cfg = cfg.scaled(args.ref_scale, queries=min(cfg.planted, args.ref_scale // 10))
    threads = host_threads()
    data = C.make_data(cfg, threads, backend=ob)
    queries = C.make_queries(cfg, data, threads, backend=ob)
    orc = O.best()
    t0 = time.perf_counter()
    oi = orc.index_build(data, cfg.dims, cfg.radius, cfg.plan_seed(ob), cfg.index_seed(ob),
                         override=(cfg.plan_kind, cfg.t), prime=M31, threads=threads)
    build_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        oi.query(queries[:500], cfg.radius, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oi.query(queries, cfg.radius, threads=threads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    nq = queries.shape[0]
    value = nq * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": ctx.G,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded Bernoulli(0.5) rows; planted queries), generated by the oracle",
        "config": config_block(cfg, ctx.G, "weak", 1),
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": threads, "kind": orc.kind,
                         "sample": f"the full {nq}-query cfg3 batch per step against the full {cfg.n}-point reference "
                                   f"index (query_r_nn, PostingTable binary search; index built once in "
                                   f"{build_s:.1f} s on {threads} threads, untimed)"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "build_s": build_s,
        "product_library_mapped": product_mapped(),
        "product_package_imported": "paper_1602_02620_b200" in sys.modules,
    }
    print(json.dumps(line), flush=True)


def product_mapped() -> bool:
    """Whether libfclsh_b200.so is mapped into this process (/proc/self/maps)."""
    try:
        with open("/proc/self/maps") as f:
            return "libfclsh_b200" in f.read()
    except OSError:
        return False


def config_block(cfg, G, scaling, spr):
    n_total = cfg.n * G if scaling == "weak" else cfg.n
    return {"workload": f"{cfg.name} (BASELINE configs[{cfg.id - 1}])", "n_total": n_total,
            "n_per_gpu": n_total // G, "d": cfg.dims, "r": cfg.radius, "plan": cfg.plan_name, "t": cfg.t,
            "tables": cfg.tables, "queries": cfg.queries, "prime": "2^31-1 (32-bit keys)",
            "data_dist": cfg.data, "shards": G * spr, "shards_per_gpu": spr,
            "l2": "flushed between steps (256 MiB device write on every GPU)",
            "parallelism": f"points sharded over {G} GPU(s) x {spr} shard(s), queries broadcast (NCCL), results "
                           f"gathered to rank 0 (NCCL)" if G * spr > 1 else "1 GPU, 1 shard"}


# ------------------------------------------------------------------ our arm

class Flush:
    """256 MiB device writes (> the 126 MB L2) on every GPU of this process."""

    def __init__(self, devices):
        import torch
        self.bufs = [torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=f"cuda:{d}") for d in devices]

    def __call__(self):
        for b in self.bufs:
            b.zero_()


def sync_all(devices):
    import torch
    for d in devices:
        torch.cuda.synchronize(d)


def make_cluster(ctx, spr):
    from paper_1602_02620_b200 import cluster as CL
    from paper_1602_02620_b200 import fclsh as F
    if ctx.torchrun:
        return CL.rank_cluster(spr, device=ctx.local)
    return F.Cluster(ctx.devices, spr)


def cluster_inputs(ctx, cfg, scaling, spr, threads):
    """(rows to build from, local_rows flag, n_total, global data on the root or
    None, queries on the root or None)."""
    from paper_1602_02620_b200 import cluster as CL
    from paper_1602_02620_b200.configs import make_data, make_queries
    G = ctx.G
    n_total = cfg.n * G if scaling == "weak" else cfg.n
    if not ctx.torchrun:
        data = make_data(cfg, threads, n=n_total)
        return data, False, n_total, data, make_queries(cfg, data, threads)
    S = G * spr
    b = CL.shard_range(n_total, S, ctx.rank * spr)[0]
    e = CL.shard_range(n_total, S, ctx.rank * spr + spr - 1)[1]
    if ctx.root:
        data = make_data(cfg, threads, n=n_total)
        return data[b:e], True, n_total, data, make_queries(cfg, data, threads)
    return make_data(cfg, threads, row0=b, n=e - b), True, n_total, None, None


def run_config(ctx, cfg, scaling, spr, args, flush, stream, clocks, hbm, peak_src, threads, headline=False):
    """One config through fclsh_cluster: build, device-resident timed steps,
    stage pass (roofline), e2e host calls, parity and the CPU baseline."""
    import ctypes as C

    import torch

    from paper_1602_02620_b200 import _native as N
    from paper_1602_02620_b200 import fclsh as F
    dev0 = ctx.devices[0]
    rows, local_rows, n_total, gdata, q = cluster_inputs(ctx, cfg, scaling, spr, threads)
    nq = cfg.queries
    plan = F.make_plan(cfg.dims, cfg.radius, 1.0, n_total, cfg.plan_seed(), cfg.override())
    cl = make_cluster(ctx, spr)
    t0 = time.perf_counter()
    cl.build(rows, cfg.radius, plan, cfg.index_seed(), n=n_total, local_rows=local_rows, prime=F.M31)
    build_wall = time.perf_counter() - t0
    info = cl.info()
    del rows
    q_dev = torch.from_numpy(q.view(np.int64)).to(f"cuda:{dev0}") if ctx.root else None

    def step():
        return cl.query_device(q_dev, cfg.radius, stream, nq=nq)

    for _ in range(max(3, args.warmup)):  # warm-up steps run like the timed ones: L2 flushed first
        flush()                           # (the first step after a first flush measured ~190 us, tools/step_variance.py)
        step()
    sync_all(ctx.devices)
    F.launch_count_reset()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ctx.barrier()
    sync_all(ctx.devices)
    with clocks:
        for k in range(args.steps):
            flush()
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
            sync_all(ctx.devices)
    launches = F.launch_count()
    total_ms = ctx.max(sum(a.elapsed_time(b) for a, b in ev))
    value = nq * args.steps / (total_ms / 1e3)

    # per-stage device times of local shard 0 (stage events cost ~4 us each,
    # so the timed steps above run without them)
    cl.stage_timing(True)
    try:
        for _ in range(2):  # the stage-timed shape is captured as its own graph
            step()
        stages = []
        for _ in range(max(5, args.steps)):
            flush()
            with clocks:
                step()
                sync_all(ctx.devices)
            stages.append(cl.stage_ms(0))
    finally:
        cl.stage_timing(False)
    stage_avg = {k: statistics.mean(s[k] for s in stages) for k in stages[0]}
    paths = cl.path_counts(0)

    # e2e: the host C-ABI call (rows in host memory, result block out), collective
    L = N.lib()
    rp = C.POINTER(N.Result)()
    if ctx.root:
        pinned = torch.from_numpy(q.view(np.int64)).pin_memory()
        qptr = pinned.numpy().view(np.uint64).ctypes.data_as(N.u64p)
    else:
        qptr = N.u64p()
    res = None

    def host_call():
        rc = L.fclsh_cluster_query(cl._h, qptr, nq, cfg.radius, C.byref(rp))
        if rc != 0:
            raise RuntimeError(L.fclsh_last_error().decode())
        tot = int(rp.contents.total) if rp else 0
        if rp:
            L.fclsh_result_free(rp)
        return tot

    for _ in range(3):
        host_call()
    e2e_steps = max(30, args.steps)
    e2e_t = []
    total = 0
    gc.collect()
    gc.disable()
    try:
        for _ in range(e2e_steps):
            flush()
            sync_all(ctx.devices)
            ctx.barrier()
            t0 = time.perf_counter()
            total = host_call()
            e2e_t.append(time.perf_counter() - t0)
    finally:
        gc.enable()
    e2e_sum = ctx.max(sum(e2e_t))
    res = cl.query_r_nn(q if ctx.root else None, cfg.radius, nq=nq)
    W = cfg.words
    e2e = {"value": nq * e2e_steps / e2e_sum, "unit": "queries/s", "h2d_bytes_per_step": int(nq * W * 8),
           "d2h_bytes_per_step": int(total * 12 + (4 * nq + 1) * 8), "steps": e2e_steps,
           "ms_per_step_median": 1e3 * statistics.median(e2e_t),
           "api": "fclsh_cluster_query + fclsh_result_free (include/fclsh_gpu.h): pinned host rows in, host result "
                  "block out (query, id, distance, offsets, counters)",
           "note": "L2 flushed before every call; Python gc paused during the timed calls"}
    replay = None
    if headline and args.replay > 1:
        replay = replay_batch(ctx, cl, q, q_dev, cfg, args, flush, stream, clocks)
    out = {"value": value, "unit": "queries/s", "ms_per_step": total_ms / args.steps, "e2e": e2e, "replay": replay,
           "gpu_launches": launches, "stages_ms_shard0": stage_avg, "query_paths_shard0": paths,
           "build": {"device_ms": info["build_ms"], "wall_s": build_wall, "layout_bucket_shards_local":
                     info["local_bucket_shards"], "device_bytes_local": info["local_device_bytes"]},
           "config": config_block(cfg, ctx.G, scaling, spr)}
    if not ctx.root:
        del cl
        return out, None
    coll = res.collisions.astype(np.float64)
    cand = res.candidates.astype(np.float64)
    found = res.found.astype(np.float64)
    out["counters"] = {"collisions_mean": float(coll.mean()), "candidates_mean": float(cand.mean()),
                       "found_mean": float(found.mean()), "found_total": int(found.sum())}
    # roofline of the dominant query kernel on shard 0: algorithmic bytes per
    # launch = per (query, table) its key (4 B) + one random 32-B bucket sector
    # (CSR: a directory and an entry sector), per distinct candidate one row (at
    # least one 32-B sector), per result 8 B, the query rows once; the counters
    # are the whole cluster's, divided over its S equal shards
    S = ctx.G * spr
    T_ = cfg.tables
    R = max(32, cfg.dims // 8)
    layout_b = info["local_bucket_shards"] > 0
    probe = 32 if layout_b else 64
    kern_stage = "dense" if T_ > 600 else "fused"
    kern_name = "k_query_dense" if kern_stage == "dense" else "k_query_warp"
    algo = (nq * T_ * (4 + probe) + cand.sum() * R + found.sum() * 8) / S + nq * cfg.dims / 8
    # the query kernel hashes its own queries (index.cu fused_fe: narrow keys,
    # per-part radius 4..7, <= 600 tables): the hash pass's bytes are its too
    fused_hash = 4 <= cfg.per_part_radius <= 7 and T_ <= 600 and kern_stage == "fused"
    if fused_hash:
        algo += nq * T_ * 4
    dur = stage_avg[kern_stage]
    ach = algo / (dur / 1e3) / 1e9
    traffic, tsrc = measured_traffic(kern_name, cfg.name)
    out["roofline"] = {"bound": "hbm", "kernel": kern_name, "achieved": ach, "peak": hbm, "unit": "GB/s",
                       "frac": ach / hbm, "traffic": traffic, "traffic_source": tsrc, "peak_source": peak_src,
                       "algorithmic_bytes_per_launch": algo, "duration_ms": dur, "hash_fused": fused_hash,
                       "bytes_note": "per (query, table) the key + one random 32-B bucket sector (also for the "
                                     "probes the L2 key filter skips), per distinct candidate max(32, d/8) B, per "
                                     "result 8 B, query rows once; traffic = measured DRAM bytes per launch (ncu)"}
    # the same kernel against the GPU's random-access ceiling: its random
    # 32-B reads (a bucket per probe, CSR: a directory and a cell entry; a row
    # per distinct candidate; the query rows) per second over the ~41.5 G
    # reads/s tools/rand_bench.cu measured (profiles/r01/rand_bench.txt), the
    # bound this kernel meets before the HBM byte bound
    reads = (nq * T_ * (1 if layout_b else 2) + cand.sum()) / S + nq
    out["roofline"]["random_reads_per_launch"] = reads
    out["roofline"]["random_reads_per_s"] = reads / (dur / 1e3)
    out["roofline"]["vs_random_read_ceiling"] = reads / (dur / 1e3) / RANDOM_READ_CEILING
    out["roofline"]["random_read_ceiling"] = {"value": RANDOM_READ_CEILING, "unit": "reads/s",
                                              "source": "tools/rand_bench.cu (profiles/r01/rand_bench.txt: 41-43 G "
                                                        "random 32-B reads/s on this B200); probes the key filter "
                                                        "skips are counted as reads"}
    hash_ms = stage_avg.get("hash", 0)
    if hash_ms > 0:
        hb = nq * (cfg.dims / 8 + T_ * 4)
        out["hash_stage_roofline"] = {"ms": hash_ms, "GB/s": hb / (hash_ms / 1e3) / 1e9,
                                      "frac": hb / (hash_ms / 1e3) / 1e9 / hbm}
    del cl
    torch.cuda.empty_cache()
    return out, (gdata, q, res, n_total)


def replay_batch(ctx, cl, q, q_dev, cfg, args, flush, stream, clocks):
    """the probe + dedup + verify pass on a replayed batch of
    >= 1M queries (the config's batch tiled args.replay times), where the
    per-batch fixed costs and the kernel's tail vanish: queries/s, the query
    kernel's sustained time per query and its roofline, and the verify-pass
    bytes (candidates x (4 + max(32, d/8)) + found x 12 + the query rows)."""
    import torch
    R = args.replay
    nq = cfg.queries * R
    qr = q_dev.repeat(R, 1) if ctx.root else None
    res = None
    for _ in range(2):
        res = cl.query_device(qr, cfg.radius, stream, nq=nq)
    sync_all(ctx.devices)
    ms = []
    for _ in range(3):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with clocks:
            a.record(stream)
            res = cl.query_device(qr, cfg.radius, stream, nq=nq)
            b.record(stream)
            sync_all(ctx.devices)
        ms.append(a.elapsed_time(b))
    step = ctx.max(statistics.median(ms))
    cl.stage_timing(True)
    try:
        cl.query_device(qr, cfg.radius, stream, nq=nq)
        sync_all(ctx.devices)
        cl.query_device(qr, cfg.radius, stream, nq=nq)
        sync_all(ctx.devices)
        st = cl.stage_ms(0)
    finally:
        cl.stage_timing(False)
    out = {"queries": nq, "replay_factor": R, "ms": step, "queries_per_s": nq / (step / 1e3), "stages_ms_shard0": st}
    if ctx.root and res is not None and res.nq:
        counts = torch.empty((3, nq), dtype=torch.int64, device=f"cuda:{ctx.devices[0]}")
        res.copy_to(None, None, counts, device=ctx.devices[0], stream=stream)
        sync_all(ctx.devices)
        cand = float(counts[1].sum().item())
        found = float(counts[2].sum().item())
        R_ = max(32, cfg.dims // 8)
        T_ = cfg.tables
        kern = "fused" if T_ <= 600 else "dense"
        dur = st[kern] + (st["hash"] if st.get("hash", 0) > 0 and kern == "fused" else 0)
        algo = nq * T_ * (4 + 32) + cand * R_ + found * 8 + nq * cfg.dims / 8
        if 4 <= cfg.per_part_radius <= 7 and T_ <= 600:  # hash fused into the kernel: its key writes too
            algo += nq * T_ * 4
        verify = cand * (4 + R_) + found * 12 + nq * cfg.dims / 8
        reads = nq * T_ + cand + nq  # bucket layout (the replayed configs' shard layout)
        out.update({"random_reads_per_s": reads / (dur / 1e3),
                    "vs_random_read_ceiling": reads / (dur / 1e3) / RANDOM_READ_CEILING})
        out.update({"kernel_ms": dur, "kernel_us_per_query": 1e3 * dur / nq,
                    "roofline_frac": algo / (dur / 1e3) / 1e9 / hbm_peak()[0], "algorithmic_bytes": algo,
                    "verify_bytes": verify, "verify_share_of_algorithmic_bytes": verify / algo,
                    "note": "the verify (candidate rows gathered with 256-bit loads, XOR + popcount) is fused into "
                            "the probe kernel, so it has no launch of its own to time: its bytes are this share of "
                            "the kernel's algorithmic bytes, and roofline_frac covers both; kernel_ms includes the "
                            "hash stage when it runs separately"})
    del qr
    torch.cuda.empty_cache()
    return out


def parity_and_cpu(ctx, cfg, gdata, q, res, n_total, threads, args, out, scaling):
    """Parity of the timed batch (N = 1: ids, offsets and every counter vs the
    reference's query_r_nn; cfg4 and N > 1: triples vs the GPU linear scan,
    itself pinned to scan_truth) and the reference CPU baseline (N = 1)."""
    from paper_1602_02620_b200 import fclsh as F
    nq = q.shape[0]
    cpu = None
    parity = None
    if ctx.G == 1 and cfg.id != 4 and not args.no_cpu:
        from oracle import oracle as O
        orc = O.best()
        t0 = time.perf_counter()
        oi = orc.index_build(gdata, cfg.dims, cfg.radius, cfg.plan_seed(), cfg.index_seed(),
                             override=(cfg.plan_kind, cfg.t), prime=M31, threads=threads)
        build_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        counters, offsets, ids = oi.query(q, cfg.radius, threads=threads)
        qps = nq / (time.perf_counter() - t0)
        s1 = min(nq, 500 if cfg.id != 1 else nq)
        t0 = time.perf_counter()
        oi.query(q[:s1], cfg.radius, threads=1)
        qps1 = s1 / (time.perf_counter() - t0)
        parity = bool((np.stack([res.collisions, res.candidates, res.found], 1) == counters).all()
                      and (res.offsets == offsets).all() and (res.id == ids).all())
        cpu = {"value": qps, "unit": "queries/s", "cores": threads, "kind": orc.kind,
               "sample": f"all {nq} {cfg.name} queries vs the full {cfg.n}-point reference index (query_r_nn on "
                         f"{threads} threads; index built in {build_s:.1f} s, untimed)",
               "T1": {"value": qps1, "cores": 1, "sample": f"the first {s1} queries, 1 thread"},
               "build_s": build_s, "build_threads": threads}
        del oi
    elif ctx.G == 1 and cfg.id == 4 and not args.no_cpu:
        # the reference index of all 10M clustered points needs ~163 GB of host
        # RAM: one 1.25M-point shard (1/8 of the points, the full query batch)
        from oracle import oracle as O
        from paper_1602_02620_b200 import cluster as CL
        orc = O.best()
        b, e = CL.shard_range(n_total, cfg.shards, 0)
        t0 = time.perf_counter()
        oi = orc.index_build(gdata[b:e], cfg.dims, cfg.radius, cfg.plan_seed(), cfg.index_seed(),
                             override=(cfg.plan_kind, cfg.t), prime=M31, threads=threads)
        build_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        oi.query(q, cfg.radius, threads=threads)
        shard_s = time.perf_counter() - t0
        cpu = {"value": nq / (shard_s * cfg.shards), "unit": "queries/s", "cores": threads, "kind": orc.kind,
               "sample": f"all {nq} queries against shard 0 of 8 ({e - b} points) on {threads} threads in "
                         f"{shard_s:.2f} s, x 8 shards (one index over all 10M points needs ~163 GB of host "
                         f"RAM); shard index built in {build_s:.1f} s, untimed",
               "build_s_shard": build_s}
        del oi
    if parity is None and ctx.root:
        # triples (ids and distances) vs the GPU linear scan over every point
        import torch
        dev = f"cuda:{ctx.devices[0]}"
        sc = F.LinearScan(ctx.devices[0])
        truth = sc.triples(torch.from_numpy(gdata.view(np.int64)).to(dev), torch.from_numpy(q.view(np.int64)).to(dev),
                           cfg.dims, cfg.radius)
        del sc
        torch.cuda.empty_cache()
        parity = bool(truth.shape == res.triples().shape and (truth == res.triples()).all())
        out["parity_kind"] = "triples vs GPU linear scan (scan_truth restated, pinned in tests)"
    else:
        out["parity_kind"] = "ids, offsets, collisions, candidates, found vs the reference query_r_nn"
    out["parity_vs_reference"] = parity
    out["cpu_baseline"] = cpu


def bench_hash(ctx, args, hbm, peak_src, flush, stream, threads, clocks):
    """cfg5: 8M x 1024-bit rows per GPU (weak), r = 10 -> 2047 keys per row,
    point-major in 1M-row chunks; step = all chunks. Algorithmic bytes = rows
    read once + every key written once = n * (d/8 + L*4)."""
    import torch

    from paper_1602_02620_b200 import fclsh as F
    from paper_1602_02620_b200.configs import CONFIGS
    cfg5 = CONFIGS[5]
    n = args.hash_points
    chunk = min(1_000_000, n)
    dev = ctx.devices[0]
    rows = F.gen_bernoulli(cfg5.root(), n, cfg5.dims, threads, row0=ctx.rank * n)
    fam = F.build_covering_family(cfg5.dims, cfg5.radius, cfg5.index_seed(), prime=F.M31)
    L = fam.table_count()
    d_rows = torch.from_numpy(rows.view(np.int64)).to(f"cuda:{dev}")
    keys = torch.empty((chunk, L), dtype=torch.int32, device=f"cuda:{dev}")

    def step():
        for c0 in range(0, n, chunk):
            m = min(chunk, n - c0)
            F.hash_batch_device(fam, d_rows[c0:c0 + m], keys, layout=1, key_stride=L, stream=stream)

    for _ in range(max(3, args.warmup)):
        flush()
        step()
    torch.cuda.synchronize(dev)
    ctx.barrier()
    ms = []
    for _ in range(args.steps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with clocks:
            a.record(stream)
            step()
            b.record(stream)
            torch.cuda.synchronize(dev)
        ms.append(a.elapsed_time(b))
    avg = ctx.max(statistics.mean(ms))
    hashing = ctx.world  # ranks hashing (one process over several GPUs: GPU 0 only)
    algo_bytes = n * (cfg5.dims / 8 + L * 4)
    ach = algo_bytes / (avg / 1e3) / 1e9
    out = {"metric": "fcLSH hash keys/sec (cfg5: 8M x 1024-bit rows per GPU, r=10, L=2047, 32-bit keys)",
           "value": hashing * n * L / (avg / 1e3), "unit": "keys/s", "ms_per_step": avg, "points_per_gpu": n,
           "gpus_hashing": hashing,
           "chunk": chunk, "scaling": "weak",
           "roofline": {"bound": "hbm", "kernel": "k_hash_f64_pt<11>", "achieved": ach, "peak": hbm, "unit": "GB/s",
                        "frac": ach / hbm, "traffic": measured_traffic("k_hash_f64_pt<11")[0],
                        "traffic_unit": "bytes per launch (one 1M-row chunk)",
                        "traffic_source": measured_traffic("k_hash_f64_pt<11")[1], "peak_source": peak_src,
                        "algorithmic_bytes_per_step": algo_bytes,
                        "algorithmic_bytes_per_launch": chunk * (cfg5.dims / 8 + L * 4)}}
    if ctx.root:
        from oracle import oracle as O
        orc = O.best()
        m0 = 64
        F.hash_batch_device(fam, d_rows[:chunk], keys, layout=1, key_stride=L, stream=stream)
        torch.cuda.synchronize(dev)
        got = keys[:m0].cpu().numpy().astype(np.uint64)
        want = orc.hash_batch(fam.mapping, fam.seeds, cfg5.dims, cfg5.radius, F.M31, rows[:m0], kind=int(fam.kind))
        out["keys_match_oracle_sample"] = bool((got == want).all())
        if ctx.G == 1 and not args.no_cpu:
            # the reference's hash_batch_into on this host: all threads and one
            cpu = {}
            for T, pts in ((threads, 100_000), (1, 10_000)):
                t0 = time.perf_counter()
                orc.hash_batch(fam.mapping, fam.seeds, cfg5.dims, cfg5.radius, F.M31, rows[:pts],
                               kind=int(fam.kind), threads=T)
                el = getattr(orc, "last_elapsed", None) or (time.perf_counter() - t0)
                cpu[f"T{T}"] = {"value": pts * L / el, "unit": "keys/s", "cores": T, "points": pts, "seconds": el}
            out["cpu_baseline"] = {"value": cpu[f"T{threads}"]["value"], "unit": "keys/s", "cores": threads,
                                   "kind": orc.kind, "sample": f"hash_batch_into (covering.cpp:169-182, P = 2^31-1) "
                                                               f"on the first 100,000 cfg5 rows, {threads} threads "
                                                               f"(shared family, per-thread scratch)",
                                   "T1": cpu["T1"]}
    del d_rows, keys
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-hash", action="store_true", help="skip the cfg5 hash microbenchmark")
    ap.add_argument("--no-configs", action="store_true", help="skip cfg1/2/4 (headline cfg3 only)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baselines and reference parity")
    ap.add_argument("--hash-points", type=int, default=8_000_000)
    ap.add_argument("--configs", default="1,2,4", help="the other configs measured beside the headline")
    ap.add_argument("--ref-scale", type=int, default=0, help=argparse.SUPPRESS)
    ap.add_argument("--replay", type=int, default=100, help="headline batch tiled this many times (>= 1M queries)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ctx = Ctx(args)
    if args.impl == "reference":
        run_reference_arm(args, ctx)
        ctx.close()
        return
    ctx.check_gpus(args)

    import torch

    from paper_1602_02620_b200.configs import CONFIGS
    torch.cuda.set_device(ctx.devices[0])
    threads = host_threads()
    hbm, peak_src = hbm_peak()
    # one dedicated stream for everything timed: the L2 flush, the CUDA events
    # and the library's work are all ordered on it
    stream = torch.cuda.Stream(device=ctx.devices[0])
    torch.cuda.set_stream(stream)
    flush = Flush(ctx.devices)
    clocks = ClockSampler(ctx.devices[0])
    spr4 = 1  # cfg4: one shard per GPU (at 8 GPUs exactly the BASELINE's 8-way sharding)
    # a small build + batch first, so the kernels' lazy module loading is not timed
    warm = CONFIGS[2].scaled(20000, queries=100)
    run_config(ctx, warm, "weak", 1, argparse.Namespace(**{**vars(args), "steps": 1, "no_cpu": True}), flush, stream,
               ClockSampler(ctx.devices[0]), hbm, peak_src, threads)

    head, extra = run_config(ctx, CONFIGS[HEADLINE], "weak", 1, args, flush, stream, clocks, hbm, peak_src, threads,
                             headline=True)
    if ctx.root:
        parity_and_cpu(ctx, CONFIGS[HEADLINE], *extra, threads, args, head, "weak")
    extra = None
    others = {}
    if not args.no_configs:
        for cid in [int(x) for x in args.configs.split(",") if x]:
            cfg = CONFIGS[cid]
            scaling, spr = ("strong", spr4) if cid == 4 else ("weak", 1)
            try:
                o, ex = run_config(ctx, cfg, scaling, spr, args, flush, stream, clocks, hbm, peak_src, threads)
                if ctx.root:
                    parity_and_cpu(ctx, cfg, *ex, threads, args, o, scaling)
                others[cfg.name] = o
            except Exception as e:  # noqa: BLE001
                others[cfg.name] = {"error": f"{type(e).__name__}: {e}"}
            ex = None
            gc.collect()
            torch.cuda.empty_cache()
    hash_block = None if args.no_hash else bench_hash(ctx, args, hbm, peak_src, flush, stream, threads, clocks)

    line = {
        "metric": METRIC, "value": head["value"], "unit": "queries/s", "n_gpus": ctx.G, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded Bernoulli(0.5) rows; 10k planted queries); BASELINE configs have no dataset",
        "config": head["config"],
        "e2e": head["e2e"], "roofline": head.get("roofline"), "cpu_baseline": head.get("cpu_baseline"),
        "gpu_launches": head["gpu_launches"],
        "gpu_launches_note": "own kernels in the timed steps (graph-replayed kernels counted; CUB's none on this path)",
        "clocks": None, "parity_vs_reference": head.get("parity_vs_reference"), "parity_kind": head.get("parity_kind"),
        "stages_ms_shard0": head["stages_ms_shard0"], "hash_stage_roofline": head.get("hash_stage_roofline"),
        "replay": head.get("replay"),
        "query_paths_shard0": head["query_paths_shard0"], "counters": head.get("counters"), "build": head["build"],
        "process_layout": "torchrun, one process per GPU" if ctx.torchrun else f"one process, {ctx.G} GPU(s)",
        "hash": hash_block,
        "configs": others,
    }
    line["clocks"] = clocks.summary()
    if ctx.root:
        print(json.dumps(line), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
