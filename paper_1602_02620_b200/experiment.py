"""run_experiment over the engine: the reference's
per-query metrics (bench.hpp:17-67, bench.cpp:64-158) and its CSV writer
(bench.cpp:160-170), computed from the GPU's batched results.

Methods: "fclsh" and "bclsh" build the covering index on the GPU ("bclsh"
hashes per mask in the reference; its buckets, and so every counter, are the
same by construction, index.hpp:17-22), "classic" builds the bit-sampling
index on the GPU (identity plan, k from choose_k, the covering plan's table
count unless overridden, bench.cpp:118-136), "linear" is the GPU scan.
"mih" (multi-index hashing, mih.cpp) is not on this engine's path.

Counters, true_near, precision and recall equal the reference's exactly
(same seeds: Rng(seed).stream("run", run).stream("plan" | "index")). Stage
times are the batch's per-stage device times divided evenly over its
queries (the reference times each query on the host).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, Optional, TextIO

import numpy as np

from . import fclsh as F


@dataclass
class ExperimentConfig:  # bench.hpp:17-38
    method: str = "fclsh"
    radius: int = 0
    c: float = 1.0
    delta: float = 0.1
    plan_override: Optional[F.PlanOverride] = None
    k_override: Optional[int] = None
    tables_override: Optional[int] = None
    seed: int = 0
    repeats: int = 5
    fresh_seeds: bool = True
    include_zero_column: bool = False
    prime: int = F.M61
    table_budget: int = F.DEFAULT_TABLE_BUDGET


@dataclass
class MetricsRow:  # bench.hpp:42-57
    query_id: int = 0
    method: str = ""
    radius: int = 0
    collisions: float = 0.0
    candidates: float = 0.0
    found: float = 0.0
    true_near: float = 0.0
    precision: float = 0.0
    recall: float = 0.0
    time_s1_us: float = 0.0
    time_s2_us: float = 0.0
    time_s3_us: float = 0.0


@dataclass
class GroundTruth:  # workload.hpp:44-47
    radius: int
    entries: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), np.uint32))  # (query, point, distance)


def _true_ids(truth: GroundTruth, nq: int, radius: int):
    e = np.asarray(truth.entries, dtype=np.uint32).reshape(-1, 3)
    if e.size and int(e[:, 0].max()) >= nq:
        raise F.DataError(f"truth: query id {int(e[:, 0].max())} out of range")  # workload.cpp:124-126
    keep = e[e[:, 2] <= radius]
    order = np.lexsort((keep[:, 1], keep[:, 0]))
    return keep[order, :2]


def _hits(found_q, found_id, true_pairs, nq: int, n: int) -> np.ndarray:
    """|found ids ∩ true ids| per query (both are sets per query)."""
    a = found_q.astype(np.int64) * (n + 1) + found_id.astype(np.int64)
    b = true_pairs[:, 0].astype(np.int64) * (n + 1) + true_pairs[:, 1].astype(np.int64)
    both = np.intersect1d(a, b, assume_unique=True)
    return np.bincount((both // (n + 1)).astype(np.int64), minlength=nq).astype(np.float64)


def run_experiment(data_rows, query_rows, dims: int, truth: GroundTruth, cfg: ExperimentConfig,
                   device: int = 0) -> list[MetricsRow]:
    """run_experiment (bench.cpp:64-158) with the engine doing every search."""
    data = np.ascontiguousarray(data_rows, dtype=np.uint64)
    queries = np.ascontiguousarray(query_rows, dtype=np.uint64)
    n, nq = data.shape[0], queries.shape[0]
    if n == 0:
        raise F.UsageError("experiment: empty dataset")
    if nq == 0:
        raise F.UsageError("experiment: no queries")
    if data.shape[1] != queries.shape[1]:
        raise F.UsageError("experiment: data and query widths differ")
    if cfg.repeats == 0:
        raise F.UsageError("experiment: repeats must be >= 1")
    if truth.radius < cfg.radius:
        raise F.DataError(f"experiment: ground truth radius {truth.radius} is below the query radius "
                          f"{cfg.radius}")
    if cfg.method not in ("fclsh", "bclsh", "classic", "linear"):
        if cfg.method == "mih":
            raise F.UsageError(f"experiment: method '{cfg.method}' is not part of the GPU engine")
        raise F.UsageError(f"unknown method '{cfg.method}'")
    true_pairs = _true_ids(truth, nq, cfg.radius)
    true_near = np.bincount(true_pairs[:, 0].astype(np.int64), minlength=nq).astype(np.float64)

    acc = {k: np.zeros(nq) for k in ("collisions", "candidates", "found", "precision", "recall", "s1", "s2", "s3")}
    root = cfg.seed
    for run in range(cfg.repeats):
        run_seed = F.rng_stream(root, "run", run if cfg.fresh_seeds else 0)
        if cfg.method == "linear":
            import torch
            dd = torch.from_numpy(data.view(np.int64)).to(f"cuda:{device}")
            qd = torch.from_numpy(queries.view(np.int64)).to(f"cuda:{device}")
            tri = F.LinearScan(device).triples(dd, qd, dims, cfg.radius)
            fq, fid = tri[:, 0], tri[:, 1]
            coll = np.full(nq, float(n))
            cand = coll
            found = np.bincount(fq.astype(np.int64), minlength=nq).astype(np.float64)
            s1 = s2 = np.zeros(nq)
            s3 = np.zeros(nq)  # the scan's device time is not split per query
        else:
            extra = {}
            if cfg.method == "classic":  # bench.cpp:121-136
                plan = F.make_plan(dims, cfg.radius, cfg.c, n, F.rng_stream(run_seed, "plan"),
                                   F.PlanOverride(F.PlanKind.identity, 1), cfg.table_budget)
                tables = cfg.tables_override
                if not tables:  # the covering family's table count under the same plan flags
                    tables = F.make_plan(dims, cfg.radius, cfg.c, n, F.rng_stream(run_seed, "plan-probe"),
                                         cfg.plan_override, cfg.table_budget).table_count()
                extra = {"method": "classic", "delta": cfg.delta, "k_override": cfg.k_override,
                         "tables_override": tables}
            else:
                plan = F.make_plan(dims, cfg.radius, cfg.c, n, F.rng_stream(run_seed, "plan"), cfg.plan_override,
                                   cfg.table_budget)
            ix = F.build_index(data, cfg.radius, plan, F.rng_stream(run_seed, "index"), prime=cfg.prime,
                               include_zero_column=cfg.include_zero_column, table_budget=cfg.table_budget,
                               device=device, dims=dims, **extra)
            ix.stage_timing(True)
            res = ix.query_r_nn(queries, cfg.radius)
            fq, fid = res.query, res.id
            coll = res.collisions.astype(np.float64)
            cand = res.candidates.astype(np.float64)
            found = res.found.astype(np.float64)
            per_q = 1e-3 / nq  # batch stage ms -> per-query seconds
            s1 = np.full(nq, max(res.time_s1_ms, 0.0) * per_q)
            s2 = np.full(nq, max(res.time_s2_ms, 0.0) * per_q)
            s3 = np.full(nq, max(res.time_s3_ms, 0.0) * per_q)
        hits = _hits(fq, fid, true_pairs, nq, n)
        acc["collisions"] += coll
        acc["candidates"] += cand
        acc["found"] += found
        with np.errstate(divide="ignore", invalid="ignore"):
            acc["precision"] += np.where(cand == 0, 1.0, hits / np.where(cand == 0, 1.0, cand))
            acc["recall"] += np.where(true_near == 0, 1.0, hits / np.where(true_near == 0, 1.0, true_near))
        acc["s1"] += s1
        acc["s2"] += s2
        acc["s3"] += s3

    inv = 1.0 / cfg.repeats
    return [MetricsRow(q, cfg.method, cfg.radius, acc["collisions"][q] * inv, acc["candidates"][q] * inv,
                       acc["found"][q] * inv, float(true_near[q]), acc["precision"][q] * inv,
                       acc["recall"][q] * inv, acc["s1"][q] * inv * 1e6, acc["s2"][q] * inv * 1e6,
                       acc["s3"][q] * inv * 1e6) for q in range(nq)]


HEADER = ("query_id,method,r,collisions,candidates,found,true_near,precision,recall,"
          "time_s1_us,time_s2_us,time_s3_us\n")


def _g(x: float) -> str:
    """A double as the reference prints it (setprecision(max_digits10), bench.cpp:163)."""
    return "%.17g" % x


def write_metrics(rows: Iterable[MetricsRow], out: TextIO) -> None:
    """write_metrics (bench.cpp:160-170)."""
    out.write(HEADER)
    for r in rows:
        out.write(f"{int(r.query_id)},{r.method},{int(r.radius)},{_g(r.collisions)},{_g(r.candidates)},"
                  f"{_g(r.found)},{_g(r.true_near)},{_g(r.precision)},{_g(r.recall)},{_g(r.time_s1_us)},"
                  f"{_g(r.time_s2_us)},{_g(r.time_s3_us)}\n")
