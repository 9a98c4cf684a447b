"""The five BASELINE.json configurations as seeded synthetic workloads.

Every config forces its plan with PlanOverride (the automatic planner would
pick other shapes) and uses P = 2^31 - 1 so keys are
32-bit and bit-exact (IndexOptions::prime, index.hpp:25). Seeds follow the
CLI `build` chain (tools/fclsh.cpp:248-249): run = Rng(seed).stream("run", 0),
plan seed = run.stream("plan"), index seed = run.stream("index").
Inputs are seeded synthetic stand-ins with the configs' shapes and value
distributions (no dataset is involved).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import fclsh as F


@dataclass(frozen=True)
class Config:
    id: int
    name: str
    n: int
    dims: int
    radius: int
    plan_kind: F.PlanKind
    t: int
    data: str            # "bernoulli" | "clustered"
    planted: int         # planted queries
    kmax: int            # flips of a planted query, uniform in [0, kmax]
    uniform: int = 0     # extra uniform-random queries
    centres: int = 0
    flip_p: float = 0.0
    hash_only: bool = False
    shards: int = 1
    seed: int = 0x1602_02620

    @property
    def words(self) -> int:
        return (self.dims + 63) // 64

    @property
    def per_part_radius(self) -> int:
        return self.radius // self.t if self.plan_kind == F.PlanKind.partition else self.radius

    @property
    def tables(self) -> int:
        parts = self.t if self.plan_kind == F.PlanKind.partition else 1
        return parts * ((1 << (self.per_part_radius + 1)) - 1)

    @property
    def queries(self) -> int:
        return self.planted + self.uniform

    def root(self) -> int:
        return self.seed + self.id

    def plan_seed(self) -> int:
        return F.rng_stream(F.rng_stream(self.root(), "run", 0), "plan")

    def index_seed(self) -> int:
        return F.rng_stream(F.rng_stream(self.root(), "run", 0), "index")

    def override(self) -> F.PlanOverride:
        return F.PlanOverride(self.plan_kind, self.t)

    def scaled(self, n: int, queries: int | None = None) -> "Config":
        """Same distributions at a smaller size (parity tests)."""
        q = self.planted if queries is None else queries
        u = 0 if queries is not None else self.uniform
        cen = self.centres
        if self.data == "clustered":  # keep ~n/centres points per cluster
            cen = max(1, round(self.centres * n / self.n))
        return Config(self.id, self.name + f"@n={n}", n, self.dims, self.radius, self.plan_kind, self.t, self.data,
                      q, self.kmax, u, cen, self.flip_p, self.hash_only, self.shards, self.seed)


CONFIGS = {
    1: Config(1, "cfg1", 100_000, 128, 4, F.PlanKind.identity, 1, "bernoulli", 1_000, 4),
    2: Config(2, "cfg2", 1_000_000, 256, 8, F.PlanKind.identity, 1, "bernoulli", 10_000, 8, uniform=1_000),
    3: Config(3, "cfg3", 4_000_000, 512, 12, F.PlanKind.partition, 2, "bernoulli", 10_000, 12),
    4: Config(4, "cfg4", 10_000_000, 256, 16, F.PlanKind.partition, 2, "clustered", 10_000, 0,
              centres=10_000, flip_p=0.05, shards=8),
    5: Config(5, "cfg5", 8_000_000, 1024, 10, F.PlanKind.identity, 1, "bernoulli", 0, 0, hash_only=True),
}


def make_data(cfg: Config, threads: int = 8) -> np.ndarray:
    if cfg.data == "clustered":
        return F.gen_clustered(cfg.root(), cfg.centres, cfg.n, cfg.dims, cfg.flip_p, threads)
    return F.gen_bernoulli(cfg.root(), cfg.n, cfg.dims, threads)


def make_queries(cfg: Config, data: np.ndarray, threads: int = 8) -> np.ndarray:
    """Planted queries (a data row with k in [0, kmax] flipped bits), then uniform
    ones; for clustered configs, fresh draws from the same cluster process."""
    if cfg.data == "clustered":
        # same centres (stream "centres" of the same root), fresh assignments/flips
        both = F.gen_clustered(cfg.root(), cfg.centres, cfg.n + cfg.planted, cfg.dims, cfg.flip_p, threads)
        # rows [n, n+planted) continue the counter streams: independent of the data rows
        return both[cfg.n:].copy()
    parts = []
    if cfg.planted:
        q, _ = F.gen_planted(cfg.root(), data, cfg.dims, cfg.planted, cfg.kmax)
        parts.append(q)
    if cfg.uniform:
        parts.append(F.gen_bernoulli(F.rng_stream(cfg.root(), "uniform-queries"), cfg.uniform, cfg.dims, threads))
    if not parts:
        return np.zeros((0, cfg.words), np.uint64)
    return np.concatenate(parts, axis=0)
