"""The five BASELINE.json configurations as seeded synthetic workloads.

Every config forces its plan with PlanOverride (the automatic planner would
pick other shapes) and uses P = 2^31 - 1 so keys are
32-bit and bit-exact (IndexOptions::prime, index.hpp:25). Seeds follow the
CLI `build` chain (tools/fclsh.cpp:248-249): run = Rng(seed).stream("run", 0),
plan seed = run.stream("plan"), index seed = run.stream("index").
Inputs are seeded synthetic stand-ins with the configs' shapes and value
distributions (no dataset is involved).

This module does not load the product library at import time: the seed
chain and the generators come from a backend -- the product's C-ABI by
default (`product_backend()`), or the CPU oracle's restatement
(oracle/workloads.py), which produces the identical bytes, for the reference
arm of bench.py (it must not map libfclsh_b200.so).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

IDENTITY, REPLICATE, PARTITION = 0, 1, 2  # PlanKind (transform.hpp:24)
PLAN_NAMES = {IDENTITY: "identity", REPLICATE: "replicate", PARTITION: "partition"}


class _ProductBackend:
    """Seeds and generators from libfclsh_b200.so (imported lazily)."""

    @staticmethod
    def _F():
        from . import fclsh as F
        return F

    def rng_stream(self, seed, label, index=None):
        return self._F().rng_stream(seed, label, index)

    def gen_bernoulli(self, seed, n, dims, threads=8, row0=0):
        return self._F().gen_bernoulli(seed, n, dims, threads, row0=row0)

    def gen_clustered(self, seed, centres, n, dims, flip_p, threads=8, row0=0):
        return self._F().gen_clustered(seed, centres, n, dims, flip_p, threads, row0=row0)

    def gen_planted(self, seed, data, dims, nq, kmax):
        return self._F().gen_planted(seed, data, dims, nq, kmax)


_PRODUCT = _ProductBackend()


def product_backend():
    return _PRODUCT


@dataclass(frozen=True)
class Config:
    id: int
    name: str
    n: int
    dims: int
    radius: int
    plan_kind: int       # IDENTITY | PARTITION
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
    def plan_name(self) -> str:
        return PLAN_NAMES[self.plan_kind]

    @property
    def per_part_radius(self) -> int:
        return self.radius // self.t if self.plan_kind == PARTITION else self.radius

    @property
    def tables(self) -> int:
        parts = self.t if self.plan_kind == PARTITION else 1
        return parts * ((1 << (self.per_part_radius + 1)) - 1)

    @property
    def queries(self) -> int:
        return self.planted + self.uniform

    def root(self) -> int:
        return self.seed + self.id

    def plan_seed(self, backend=None) -> int:
        b = backend or _PRODUCT
        return b.rng_stream(b.rng_stream(self.root(), "run", 0), "plan")

    def index_seed(self, backend=None) -> int:
        b = backend or _PRODUCT
        return b.rng_stream(b.rng_stream(self.root(), "run", 0), "index")

    def override(self):
        from . import fclsh as F
        return F.PlanOverride(F.PlanKind(self.plan_kind), self.t)

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
    1: Config(1, "cfg1", 100_000, 128, 4, IDENTITY, 1, "bernoulli", 1_000, 4),
    2: Config(2, "cfg2", 1_000_000, 256, 8, IDENTITY, 1, "bernoulli", 10_000, 8, uniform=1_000),
    3: Config(3, "cfg3", 4_000_000, 512, 12, PARTITION, 2, "bernoulli", 10_000, 12),
    4: Config(4, "cfg4", 10_000_000, 256, 16, PARTITION, 2, "clustered", 10_000, 0,
              centres=10_000, flip_p=0.05, shards=8),
    5: Config(5, "cfg5", 8_000_000, 1024, 10, IDENTITY, 1, "bernoulli", 0, 0, hash_only=True),
}


def make_data(cfg: Config, threads: int = 8, backend=None, row0: int = 0, n: int | None = None) -> np.ndarray:
    """Rows [row0, row0 + n) of the config's dataset (default: all cfg.n rows);
    a slice of a larger global dataset (weak scaling) continues the same stream."""
    b = backend or _PRODUCT
    count = cfg.n if n is None else n
    if cfg.data == "clustered":
        return b.gen_clustered(cfg.root(), cfg.centres, count, cfg.dims, cfg.flip_p, threads, row0=row0)
    return b.gen_bernoulli(cfg.root(), count, cfg.dims, threads, row0=row0)


def make_queries(cfg: Config, data: np.ndarray | None, threads: int = 8, backend=None,
                 n_data: int | None = None) -> np.ndarray:
    """Planted queries (a row of `data` -- the whole dataset -- with k in [0, kmax]
    flipped bits), then uniform ones; for clustered configs, fresh draws from the
    same cluster process (rows [n_data, n_data + planted) of its stream, n_data =
    len(data) by default: independent of the data rows; `data` is not read)."""
    b = backend or _PRODUCT
    if cfg.data == "clustered":
        return b.gen_clustered(cfg.root(), cfg.centres, cfg.planted, cfg.dims, cfg.flip_p, threads,
                               row0=data.shape[0] if n_data is None else n_data)
    parts = []
    if cfg.planted:
        q, _ = b.gen_planted(cfg.root(), data, cfg.dims, cfg.planted, cfg.kmax)
        parts.append(q)
    if cfg.uniform:
        parts.append(b.gen_bernoulli(b.rng_stream(cfg.root(), "uniform-queries"), cfg.uniform, cfg.dims, threads))
    if not parts:
        return np.zeros((0, cfg.words), np.uint64)
    return np.concatenate(parts, axis=0)
