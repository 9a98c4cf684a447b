"""Test helpers: BitVector-layout rows in numpy (bit i -> word i/64, offset i%64)."""
from __future__ import annotations

import numpy as np


def from_string(s: str) -> np.ndarray:
    """BitVector::from_string (bitvec.cpp:23-31): leftmost char = position 0."""
    d = len(s)
    w = np.zeros((d + 63) // 64, np.uint64)
    for i, ch in enumerate(s):
        if ch == "1":
            w[i // 64] |= np.uint64(1 << (i % 64))
    return w


def to_string(row: np.ndarray, dims: int) -> str:
    return "".join("1" if (int(row[i // 64]) >> (i % 64)) & 1 else "0" for i in range(dims))


def random_rows(rng: np.random.Generator, n: int, dims: int) -> np.ndarray:
    w = (dims + 63) // 64
    r = rng.integers(0, 2**64, size=(n, w), dtype=np.uint64)
    if dims % 64:
        r[:, -1] &= np.uint64((1 << (dims % 64)) - 1)
    return r


def flip(row: np.ndarray, positions) -> np.ndarray:
    r = row.copy()
    for p in positions:
        r[p // 64] ^= np.uint64(1 << (p % 64))
    return r


def planted_queries(rng: np.random.Generator, data: np.ndarray, dims: int, nq: int, kmax: int) -> np.ndarray:
    out = np.empty((nq, data.shape[1]), np.uint64)
    for i in range(nq):
        src = data[rng.integers(0, data.shape[0])]
        k = int(rng.integers(0, kmax + 1))
        out[i] = flip(src, rng.choice(dims, size=k, replace=False))
    return out


def hamming(a: np.ndarray, b: np.ndarray) -> int:
    return int(sum(bin(int(x) ^ int(y)).count("1") for x, y in zip(a, b)))


def popcount_rows(x: np.ndarray) -> np.ndarray:
    """Row-wise popcount of a uint64 [n, W] array."""
    b = x.view(np.uint8)
    return np.unpackbits(b, axis=1).sum(axis=1)
