"""Generates tests/golden/golden.json from the COMPILED REFERENCE
(oracle/_ref/libfclsh_ref.so, built from /root/reference/proj/src by
oracle/Makefile). Run in the build container: python tests/golden/make_golden.py

Contents: families (mapping, seeds, kind) from build_covering_family and the
keys hash_batch_into gives a few rows; small indexes (make_plan +
build_index) with query_r_nn ids and QueryReport counters. The same seeds
and shapes as the BASELINE configs are included (P = 2^31-1).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

M31, M61 = (1 << 31) - 1, (1 << 61) - 1


def rows_for(rng, n, d):
    w = (d + 63) // 64
    r = rng.integers(0, 2**64, size=(n, w), dtype=np.uint64)
    if d % 64:
        r[:, -1] &= np.uint64((1 << (d % 64)) - 1)
    return r


def main():
    ref = O.reference()
    rng = np.random.default_rng(1602)
    fams = []
    shapes = [(128, 4, M31, 0), (256, 8, M31, 0), (256, 6, M31, 0), (128, 8, M31, 0), (1024, 10, M31, 0),
              (100, 2, M61, 0), (300, 3, M61, 1), (17, 4, 101, 0), (40, 5, 97, 1), (4, 1, 5, 0)]
    for i, (d, r, p, iz) in enumerate(shapes):
        seed = 77 + i
        m, s, k = ref.build_family(d, r, seed, prime=p, include_zero=bool(iz))
        rows = rows_for(rng, 2, d)
        rows[1] = 0 if i % 3 == 0 else rows[1]
        keys = ref.hash_batch(m, s, d, r, p, rows, kind=k)
        fams.append({"dims": d, "radius": r, "prime": p, "include_zero": bool(iz), "seed": seed,
                     "mapping": m.tolist(), "seeds": [int(x) for x in s], "kind": k,
                     "rows": [int(x) for x in rows.reshape(-1)], "keys": [[int(x) for x in kr] for kr in keys]})
    idxs = []
    for j, (n, d, r, ov, p) in enumerate([(400, 64, 3, (0, 1), M31), (500, 128, 8, (2, 2), M31),
                                           (300, 64, 2, (1, 2), M61), (256, 32, 2, (0, 1), 101)]):
        rows = rows_for(rng, n, d)
        q = rows[rng.integers(0, n, 12)].copy()
        for i in range(12):
            for b in rng.choice(d, int(rng.integers(0, r + 2)), replace=False):
                q[i, b // 64] ^= np.uint64(1 << int(b % 64))
        h = ref.index_build(rows, d, r, 500 + j, 600 + j, override=ov, prime=p)
        counters, offsets, ids = h.query(q, r)
        idxs.append({"n": n, "dims": d, "radius": r, "override": list(ov), "prime": p, "plan_seed": 500 + j,
                     "index_seed": 600 + j, "rows": [int(x) for x in rows.reshape(-1)],
                     "queries": [int(x) for x in q.reshape(-1)], "counters": counters.tolist(),
                     "offsets": offsets.tolist(), "ids": ids.tolist()})
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    json.dump({"generator": "oracle/_ref (reference sources compiled by oracle/Makefile)",
               "families": fams, "indexes": idxs}, open(out, "w"))
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
