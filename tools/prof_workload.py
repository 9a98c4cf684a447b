"""Small, ncu-friendly workload: cfg2 index + two query batches, and two
1M-row chunks of the cfg5 hash (point-major, as the bench). Used for the
launch list and the `ncu --set full` captures under profiles/ (never a bench
number)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_02620_b200 import fclsh as F  # noqa: E402
from paper_1602_02620_b200.configs import CONFIGS, make_data, make_queries  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("all", "query", "cfg2", "cfg3", "cfg1"):
    cfg = CONFIGS[{"cfg3": 3, "cfg1": 1}.get(what, 2)]
    data = make_data(cfg)
    q = make_queries(cfg, data)
    if os.environ.get("NQ"):  # a smaller batch (latency studies)
        q = q[:int(os.environ["NQ"])]
    plan = F.make_plan(cfg.dims, cfg.radius, 1.0, cfg.n, cfg.plan_seed(), cfg.override())
    ix = F.build_index(data, cfg.radius, plan, cfg.index_seed(), prime=F.M31)
    qd = torch.from_numpy(q.view(np.int64)).cuda()
    for _ in range(2):
        ix.query_device(qd, cfg.radius)
    torch.cuda.synchronize()
if what in ("cfg4shard", "cfg4", "cfg4csr"):
    # cfg4: shard 0 of the 8-shard layout (buckets), or the whole 10M index
    # (automatic layout, or CSR forced)
    from paper_1602_02620_b200 import cluster
    cfg = CONFIGS[4]
    data = make_data(cfg, 16)
    q = make_queries(cfg, data, 16)
    b, e = cluster.shard_range(cfg.n, cfg.shards, 0) if what == "cfg4shard" else (0, cfg.n)
    plan = F.make_plan(cfg.dims, cfg.radius, 1.0, cfg.n, cfg.plan_seed(), cfg.override())
    kw = {"layout": "csr"} if what == "cfg4csr" else {}
    ix = F.build_index(data[b:e], cfg.radius, plan, cfg.index_seed(), prime=F.M31, id_offset=b, **kw)
    qd = torch.from_numpy(q.view(np.int64)).cuda()
    ix.stage_timing(True)
    for _ in range(3):
        ix.query_device(qd, cfg.radius)
    torch.cuda.synchronize()
    print(what, ix.layout, ix.stage_ms(), ix.path_counts())
if what in ("all", "hash"):
    cfg5 = CONFIGS[5]
    n = 1_000_000
    rows = F.gen_bernoulli(cfg5.root(), n, cfg5.dims)
    fam = F.build_covering_family(cfg5.dims, cfg5.radius, cfg5.index_seed(), prime=F.M31)
    d = torch.from_numpy(rows.view(np.int64)).cuda()
    keys = torch.empty((n, fam.table_count()), dtype=torch.int32, device="cuda")
    for _ in range(2):
        F.hash_batch_device(fam, d, keys, layout=1, key_stride=fam.table_count())
    torch.cuda.synchronize()
print("done")
