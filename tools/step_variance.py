"""Per-step device times of the cfg3 batch in one process (L2 flushed between
steps): is a slow run slow in every step (placement) or in a few (interference)?"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_02620_b200 import fclsh as F  # noqa: E402
from paper_1602_02620_b200.configs import CONFIGS, make_data, make_queries  # noqa: E402

cfg = CONFIGS[3]
data = make_data(cfg, 16)
q = make_queries(cfg, data, 16)
plan = F.make_plan(cfg.dims, cfg.radius, 1.0, cfg.n, cfg.plan_seed(), cfg.override())
ix = F.build_index(data, cfg.radius, plan, cfg.index_seed(), prime=F.M31)
qd = torch.from_numpy(q.view(np.int64)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    ix.query_device(qd, cfg.radius)
torch.cuda.synchronize()
ts = []
for _ in range(40):
    flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ix.query_device(qd, cfg.radius)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
free, total = torch.cuda.mem_get_info()
print(f"us/step min {min(ts):.1f} median {statistics.median(ts):.1f} max {max(ts):.1f}  p90 {sorted(ts)[35]:.1f}  "
      f"free {free >> 20} MiB  slow steps (> 1.3 x median): {[(i, round(t, 1)) for i, t in enumerate(ts) if t > 1.3 * statistics.median(ts)]}")
