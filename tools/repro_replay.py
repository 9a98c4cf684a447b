"""cfg3 index, a 10k batch, then the batch tiled to NQ queries (default 1M)
through query_device: the bench's replay step in isolation (debugging)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_02620_b200 import fclsh as F  # noqa: E402
from paper_1602_02620_b200.configs import CONFIGS, make_data, make_queries  # noqa: E402

nq = int(os.environ.get("NQ", "1000000"))
cfg = CONFIGS[3]
data = make_data(cfg, 16)
q = make_queries(cfg, data, 16)
plan = F.make_plan(cfg.dims, cfg.radius, 1.0, cfg.n, cfg.plan_seed(), cfg.override())
cl = F.Cluster([0], 1).build(data, cfg.radius, plan, cfg.index_seed(), prime=F.M31)
qd = torch.from_numpy(q.view(np.int64)).cuda()
for _ in range(3):
    r = cl.query_device(qd, cfg.radius)
torch.cuda.synchronize()
print("10k ok", r.total, flush=True)
qq = np.tile(q, ((nq + q.shape[0] - 1) // q.shape[0], 1))[:nq]
qr = torch.from_numpy(qq.view(np.int64)).cuda()
for i in range(3):
    r = cl.query_device(qr, cfg.radius)
    torch.cuda.synchronize()
    print(nq, "ok", i, r.total, flush=True)
