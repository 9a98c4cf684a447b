import numpy as np, sys, os
sys.path.insert(0, '.')
from paper_1602_02620_b200 import fclsh as F
from paper_1602_02620_b200.configs import CONFIGS, make_data, make_queries
cfg = CONFIGS[2]
data = make_data(cfg, 16); q = make_queries(cfg, data, 16)
plan = F.make_plan(cfg.dims, cfg.radius, 1.0, cfg.n, cfg.plan_seed(), cfg.override())
ix = F.build_index(data, cfg.radius, plan, cfg.index_seed(), prime=F.M31)
ix.stage_timing(True)
for it in range(8):
    res = ix.query_r_nn(q, cfg.radius)
print(ix.stage_ms(), ix.batch_ms())
