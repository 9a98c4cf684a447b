"""Times build_index for a BASELINE config several times in one process
(device time of each build, CUDA events inside the library)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1602_02620_b200 import fclsh as F  # noqa: E402
from paper_1602_02620_b200.configs import CONFIGS, make_data  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS[cid]
data = make_data(cfg, 16)
plan = F.make_plan(cfg.dims, cfg.radius, 1.0, cfg.n, cfg.plan_seed(), cfg.override())
for k in range(reps):
    t0 = time.perf_counter()
    ix = F.build_index(data, cfg.radius, plan, cfg.index_seed(), prime=F.M31)
    print(f"cfg{cid} build {k}: device {ix.build_ms:.1f} ms, wall {1e3 * (time.perf_counter() - t0):.1f} ms, "
          f"layout {ix.layout}", flush=True)
    del ix
