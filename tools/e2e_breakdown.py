"""Where the end-to-end query call spends its time (cfg2 batch): the C call
alone (fclsh_query + fclsh_result_free) vs the Python wrapper, against the
device time of the batch."""
import ctypes as C
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_02620_b200 import _native as N  # noqa: E402
from paper_1602_02620_b200 import fclsh as F  # noqa: E402
from paper_1602_02620_b200.configs import CONFIGS, make_data, make_queries  # noqa: E402

cfg = CONFIGS[2]
data = make_data(cfg, 16)
q = make_queries(cfg, data, 16)
plan = F.make_plan(cfg.dims, cfg.radius, 1.0, cfg.n, cfg.plan_seed(), cfg.override())
ix = F.build_index(data, cfg.radius, plan, cfg.index_seed(), prime=F.M31)
pq = torch.from_numpy(q.view(np.int64)).pin_memory().numpy().view(np.uint64)
L = N.lib()
rp = C.POINTER(N.Result)()
for _ in range(5):
    ix.query_r_nn(pq, cfg.radius)
c_t, py_t, dev_t = [], [], []
for _ in range(50):
    t0 = time.perf_counter()
    L.fclsh_query(ix._h, pq.ctypes.data_as(N.u64p), q.shape[0], cfg.radius, C.byref(rp))
    t1 = time.perf_counter()
    L.fclsh_result_free(rp)
    c_t.append(t1 - t0)
ix.stage_timing(True)  # the batch's device time (its events add ~8 us)
for _ in range(50):
    L.fclsh_query(ix._h, pq.ctypes.data_as(N.u64p), q.shape[0], cfg.radius, C.byref(rp))
    L.fclsh_result_free(rp)
    dev_t.append(ix.batch_ms())
ix.stage_timing(False)
for _ in range(50):
    t0 = time.perf_counter()
    r = ix.query_r_nn(pq, cfg.radius)
    py_t.append(time.perf_counter() - t0)
    del r
med = lambda v: 1e3 * statistics.median(v)  # noqa: E731
print(f"device batch {statistics.median(dev_t):.3f} ms | C fclsh_query {med(c_t):.3f} ms | "
      f"Python query_r_nn {med(py_t):.3f} ms (medians of 50)")

# the bench's order: a stage-timed pass first, then end-to-end calls
ix.stage_timing(True)
for _ in range(3):
    ix.query_r_nn(pq, cfg.radius)
ix.stage_timing(False)
ts = []
for _ in range(40):
    t0 = time.perf_counter()
    r = ix.query_r_nn(pq, cfg.radius)
    ts.append(1e3 * (time.perf_counter() - t0))
print("per call ms:", " ".join(f"{t:.2f}" for t in ts))
