"""Query-kernel time against batch size (device-resident rows, L2 flushed
before each batch): the intercept of time(nq) is the batch's ramp + tail, the
slope its steady-state cost per query. Usage: python tools/batch_sweep.py cfg3"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_02620_b200 import fclsh as F  # noqa: E402
from paper_1602_02620_b200.configs import CONFIGS, make_data, make_queries  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1250, 2500, 5000, 10000, 20000, 40000, 100000]
cfg = CONFIGS[int(what[3:])]
data = make_data(cfg, 16)
q = make_queries(cfg, data, 16)
plan = F.make_plan(cfg.dims, cfg.radius, 1.0, cfg.n, cfg.plan_seed(), cfg.override())
ix = F.build_index(data, cfg.radius, plan, cfg.index_seed(), prime=F.M31)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rbuf = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
mode = os.environ.get("FLUSH", "write")  # write | write+read | none


def do_flush():
    if mode == "none":
        return
    flush.fill_(1)
    if mode == "write+read":
        rbuf.view(torch.int64).sum()

for nq in sizes:
    reps = (nq + q.shape[0] - 1) // q.shape[0]
    qq = np.tile(q, (reps, 1))[:nq]
    qd = torch.from_numpy(qq.view(np.int64)).cuda()
    for _ in range(3):
        ix.query_device(qd, cfg.radius)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        do_flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ix.query_device(qd, cfg.radius)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ix.stage_timing(True)
    ix.query_device(qd, cfg.radius)
    ix.query_device(qd, cfg.radius)
    torch.cuda.synchronize()
    st = ix.stage_ms()
    ix.stage_timing(False)
    ms = float(np.median(ts))
    print(f"{what} flush={mode} nq={nq:7d} step={ms * 1e3:8.1f} us  {nq / ms / 1e3:7.2f} Mq/s  probe={st['fused'] * 1e3:8.1f} us "
          f"hash={st['hash'] * 1e3:6.1f} dense={st['dense'] * 1e3:6.1f} compact={st['compact'] * 1e3:6.1f}", flush=True)
