"""Batch timeline of the query path (FCLSH_TRACE build): per batch the step as
the bench times it (CUDA events around query_device, L2 flushed before) and
the device-side stamps of every kernel (globaltimer, us after the prologue
starts): prologue, warp-kernel CTA entry / PDL wait / last warp exit, hand-over
kernel, compaction entry / wait / exit, publish.

  make -C paper_1602_02620_b200 EXTRA=-DFCLSH_TRACE BUILD=build_trace OUT=lib/libfclsh_b200_trace.so
  FCLSH_LIB=$PWD/paper_1602_02620_b200/lib/libfclsh_b200_trace.so python tools/timeline.py cfg3 [nq,...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = "/tmp/fclsh_tl.txt"
os.environ["FCLSH_TL_OUT"] = OUT

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_02620_b200 import fclsh as F  # noqa: E402
from paper_1602_02620_b200.configs import CONFIGS, make_data, make_queries  # noqa: E402

NAMES = ["pro_in", "pro_out", "warp_in", "warp_in_last", "warp_wait", "warp_out", "dense_in", "dense_wait",
         "dense_out", "comp_in", "comp_wait", "comp_out", "publish", "comp_loaded", "comp_scanned"]
what = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [10000]
cfg = CONFIGS[int(what[3:])]
data = make_data(cfg, 16)
q = make_queries(cfg, data, 16)
plan = F.make_plan(cfg.dims, cfg.radius, 1.0, cfg.n, cfg.plan_seed(), cfg.override())
ix = F.build_index(data, cfg.radius, plan, cfg.index_seed(), prime=F.M31)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for nq in sizes:
    qq = np.tile(q, ((nq + q.shape[0] - 1) // q.shape[0], 1))[:nq]
    qd = torch.from_numpy(qq.view(np.int64)).cuda()
    for _ in range(3):
        ix.query_device(qd, cfg.radius)
    torch.cuda.synchronize()
    if os.path.exists(OUT):
        os.remove(OUT)
    steps = []
    for _ in range(7):
        if os.environ.get("FLUSH", "1") != "0":
            flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ix.query_device(qd, cfg.radius)
        b.record()
        torch.cuda.synchronize()
        steps.append(a.elapsed_time(b) * 1e3)
    rows = [[float(x) for x in ln.split()[1:]] for ln in open(OUT)]
    print(f"{what} nq={nq}: step (events) median {np.median(steps):.1f} us  {[round(s, 1) for s in steps]}")
    print("   " + " ".join(f"{n:>12}" for n in NAMES))
    for s, r in zip(steps, rows):
        print(f"   " + " ".join(f"{x:12.2f}" for x in r) + f"   step {s:.1f}")
