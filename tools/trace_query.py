"""Per-query phase timeline of the warp query kernel (FCLSH_TRACE build).

  make -C paper_1602_02620_b200 EXTRA=-DFCLSH_TRACE BUILD=build_trace OUT=lib/libfclsh_b200_trace.so
  FCLSH_LIB=$PWD/paper_1602_02620_b200/lib/libfclsh_b200_trace.so python tools/trace_query.py cfg3 [nq]

Stamps per query (index.cu, FCLSH_TRACE_STAMP): globaltimer at start/end,
SM clocks after the hash, the probes and the verify. Prints when queries
start and end relative to the first warp's entry, and the phase split."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = "/tmp/fclsh_trace.bin"
os.environ["FCLSH_TRACE_OUT"] = OUT

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_02620_b200 import fclsh as F  # noqa: E402
from paper_1602_02620_b200.configs import CONFIGS, make_data, make_queries  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
ghz = float(os.environ.get("SM_GHZ", "1.965"))
cfg = CONFIGS[int(what[3:])]
data = make_data(cfg, 16)
q = make_queries(cfg, data, 16)
q = np.tile(q, ((nq + q.shape[0] - 1) // q.shape[0], 1))[:nq]
plan = F.make_plan(cfg.dims, cfg.radius, 1.0, cfg.n, cfg.plan_seed(), cfg.override())
ix = F.build_index(data, cfg.radius, plan, cfg.index_seed(), prime=F.M31)
qd = torch.from_numpy(q.view(np.int64)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ix.query_device(qd, cfg.radius)
torch.cuda.synchronize()
if os.path.exists(OUT):
    os.remove(OUT)
flush.fill_(1)
torch.cuda.synchronize()
ix.query_device(qd, cfg.radius)
torch.cuda.synchronize()
raw = np.fromfile(OUT, dtype=np.uint64)
n, k = int(raw[0]), int(raw[1])
t = raw[2:2 + n * k].reshape(n, k).astype(np.int64)
ok = t[:, 1] > 0
t = t[ok]
k0 = t[:, 6].min()
st, en = (t[:, 0] - k0) / 1e3, (t[:, 1] - k0) / 1e3
hs, pr, vf = t[:, 2] / ghz / 1e3, (t[:, 3] - t[:, 2]) / ghz / 1e3, (t[:, 4] - t[:, 3]) / ghz / 1e3
print(f"{what} nq={nq} traced={ok.sum()} kernel span (first entry -> last end) {en.max():.1f} us; "
      f"warp entries spread {(t[:, 6].max() - k0) / 1e3:.1f} us")
pct = lambda a: " ".join(f"{np.percentile(a, p):6.1f}" for p in (0, 10, 50, 90, 99, 100))
print("percentiles        p0    p10    p50    p90    p99   p100 (us)")
print("start          ", pct(st))
print("end            ", pct(en))
print("duration       ", pct(en - st))
print("  hash         ", pct(hs))
print("  probes       ", pct(pr))
print("  verify+out   ", pct(vf))
prev = t[:, 2]
for r in range(8):
    c = t[:, 8 + r]
    if not (c > 0).any():
        break
    print(f"  round {r}      ", pct((c - prev) / ghz / 1e3))
    prev = c
order = np.argsort(st)
for lo in range(0, int(en.max()) + 10, 10):
    live = ((st <= lo + 10) & (en >= lo)).sum()
    done = (en < lo + 10).sum()
    print(f"  [{lo:4d},{lo + 10:4d}) us: queries live {live:6d}, finished by end {done:6d}")
