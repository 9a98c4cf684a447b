"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
launches per kernel, mean and total time. Usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(anonymous namespace\)::|<?unnamed>::|fclsh_b200::", "", name)
    base = name.split("(")[0].replace("void ", "")
    return base[:74]


rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
agg = collections.OrderedDict()
for r in rows:
    k = short(r[4])
    us = float(r[-1].replace(",", "")) / (1e3 if r[-2] == "ns" else 1)
    n, t = agg.get(k, (0, 0.0))
    agg[k] = (n + 1, t + us)
print(f"{len(rows)} launches")
print(f"{'kernel':74s} {'n':>5} {'mean us':>10} {'total ms':>10}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:74s} {n:5d} {t / n:10.1f} {t / 1e3:10.2f}")
