"""Share of the step per kernel from an ncu --metrics gpu__time_duration.sum
--csv launch list (per-launch times are cold-cache and serialised: compare
shares, not absolutes). Usage: launch_share.py LAUNCHES.csv [skip-regex]"""
import collections
import csv
import re
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
skip = re.compile(sys.argv[2] if len(sys.argv) > 2 else r"render|pipes|elementwise|fill|copy|reduce|^kern<")
tot, cnt = collections.Counter(), collections.Counter()
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
for r in rows[1:]:
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("(anonymous namespace)::", "")
    if skip.search(name):
        continue
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[name] += 1
all_us = sum(tot.values())
print(f"{'kernel':70s} {'launches':>8s} {'us/launch':>10s} {'share':>6s}")
for k, v in tot.most_common():
    print(f"{k[:70]:70s} {cnt[k]:8d} {v / cnt[k]:10.1f} {100 * v / all_us:5.1f}%")
