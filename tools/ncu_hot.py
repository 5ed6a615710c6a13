"""Aggregate warp-stall samples of an ncu report by CUDA source line."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kern = ["--kernel-name", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []  # reports with several kernels
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", *kern],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hk = next(k for k, r in enumerate(rows[:6]) if "Line No" in r)
cur, agg, fname = None, {}, ""
for r in rows[hk + 1:]:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 6:
        continue
    if r[0] and r[0] != "Line No":
        cur = (fname + ":" + r[0], r[1][:90])
    try:
        s = int(r[4])
    except ValueError:
        continue
    agg[cur] = agg.get(cur, 0) + s
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:7d} {100 * v / tot:5.1f}% {k[0]:>16s} {k[1]}")
