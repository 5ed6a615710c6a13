"""Per-CUDA-source-line totals of an ncu report (instructions executed and
warp-stall samples), top lines first:  ncu_src_top.py report.ncu-rep [file.cu] [N]
(NCU_KERNEL=regex:<name> selects one kernel of a multi-kernel report)"""
import csv
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
import os

kf = ["--kernel-name", os.environ["NCU_KERNEL"]] if os.environ.get("NCU_KERNEL") else []  # multi-kernel reports
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", *kf],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
h = next(r for r in rows[:10] if "Instructions Executed" in r)
ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
fname, line, src = "", -1, {}
ins, smp = {}, {}
for r in rows:
    if r and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if len(r) < len(h) or r[0] == "Line No":
        continue
    if r[0]:
        line = (fname, int(r[0]))
        src[line] = r[1].strip()[:80]
    try:
        n, s = int(r[ie]), int(r[ss])
    except ValueError:
        continue
    ins[line] = ins.get(line, 0) + n
    smp[line] = smp.get(line, 0) + s
ti, ts = sum(ins.values()) or 1, sum(smp.values()) or 1
print(f"total instructions {ti}  stall samples {ts}")
keys = [k for k in ins if not want or k[0] == want]
for k in sorted(keys, key=lambda k: -ins[k])[:top]:
    print(f"{k[0]}:{k[1]:5d} instr {100 * ins[k] / ti:5.1f}%  samples {100 * smp[k] / ts:5.1f}%  {src.get(k, '')}")
