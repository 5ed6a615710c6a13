"""Instructions executed + stall samples of an ncu report summed over line
ranges of one source file: ncu_lines.py rep file.cu a-b:name ..."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hk = next(k for k, r in enumerate(rows[:6]) if "Line No" in r)
h = rows[hk]
ie = h.index("Instructions Executed")
cur, ins, smp, fname = None, {}, {}, ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1]
        continue
    if len(r) < 6 or r[0] == "Line No":
        continue
    if r[0]:
        cur = int(r[0]) if fname.endswith(sys.argv[2].split(":")[0]) else -1
    try:
        n = int(r[ie])
        s = int(r[4])
    except ValueError:
        continue
    ins[cur] = ins.get(cur, 0) + n
    smp[cur] = smp.get(cur, 0) + s
ti, ts = sum(ins.values()) or 1, sum(smp.values()) or 1
for spec in sys.argv[3:]:
    rng, name = spec.split(":")
    a, b = map(int, rng.split("-"))
    i = sum(v for k, v in ins.items() if a <= k <= b)
    s = sum(v for k, v in smp.items() if a <= k <= b)
    print(f"{name:12s} instr {i:12d} ({100 * i / ti:5.1f}%)  samples {s:8d} ({100 * s / ts:5.1f}%)")
