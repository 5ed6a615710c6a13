"""Print kernel name + duration (ns) rows of an ncu --csv launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
for r in rows[1:]:
    if "render" not in r[ki]:
        print("  ", r[ki][:50], r[vi])
