# ncu launch list + full capture of the tensor-core kernel for one config
cfg=${1:-c5}
python tools/profile_case.py $cfg 1 > /dev/null || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/profile_case.py $cfg 1 2>/dev/null | grep -v "^==\|^ok" > gpurun_out/tc_launch_$cfg.csv
ncu --set full --import-source on --clock-control none -k regex:bfs_tc_kernel -c 1 -o gpurun_out/tc_full_$cfg python tools/profile_case.py $cfg 1 > gpurun_out/tc_full_$cfg.log 2>&1
python - $cfg <<'PY'
import csv, sys
r = list(csv.reader(open(f"gpurun_out/tc_launch_{sys.argv[1]}.csv")))
h = r[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
for row in r[1:]:
    print(row[ki][:50], row[vi])
PY
