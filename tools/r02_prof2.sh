# steady-state ncu: refine + launch list of a short bench
O=${OUT:-gpurun_out/r02h}; mkdir -p $O
python tools/profile_seq.py c5 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:refine_strip -s 1 -c 1 -o $O/refine python tools/profile_seq.py c5 2 > $O/refine.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --pairs 16 --no-cpu-baseline --no-e2e > $O/ncu_bench.log 2>&1
ls $O
