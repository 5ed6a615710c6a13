mkdir -p gpurun_out/cap2
for c in c1 c2 c3 c3x c4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cap2/bench_$c.json 2> gpurun_out/cap2/bench_$c.err
done
timeout 900 python bench.py > gpurun_out/cap2/bench_c5.json 2> gpurun_out/cap2/bench_c5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/cap2/bench_ref_c5.json 2> gpurun_out/cap2/bench_ref_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cap2/launches_bench_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cap2/ncu_bench.log 2>&1
ls gpurun_out/cap2
