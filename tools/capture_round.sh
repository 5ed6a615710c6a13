# One GPU call: GPU tests, bench lines for every config, the reference arm,
# the ncu launch list of the default bench command and full captures of the
# top kernels (steady state: second pair of a fixed-first sequence).
# Outputs under ${OUT:-gpurun_out/cap}/.
set -x
O=${OUT:-gpurun_out/cap}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1
for c in c1 c2 c2b c3 c3x c4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_c5.json 2> $O/bench_ref_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_bench.log 2>&1
OUT=$O/prof bash tools/prof_steady.sh
ls -la $O
