# One GPU call: GPU tests, bench lines for every config, the reference arm,
# the ncu launch list of the default bench command and full captures of the
# top kernels. Outputs under ${OUT:-gpurun_out/cap}/.
set -x
mkdir -p ${OUT:-gpurun_out/cap}
timeout 600 python -m pytest tests -m gpu -x -q > ${OUT:-gpurun_out/cap}/pytest_gpu.txt 2>&1
for c in c1 c2 c3 c3x c4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > ${OUT:-gpurun_out/cap}/bench_$c.json 2> ${OUT:-gpurun_out/cap}/bench_$c.err
done
timeout 900 python bench.py > ${OUT:-gpurun_out/cap}/bench_c5.json 2> ${OUT:-gpurun_out/cap}/bench_c5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > ${OUT:-gpurun_out/cap}/bench_ref_c5.json 2> ${OUT:-gpurun_out/cap}/bench_ref_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${OUT:-gpurun_out/cap}/launches_bench_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > ${OUT:-gpurun_out/cap}/ncu_bench.log 2>&1
python tools/profile_case.py c5 1 > /dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bs_kernel -c 1 -o ${OUT:-gpurun_out/cap}/full_bs_c5 python tools/profile_case.py c5 1 > ${OUT:-gpurun_out/cap}/full_bs_c5.log 2>&1
DICB200_BFS_TC=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:bfs_tc_kernel -c 1 -o ${OUT:-gpurun_out/cap}/full_bfs_tc_c5 python tools/profile_case.py c5 1 > ${OUT:-gpurun_out/cap}/full_bfs_tc_c5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:refine_strip -c 1 -o ${OUT:-gpurun_out/cap}/full_refine_c5 python tools/profile_case.py c5 1 > ${OUT:-gpurun_out/cap}/full_refine_c5.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"tc_argmax|tc_stats|tc_strips|tc_prep" -c 4 -o ${OUT:-gpurun_out/cap}/full_aux_c5 python tools/profile_case.py c5 1 > ${OUT:-gpurun_out/cap}/full_aux_c5.log 2>&1
ls -la ${OUT:-gpurun_out/cap}
