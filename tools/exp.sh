mkdir -p gpurun_out/x2
for pv in 0 1; do
  DICB200_BS_PV=$pv DICB200_BS_PROF=1 python tools/profile_seq.py c5 2 > gpurun_out/x2/prof_pv$pv.txt 2>&1
  DICB200_BS_PV=$pv CONFIGS=c5 bash tools/quick_bench.sh > gpurun_out/x2/qb_pv$pv.txt 2>&1
  cp gpurun_out/qb_c5.json gpurun_out/x2/qb_c5_pv$pv.json
done
DICB200_BS_PV=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_memory_safety.py -m gpu -x -q > gpurun_out/x2/pytest_gpu.txt 2>&1
tail -3 gpurun_out/x2/pytest_gpu.txt
cat gpurun_out/x2/prof_pv*.txt gpurun_out/x2/qb_pv*.txt
