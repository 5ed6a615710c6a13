mkdir -p gpurun_out/x10
for k in 0 6 8 12 16; do
echo "park_iter $k" >> gpurun_out/x10/qb.txt
DICB200_NR_PARK_ITER=$k CONFIGS="c3 c2" bash tools/quick_bench.sh >> gpurun_out/x10/qb.txt 2>&1
done
cat gpurun_out/x10/qb.txt | cut -c1-170
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_bicubic.py tests/test_gpu_memory_safety.py tests/test_accuracy.py -m gpu -x -q > gpurun_out/x10/pytest.txt 2>&1
tail -3 gpurun_out/x10/pytest.txt
