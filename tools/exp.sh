mkdir -p gpurun_out/x8
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_memory_safety.py -m gpu -x -q > gpurun_out/x8/pytest.txt 2>&1
tail -2 gpurun_out/x8/pytest.txt
CONFIGS="c5 c4" bash tools/quick_bench.sh > gpurun_out/x8/qb.txt 2>&1
cat gpurun_out/x8/qb.txt
