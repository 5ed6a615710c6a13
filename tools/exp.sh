mkdir -p gpurun_out/x5
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_memory_safety.py tests/test_gpu_known_answers.py -m gpu -x -q > gpurun_out/x5/pytest_gpu.txt 2>&1
tail -3 gpurun_out/x5/pytest_gpu.txt
CONFIGS="c5 c4" bash tools/quick_bench.sh > gpurun_out/x5/qb.txt 2>&1
cat gpurun_out/x5/qb.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:refine_strip -s 1 -c 1 -o gpurun_out/x5/refine python tools/profile_seq.py c5 2 > gpurun_out/x5/refine.log 2>&1
python tools/summarize_ncu.py gpurun_out/x5/refine.ncu-rep refine_c5 > gpurun_out/x5/refine_summary.jsonl
cat gpurun_out/x5/refine_summary.jsonl
