# GPU check after kernel changes: targeted parity tests + quick bench lines
O=gpurun_out/r02g; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_known_answers.py tests/test_gpu_tensor_search.py tests/test_gpu_fullsize.py tests/test_gpu_memory_safety.py tests/test_gpu_parity.py tests/test_gpu_bicubic.py -x -q > $O/pytest.txt 2>&1
tail -3 $O/pytest.txt
for c in ${CONFIGS:-c5 c4 c3}; do CONFIGS=$c bash tools/quick_bench.sh; done > $O/qb.txt 2>&1
cat $O/qb.txt
