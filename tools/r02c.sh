# GPU check of the block-sum variants: parity tests, then quick C5/C4 lines (ws / classic / dy slicing)
mkdir -p gpurun_out/r02c; : > gpurun_out/r02c/qb.txt
timeout 900 python -m pytest tests/test_gpu_tensor_search.py tests/test_gpu_known_answers.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r02c/pytest.txt 2>&1
for c in c5 c4; do CONFIGS=$c bash tools/quick_bench.sh | sed "s/^/ws /" >> gpurun_out/r02c/qb.txt; done
for ns in ${NSPLITS:-}; do DICB200_BS_NSPLIT=$ns CONFIGS=c5 bash tools/quick_bench.sh | sed "s/^/ns$ns /" >> gpurun_out/r02c/qb.txt; done
tail -3 gpurun_out/r02c/pytest.txt; cat gpurun_out/r02c/qb.txt
