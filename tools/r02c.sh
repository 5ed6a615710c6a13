mkdir -p gpurun_out/r02c
timeout 900 python -m pytest tests/test_gpu_tensor_search.py tests/test_gpu_known_answers.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r02c/pytest.txt 2>&1
for v in ws classic; do
  if [ $v = classic ]; then export DICB200_BS_CLASSIC=1; else unset DICB200_BS_CLASSIC; fi
  for c in c5 c4; do
    CONFIGS=$c bash tools/quick_bench.sh | sed "s/^/$v /" >> gpurun_out/r02c/qb.txt
  done
done
unset DICB200_BS_CLASSIC
for ns in 2 3 5 7; do DICB200_BS_NSPLIT=$ns CONFIGS=c5 bash tools/quick_bench.sh | sed "s/^/ns$ns /" >> gpurun_out/r02c/qb.txt; done
tail -3 gpurun_out/r02c/pytest.txt; cat gpurun_out/r02c/qb.txt
