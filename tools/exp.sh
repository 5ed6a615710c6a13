mkdir -p gpurun_out/x7
timeout 900 python -m pytest tests/test_gpu_shim.py tests/test_gpu_known_answers.py tests/test_gpu_parity.py tests/test_gpu_memory_safety.py tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/x7/pytest.txt 2>&1
tail -8 gpurun_out/x7/pytest.txt
for ch in 0 8 16; do
DICB200_SHIM_CHUNK=$ch DICB200_SHIM_TRACE=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/x7/bench_c5_$ch.json 2> gpurun_out/x7/bench_c5_$ch.err
python - $ch <<'PY'
import json,sys
d=json.loads(open('gpurun_out/x7/bench_c5_%s.json'%sys.argv[1]).read().strip().splitlines()[-1])
print('chunk',sys.argv[1],'value',d['value'],'e2e',d['e2e']['value'],'shim',d['e2e_shim']['value'],d['e2e_shim'].get('trace'))
PY
done
