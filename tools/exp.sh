mkdir -p gpurun_out/x3
timeout 600 python -m pytest tests/test_gpu_shim.py tests/test_io.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/x3/pytest_gpu.txt 2>&1
tail -3 gpurun_out/x3/pytest_gpu.txt
nproc; lscpu | grep -i "model name\|flags" | cut -c1-300 | head -3
DICB200_SHIM_TRACE=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/x3/bench_c5.json 2> gpurun_out/x3/bench_c5.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/x3/bench_c5.json').read().strip().splitlines()[-1])
print('value',d['value'],'e2e',d['e2e']['value'],'shim',d['e2e_shim'])
PY
