mkdir -p gpurun_out/x6
timeout 600 python -m pytest tests/test_gpu_shim.py -m gpu -x -q > gpurun_out/x6/pytest_shim.txt 2>&1
tail -15 gpurun_out/x6/pytest_shim.txt
DICB200_SHIM_TRACE=1 python bench.py --steps 5 --warmup 3 > gpurun_out/x6/bench_c5.json 2> gpurun_out/x6/bench_c5.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/x6/bench_c5.json').read().strip().splitlines()[-1])
print('value',d['value'],'e2e',d['e2e']['value'],'shim',d['e2e_shim'])
print('parity',d.get('parity'))
for k,v in (d.get('other_configs') or {}).items():
    print(k, {a:(v.get(a) if a!='parity' else {x:v['parity'][x] for x in ('integer_mismatches','converged_mismatches','max_du','max_dzncc','pass')} if v.get('parity') else None) for a in ('value','e2e','parity','unavailable')})
PY
