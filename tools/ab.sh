#!/bin/bash
# A/B timing of two library builds on the same box: tools/ab.sh "c4 c5" A B
cfgs="$1"; shift
for rep in 1 2; do for v in "$@"; do for c in $cfgs; do
  DICB200_LIB=$PWD/abtest/lib$v.so python bench.py --config $c --steps 3 --warmup 2 --pairs 16 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_$c.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_${v}_$c.json').read().strip().splitlines()[-1]);print('AB $v $c', {k:round(x['avg_ms'],3) for k,x in d['stages'].items()})"
done; done; done
