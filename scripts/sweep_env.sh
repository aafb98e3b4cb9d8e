#!/bin/bash
# usage: sweep_env.sh VAR v1 v2 ...  -> one short bench per value of the env var VAR
var=$1; shift
for e in "$@"; do
  env $var=$e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-memo-run 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['roofline']['kernels_ms_per_step']
print('$var', '$e', 'it/s %.2f'%d['value'], ' '.join('%s=%.2f'%(n.replace('k_fu2d_',''),v) for n,v in k.items()))"
done
