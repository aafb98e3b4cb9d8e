#!/bin/bash
# usage: sweep_n.sh N VAR v1 v2 ...  -> one short memo-off bench at N^3 per value of env var VAR
n=$1; var=$2; shift 2
for e in "$@"; do
  env $var=$e timeout 900 python bench.py --n $n --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-memo-run --no-offload-run 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['roofline']['kernels_ms_per_step']
print('n=$n', '$var', '$e', 'it/s %.3f'%d['value'], ' '.join('%s=%.1f'%(n.replace('k_fu2d_',''),v) for n,v in k.items()))"
done
