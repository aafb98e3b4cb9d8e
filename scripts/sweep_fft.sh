#!/bin/bash
# FFT pass tile sweep: one short bench per MLRG_FFT_ELEMS value.
for e in "$@"; do
  MLRG_FFT_ELEMS=$e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-memo-run 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['roofline']['kernels_ms_per_step']
print('elems', $e, 'it/s %.2f'%d['value'], ' '.join('%s=%.2f'%(n.replace('k_fu2d_',''),v) for n,v in k.items()))"
done
