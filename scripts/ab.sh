# A/B of env settings on the 256^3 memo-off bench:  bash scripts/ab.sh "A=1" "A=0 B=2" ...
mkdir -p gpurun_out
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-memo-run --no-offload-run --no-extra > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/ab_$i.json')); k=d['roofline']['kernels_ms_per_step']
print('[$envs]', 'it/s %.2f'%d['value'], ' '.join('%s=%.2f'%(n.replace('k_fu2d_',''),v) for n,v in k.items()))" || tail -5 gpurun_out/ab_$i.err
done
