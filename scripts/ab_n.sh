# A/B of env settings at a given size:  N=512 STEPS=4 bash scripts/ab_n.sh "A=1" "B=2" ...
mkdir -p gpurun_out
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs timeout 900 python bench.py --n ${N:-512} --steps ${STEPS:-4} --warmup 2 --no-cpu-baseline --no-e2e --no-memo-run --no-offload-run --no-extra > gpurun_out/abn_$i.json 2> gpurun_out/abn_$i.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/abn_$i.json')); k=d['roofline']['kernels_ms_per_step']
print('[$envs]', 'it/s %.3f'%d['value'], ' '.join('%s=%.1f'%(n.replace('k_fu2d_',''),v) for n,v in k.items()))" || tail -5 gpurun_out/abn_$i.err
done
