timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_cols4.py -q -x 2>&1 | tail -1
for v in default gen; do
  if [ $v = default ]; then unset MLRG_LIB; else export MLRG_LIB=$PWD/paper_2511_01893_b200/libv/$v/libmlr.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-memo-run --no-offload-run --no-extra > gpurun_out/b_$v.json 2> gpurun_out/b_$v.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/b_$v.json')); k=d['roofline']['kernels_ms_per_step']
print('$v', 'it/s %.2f'%d['value'], ' '.join('%s=%.2f'%(n.replace('k_fu2d_',''),v) for n,v in k.items()))"
done
