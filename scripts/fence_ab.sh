# Fence overhead on one GPU: the sharded 256^3 solve with 2 ranks (gloo control plane,
# both ranks on cuda:0, time-sliced), stream-ordered event fences vs stream sync + barrier.
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_dist.py 2>&1 | tail -2
for f in default event sync; do
  MLRG_FENCE=$f timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --same-gpu --steps 5 --warmup 3 --no-memo-run --no-offload-run --no-extra \
    --no-cpu-baseline --no-e2e > gpurun_out/fence_$f.json 2> gpurun_out/fence_$f.err
  python -c "import json; d=json.load(open('gpurun_out/fence_$f.json')); print('$f', round(d['value'],3), 'it/s', round(d['ms_per_step'],2), 'ms/step')" || tail -3 gpurun_out/fence_$f.err
done
