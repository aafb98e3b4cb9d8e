set -x
DIAG_KERNELS=gaussian,es timeout 900 python scripts/diag_precision.py > gpurun_out/diag.txt 2>&1
tail -5 gpurun_out/diag.txt
timeout 900 python -m pytest tests/test_gpu_recon.py tests/test_gpu_ops.py -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-offload-run --kernel gaussian > gpurun_out/b_g.json 2> gpurun_out/b_g.err
python -c "
import json
for f in ['gpurun_out/b_g.json']:
    d=json.load(open(f)); print(f, d['value'], d['memo_on']['value'] if d['memo_on'] else None, d['memo_on'] and d['memo_on']['hit_rate']); print(json.dumps(d['roofline']['kernels_ms_per_step']))
"
