timeout 1200 python -m pytest tests/test_gpu_cold_tier.py -q -x > gpurun_out/cold.txt 2>&1; tail -1 gpurun_out/cold.txt
timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-offload-run > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -2 gpurun_out/bench_full.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_full.json'))
print('value', d['value'], 'memo_on', json.dumps(d['memo_on']))
for k,v in (d['configs_extra'] or {}).items(): print(k, v['value'], json.dumps(v.get('memo_on'))[:500])
PY
nvidia-smi --query-gpu=memory.total --format=csv; free -g | head -2
