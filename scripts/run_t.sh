mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/t.log 2>&1; echo "pytest rc $?" >> gpurun_out/t.log
tail -3 gpurun_out/t.log
timeout 600 python scripts/memo_breakdown.py --steps 10 --memo off,local --no-prof 2>&1 | tail -24
