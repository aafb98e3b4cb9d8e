mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/tc.log 2>&1; echo "pytest rc $?" >> gpurun_out/tc.log
tail -3 gpurun_out/tc.log
timeout 900 python scripts/memo_breakdown.py --n 512 --steps 3 --warmup 2 --memo off 2>&1 | tail -16
