mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py tests/test_gpu_recon.py tests/test_gpu_parity_large.py tests/test_gpu_large_n.py -m gpu -q -x --timeout 600 > gpurun_out/ts.log 2>&1; echo "pytest rc $?" >> gpurun_out/ts.log
tail -3 gpurun_out/ts.log
bash scripts/ncu_kernels.sh ${TAG:-sp3} k_fu2d_adj_spread
timeout 600 python scripts/memo_breakdown.py --steps 10 --memo off 2>&1 | grep -E "k_fu2d_adj_spread|kern" | tail -3
