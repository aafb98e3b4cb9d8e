nproc
timeout 1500 python -m pytest tests/test_gpu_parity_large.py tests/test_gpu_cold_tier.py -q -x 2>&1 | tail -25
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity_large.py --deselect tests/test_gpu_cold_tier.py 2>&1 | tail -5
