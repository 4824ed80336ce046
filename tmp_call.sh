timeout 900 python -m pytest tests/test_gpu_pool.py tests/test_gpu_toylm.py -q -x 2>&1 | tail -15
