timeout 900 python -m pytest tests/test_gpu_pool.py -q -x 2>&1 | tail -3
for ex in native python; do timeout 600 python bench.py --config pool --pool-exec $ex > gpurun_out/b20_pool_$ex.json 2>&1; done
timeout 600 python bench.py --config pool --pool-mode alg3 > gpurun_out/b20_pool_alg3_native.json 2>&1
timeout 600 python bench.py --config pool --pool-lengths uniform > gpurun_out/b20_pool_uniform_native.json 2>&1
timeout 600 python bench.py --config pool --min-group 8 > gpurun_out/b20_pool_mg8_native.json 2>&1
