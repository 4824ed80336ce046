timeout 600 python -m pytest tests/test_gpu_verify.py tests/test_gpu_golden.py tests/test_gpu_fuzz.py tests/test_gpu_pool.py -x -q 2>&1 | tail -3
for B in 1 3 8; do for e in 0 1 5 4; do echo "B=$B EXP=$e $(SPECDEC_K1_EXP=$e timeout 120 python tools/k1bench.py --B $B --ring 16 2>&1 | tail -1)"; done; done
for est in "0 0" "0 10"; do echo "est=$est $(timeout 300 python bench.py --config pool --pool-est $est 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"])')"; done
timeout 300 python bench.py > gpurun_out/r6_bench.json 2>&1; tail -1 gpurun_out/r6_bench.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["kernels_ms_per_step"], d["e2e"]["value"])'
timeout 300 python bench.py --B 1 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("B1", d["value"], d["kernels_ms_per_step"], d["e2e"]["value"])'
