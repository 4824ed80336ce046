timeout 600 python -m pytest tests/test_gpu_pool.py tests/test_gpu_golden.py -x -q 2>&1 | tail -3
for ring in 8 16; do for B in 1 3 8; do for e in 0 1 5 4 3 2; do echo "ring=$ring B=$B EXP=$e $(SPECDEC_K1_EXP=$e timeout 120 python tools/k1bench.py --B $B --ring $ring 2>&1 | tail -1)"; done; done; done > gpurun_out/r5_k1.txt
cat gpurun_out/r5_k1.txt
for est in "0 0" "0 10" "0 14" "0 20"; do echo "est=$est $(timeout 300 python bench.py --config pool --pool-est $est 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["pool"]["serial_kernel_ms"])')"; done
