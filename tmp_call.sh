timeout 900 python tools/grouping_sweep.py > gpurun_out/grouping_sweep.txt 2>&1; tail -3 gpurun_out/grouping_sweep.txt
for m in epoch alg3; do timeout 600 python bench.py --config pool --pool-mode $m > gpurun_out/b17_pool_$m.json 2>&1; done
timeout 600 python bench.py --draft-kv --no-cpu-baseline > gpurun_out/b17_qwen3_draftkv.json 2>&1
timeout 600 python bench.py --config vicuna --draft-kv --no-cpu-baseline > gpurun_out/b17_vicuna_draftkv.json 2>&1
