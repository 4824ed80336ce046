timeout 600 python -m pytest tests/test_gpu_round.py -q -x -k "rounds" 2>&1 | tail -2
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b34_q8.json 2>&1
python bench.py --config qwen3 --B 1 --no-cpu-baseline --no-e2e > gpurun_out/b34_q1.json 2>&1
python bench.py --config toy --no-cpu-baseline --no-e2e > gpurun_out/b34_toy.json 2>&1
timeout 900 python tools/grouping_sweep.py > gpurun_out/grouping_sweep_v2.txt 2>&1
