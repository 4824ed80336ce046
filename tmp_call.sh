timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python bench.py --no-cpu-baseline > gpurun_out/b6_qwen3.json 2>&1
python bench.py --config qwen3 --B 1 --no-cpu-baseline > gpurun_out/b6_qwen3_B1.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"verify|repad|realign" --csv --log-file gpurun_out/launches6.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:verify -s 8 -c 1 -o gpurun_out/prof6_verify python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > /dev/null 2>&1
