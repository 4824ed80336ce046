python bench.py > gpurun_out/final_qwen3.json 2> gpurun_out/final_qwen3.err
for c in vicuna glm4 toy; do python bench.py --config $c --no-cpu-baseline > gpurun_out/final_$c.json 2>&1; done
for b in 1 2 4; do python bench.py --config qwen3 --B $b --no-cpu-baseline > gpurun_out/final_qwen3_B$b.json 2>&1; done
python bench.py --anchor --no-cpu-baseline > gpurun_out/final_qwen3_anchor.json 2>&1
python bench.py --config vicuna --anchor --no-cpu-baseline > gpurun_out/final_vicuna_anchor.json 2>&1
python bench.py --draft-kv --no-cpu-baseline > gpurun_out/final_qwen3_draft.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_reference.json 2>&1
for m in random uniform; do python bench.py --config pool --pool-lengths $m > gpurun_out/final_pool_$m.json 2>&1; done
python bench.py --config pool --min-group 8 > gpurun_out/final_pool_mg8.json 2>&1
python bench.py --config pool --pool-mode alg3 > gpurun_out/final_pool_alg3.json 2>&1
export SPECDEC_BENCH_LAUNCH_LOG=gpurun_out/final_launch_bytes_qwen3.json
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"verify|repad|realign" --csv --log-file gpurun_out/final_launches_qwen3.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"realign|verify|repad" -s 0 -c 3 -o gpurun_out/final_ncu_round_qwen3 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
