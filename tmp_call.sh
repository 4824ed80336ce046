export SPECDEC_BENCH_LAUNCH_LOG=gpurun_out/launch_bytes_qwen3.json
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"verify|repad|realign" --csv --log-file gpurun_out/launches14.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"realign|verify|repad" -s 0 -c 3 -o gpurun_out/prof14_round python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
export SPECDEC_BENCH_LAUNCH_LOG=gpurun_out/launch_bytes_vicuna.json
ncu --set full --clock-control none --import-source on -k regex:"realign" -s 0 -c 1 -o gpurun_out/prof14_vicuna python bench.py --config vicuna --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
unset SPECDEC_BENCH_LAUNCH_LOG
python bench.py > gpurun_out/b14_qwen3.json 2>&1
