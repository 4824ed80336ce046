for c in qwen3 vicuna glm4; do python bench.py --config $c --anchor --no-cpu-baseline > gpurun_out/b19_${c}_anchor.json 2>&1; done
python bench.py --anchor --draft-kv --no-cpu-baseline > gpurun_out/b19_qwen3_anchor_draft.json 2>&1
python bench.py --config qwen3 --B 4 --anchor --no-cpu-baseline > gpurun_out/b19_qwen3B4_anchor.json 2>&1
