for m in graph-fork graph-serial direct-fork direct-serial; do python bench.py --round-mode $m --no-cpu-baseline --no-e2e > gpurun_out/b12_$m.json 2>&1; done
for m in graph-fork graph-serial direct-serial; do python bench.py --config vicuna --round-mode $m --no-cpu-baseline --no-e2e > gpurun_out/b12_vic_$m.json 2>&1; done
