for s in 20 100 300; do python bench.py --steps $s --no-cpu-baseline > gpurun_out/b22_steps$s.json 2>&1; done
python bench.py --steps 100 --episode 0 --no-cpu-baseline > gpurun_out/b22_noepisode.json 2>&1
