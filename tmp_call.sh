echo "B8 noseg $(python tools/kbench.py)"
echo "B8 seg128K $(python tools/kbench.py --seg)"
echo "B8 seg512K $(SPECDEC_REALIGN_SEG=524288 python tools/kbench.py --seg)"
echo "B2 noseg $(python tools/kbench.py --B 2)"
echo "B2 seg128K $(python tools/kbench.py --B 2 --seg)"
echo "GLM B2 noseg $(python tools/kbench.py --B 2 --planes 80 --H 2 --cap 4200 --kept 4000)"
echo "GLM B2 seg128K $(python tools/kbench.py --B 2 --planes 80 --H 2 --cap 4200 --kept 4000 --seg)"
echo "GLM B2 seg256K $(SPECDEC_REALIGN_SEG=262144 python tools/kbench.py --B 2 --planes 80 --H 2 --cap 4200 --kept 4000 --seg)"
for sg in 0 1; do SPECDEC_SEGMENT=$sg python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b26_q8_seg$sg.json 2>&1; SPECDEC_SEGMENT=$sg python bench.py --config glm4 --B 2 --no-cpu-baseline --no-e2e > gpurun_out/b26_glmB2_seg$sg.json 2>&1; SPECDEC_SEGMENT=$sg python bench.py --config qwen3 --B 2 --no-cpu-baseline --no-e2e > gpurun_out/b26_qB2_seg$sg.json 2>&1; done
