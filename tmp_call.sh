for cfg in 0 3 10 11 12 13 14 2; do for ctas in 1 2; do
  echo "cfg=$cfg ctas=$ctas $(SPECDEC_REALIGN_CFG=$cfg SPECDEC_REALIGN_CTAS=$ctas python tools/kbench.py)"
done; done
for cfg in 10 11 12; do SPECDEC_REALIGN_CFG=$cfg SPECDEC_REALIGN_CTAS=1 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b10_cfg${cfg}_c1.json 2>&1; done
for cfg in 10 12; do SPECDEC_REALIGN_CFG=$cfg SPECDEC_REALIGN_CTAS=1 python bench.py --config glm4 --B 2 --no-cpu-baseline --no-e2e > gpurun_out/b10_glmB2_cfg${cfg}_c1.json 2>&1; done
python bench.py --config glm4 --B 2 --no-cpu-baseline --no-e2e > gpurun_out/b10_glmB2_default.json 2>&1
