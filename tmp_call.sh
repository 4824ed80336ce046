for pdl in 0 1; do
  SPECDEC_PDL=$pdl python bench.py --no-cpu-baseline > gpurun_out/b30_q8_pdl$pdl.json 2>&1
  SPECDEC_PDL=$pdl python bench.py --config vicuna --no-cpu-baseline > gpurun_out/b30_vic_pdl$pdl.json 2>&1
  SPECDEC_PDL=$pdl python bench.py --config qwen3 --B 1 --no-cpu-baseline > gpurun_out/b30_q1_pdl$pdl.json 2>&1
  SPECDEC_PDL=$pdl python bench.py --config glm4 --no-cpu-baseline > gpurun_out/b30_glm_pdl$pdl.json 2>&1
done
