export SPECDEC_BENCH_SHARE_GPU=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/b27_w2.json 2> gpurun_out/b27_w2.err; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 2 --config pool --pool-n 256 --max-new 32 > gpurun_out/b27_pool_w2.json 2> gpurun_out/b27_pool_w2.err; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29523 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/b27_ref_w2.json 2> gpurun_out/b27_ref_w2.err; echo rc=$?
tail -3 gpurun_out/b27_w2.err gpurun_out/b27_pool_w2.err
