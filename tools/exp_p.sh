make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -15
SOMB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/p_bench2.json 2> gpurun_out/p_bench2.err
cat gpurun_out/p_bench2.json | cut -c1-600; tail -5 gpurun_out/p_bench2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/p_ref2.json 2> gpurun_out/p_ref2.err
cat gpurun_out/p_ref2.json | cut -c1-400; tail -3 gpurun_out/p_ref2.err
