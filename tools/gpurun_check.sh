set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 > gpurun_out/r1s2_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1s2_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r1s2_bench_cfg2.json 2> gpurun_out/r1s2_bench_cfg2.err
cat gpurun_out/r1s2_pytest_gpu.txt gpurun_out/r1s2_smoke.txt gpurun_out/r1s2_bench_cfg2.json; tail -5 gpurun_out/r1s2_bench_cfg2.err
