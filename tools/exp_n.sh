make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 python bench.py > gpurun_out/n_bench_cfg2.json 2> gpurun_out/n_bench_cfg2.err
cat gpurun_out/n_bench_cfg2.json; tail -3 gpurun_out/n_bench_cfg2.err
