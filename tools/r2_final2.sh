make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
bash tools/r2_bench_all.sh
timeout 900 python bench.py --impl reference > gpurun_out/r2h_bench_ref_cfg2.json 2> gpurun_out/r2h_bench_ref_cfg2.err; head -c 250 gpurun_out/r2h_bench_ref_cfg2.json
