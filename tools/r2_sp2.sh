make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests -x -q -m gpu -k "sparse" 2>&1 | tail -2
timeout 900 python tools/parity_sweep.py cfg3 sparse 500000 3 2>&1 | grep -E "SUMMARY|epoch\": 1,"
timeout 600 python tools/e2e_sparse_phases.py 2>&1 | tail -1
timeout 1500 python bench.py --config cfg3 > gpurun_out/r2j_bench_cfg3.json 2> gpurun_out/r2j_bench_cfg3.err; tail -1 gpurun_out/r2j_bench_cfg3.json | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['ms_per_step'],2), j['phase_ms'], j['e2e']['seconds'])"
