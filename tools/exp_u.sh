make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/u_bench_cfg2.json 2> gpurun_out/u_bench_cfg2.err
python -c "
import json; j=json.load(open('gpurun_out/u_bench_cfg2.json')); print(j['ms_per_step'], j['phase_ms'], j['roofline']['frac'], j['e2e']['seconds'], j['clocks'])"
