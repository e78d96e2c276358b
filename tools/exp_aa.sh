make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/aa_bench.json 2> gpurun_out/aa_bench.err
python -c "
import json; j=json.load(open('gpurun_out/aa_bench.json')); print(j['ms_per_step'], j['phase_ms'], j['roofline']['frac'], j['e2e'])"
tail -2 gpurun_out/aa_bench.err
