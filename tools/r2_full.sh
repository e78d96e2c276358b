make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 python tools/e2e_sparse_profile.py 2>&1 | head -45
for c in cfg4 cfg5; do
  timeout 1500 python bench.py --config $c > gpurun_out/r2g_bench_$c.json 2> gpurun_out/r2g_bench_$c.err
  python -c "
import json; j=json.loads(open('gpurun_out/r2g_bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(j['ms_per_step'],2), round(j['roofline']['frac'],3), round(j['roofline']['tmem_read']['frac'],3), j['e2e'] and round(j['e2e']['seconds'],3), {k: round(v,2) for k,v in j['phase_ms'].items()})"
done
