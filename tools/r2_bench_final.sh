# Final bench lines for every BASELINE config + smoke + the reference arm.  Usage: bash tools/r2_bench_final.sh TAG
TAG=${1:-s5}
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in cfg2 cfg1 cfg4 cfg5 cfg3; do
  timeout 1500 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  python -c "
import json; j=json.loads(open('gpurun_out/${TAG}_bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(j['ms_per_step'],2), round(j['roofline']['frac'],3), j['e2e'] and round(j['e2e']['seconds'],3), j['cpu_baseline'] and '%.3g' % j['cpu_baseline']['value'], {k: round(v,2) for k,v in j['phase_ms'].items()}, j['clocks'])" || tail -3 gpurun_out/${TAG}_bench_$c.err
done
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref_cfg2.json 2> gpurun_out/${TAG}_bench_ref_cfg2.err
head -c 400 gpurun_out/${TAG}_bench_ref_cfg2.json
