# Quick perf + correctness pass: smoke, bench lines for the dense configs, then the GPU tests.
#   bash tools/gpurun_quick.sh TAG [pytest-args]
TAG=${1:-q}
shift
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
for c in cfg5 cfg4 cfg2; do
  timeout 900 python bench.py --config $c --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
if [ "$#" -gt 0 ]; then timeout 1500 python -m pytest tests -x -q -m gpu "$@" 2>&1 | tail -30 > gpurun_out/${TAG}_pytest.txt; fi
cat gpurun_out/${TAG}_smoke.txt
for c in cfg5 cfg4 cfg2; do python -c "
import json; j=json.load(open('gpurun_out/${TAG}_bench_$c.json')); print('$c', round(j['ms_per_step'],2), {k: round(v,2) for k,v in j['phase_ms'].items()}, j.get('candidates_per_row'))" || tail -3 gpurun_out/${TAG}_bench_$c.err; done
cat gpurun_out/${TAG}_pytest.txt 2>/dev/null
