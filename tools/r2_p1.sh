make -j16 >/dev/null 2>&1 || echo BUILD FAILED
for CFG in cfg5 cfg4; do for P in 1 2; do
  timeout 900 python bench.py --config $CFG --steps 3 --passes $P --no-e2e --no-cpu-baseline > gpurun_out/p1_${CFG}_$P.json 2>/dev/null
  python -c "
import json; j=json.load(open('gpurun_out/p1_${CFG}_$P.json')); print('$CFG passes=$P', round(j['ms_per_step'],2), {k: round(v,2) for k,v in j['phase_ms'].items()}, j['candidates_per_row'], j['window_spilled_rows'])"
done; done
