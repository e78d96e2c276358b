make -j16 >/dev/null 2>&1 || echo BUILD FAILED
B="python bench.py --no-e2e --no-cpu-baseline --steps 7 --warmup 3"
timeout 300 $B > gpurun_out/a_cfg2.json 2>&1
timeout 300 $B --no-rerank-order > gpurun_out/a_cfg2_noorder.json 2>&1
timeout 300 $B --config cfg5 --steps 3 > gpurun_out/a_cfg5.json 2>&1
timeout 300 $B --config cfg5 --steps 3 --passes 1 > gpurun_out/a_cfg5_p1.json 2>&1
timeout 300 $B --config cfg4 --steps 3 --passes 1 > gpurun_out/a_cfg4_p1.json 2>&1
for f in gpurun_out/a_*.json; do echo $f; python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        j=json.loads(l); print(j['ms_per_step'], j['phase_ms'], j['roofline']['frac'], j.get('window_truncated_rows'), j.get('candidates_per_row'))
    else: print(l[:300])
"; done
