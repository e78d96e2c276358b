make -j16 >/dev/null 2>&1 || echo BUILD FAILED
for v in -1 0 2 4 5 8 -1; do
  SOMB_RERANK_F2F=$v timeout 900 python bench.py --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/f2f_$v.json 2>/dev/null
  python -c "
import json; j=json.loads(open('gpurun_out/f2f_$v.json').read().strip().splitlines()[-1]); print('f2f $v', round(j['ms_per_step'],2), round(j['phase_ms']['rerank'],2), j['clocks']['sm_mhz'])"
done
