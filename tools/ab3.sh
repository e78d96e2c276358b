# grouped re-rank on / off on the tree build (SOMB_RERANK_GROUP), bench lines + the parity test
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests -x -q -m gpu -k "grouped_rerank or overflow or one_call" 2>&1 | tail -3
for CFG in ${CFGS:-cfg2 cfg5 cfg4}; do
  for v in 1 0; do
    SOMB_RERANK_GROUP=$v timeout 900 python bench.py --config $CFG --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/ab3_${CFG}_$v.json 2>/dev/null
    python -c "
import json; j=json.load(open('gpurun_out/ab3_${CFG}_$v.json')); print('$CFG group=$v', round(j['ms_per_step'],2), {k: round(v,2) for k,v in j['phase_ms'].items()})"
  done
done
