# bench lines: tree build (grouped re-rank on / off) vs the base build
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests -x -q -m gpu -k "grouped_rerank or overflow or hand_cases or one_call or golden" 2>&1 | tail -4
for CFG in cfg5 cfg4 cfg2; do
  for v in A A0 B; do
    unset SOMB_LIB_PATH SOMB_RERANK_GROUP
    [ $v = B ] && export SOMB_LIB_PATH=$PWD/build_ab/libsomb200_base.so
    [ $v = A0 ] && export SOMB_RERANK_GROUP=0
    timeout 900 python bench.py --config $CFG --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/ab2_${CFG}_$v.json 2>/dev/null
    python -c "
import json; j=json.load(open('gpurun_out/ab2_${CFG}_$v.json')); print('$CFG $v', round(j['ms_per_step'],2), {k: round(v,2) for k,v in j['phase_ms'].items()}, j['candidates_per_row']['mean'])"
  done
done
