# bench a config under two settings of one environment knob:  bash tools/ab_env.sh TAG CFG VAR V1 V2 [STEPS]
TAG=$1; CFG=$2; VAR=$3; V1=$4; V2=$5; STEPS=${6:-3}
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
for r in 1 2; do for v in $V1 $V2; do
  env $VAR=$v timeout 900 python bench.py --config $CFG --steps $STEPS --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${CFG}_$v$r.json 2>/dev/null
  python -c "
import json; j=json.load(open('gpurun_out/${TAG}_${CFG}_$v$r.json')); print('$CFG $VAR=$v', round(j['ms_per_step'],2), {k: round(v,2) for k,v in j['phase_ms'].items()})" || echo failed
done; done
