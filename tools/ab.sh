# A/B timing of two builds of the library on the same box:
#   bash tools/ab.sh TAG CONFIG [STEPS]   (B = build_ab/libsomb200_base.so, A = the tree's build)
TAG=$1; CFG=$2; STEPS=${3:-3}
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
for r in 1 2; do
  for v in A B; do
    if [ $v = B ]; then export SOMB_LIB_PATH=$PWD/build_ab/libsomb200_base.so; else unset SOMB_LIB_PATH; fi
    timeout 900 python bench.py --config $CFG --steps $STEPS --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${CFG}_$v$r.json 2>/dev/null
    python -c "
import json; j=json.load(open('gpurun_out/${TAG}_${CFG}_$v$r.json')); print('$CFG $v$r', round(j['ms_per_step'],2), {k: round(v,2) for k,v in j['phase_ms'].items()})"
  done
done
