make -j16 >/dev/null 2>&1 || echo BUILD FAILED
run() { tag=$1; shift; env "$@" timeout 300 python tools/epoch_profile.py cfg2 > gpurun_out/d_$tag.txt 2>&1; }
run smem0 SOMB_CAND_GMEM=0
run gm0 SOMB_CAND_GMEM=1
run gm_lag4 SOMB_CAND_GMEM=1 SOMB_SCREEN_LAG=4
run gm_lag16 SOMB_CAND_GMEM=1 SOMB_SCREEN_LAG=16
run smem_lag8 SOMB_CAND_GMEM=0 SOMB_SCREEN_LAG=8
for f in gpurun_out/d_*.txt; do echo $f; python - "$f" <<'PY'
import json,sys
L=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')]
ep=[l for l in L if 'epoch' in l]
print(' screen', [l['screen'] for l in ep]); print(' rerank', [l['rerank'] for l in ep])
print(' total screen %.1f rerank %.1f' % (sum(l['screen'] for l in ep), sum(l['rerank'] for l in ep)), L[-1])
PY
done
