make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/epoch_profile.py cfg2 > gpurun_out/t_prof_fused.txt 2>&1
SOMB_FUSED_RERANK=0 timeout 300 python tools/epoch_profile.py cfg2 > gpurun_out/t_prof_sep.txt 2>&1
for f in gpurun_out/t_prof*.txt; do echo $f; python - "$f" <<'PY'
import json,sys
L=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')]
ep=[l for l in L if 'epoch' in l]
print(' screen', [l['screen'] for l in ep]); print(' rerank', [l['rerank'] for l in ep])
print(' total screen+rerank %.1f' % (sum(l['screen']+l['rerank'] for l in ep)), L[-1])
PY
done
tail -2 gpurun_out/t_prof_fused.txt
