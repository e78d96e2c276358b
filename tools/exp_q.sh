make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for m in 1 2; do SOMB_RERANK_PIPE=$m timeout 300 python tools/epoch_profile.py cfg2 > gpurun_out/q_prof_$m.txt 2>&1; done
SOMB_RERANK_PIPE=2 timeout 300 python tools/epoch_profile.py cfg5 > gpurun_out/q_prof5.txt 2>&1
for f in gpurun_out/q_prof*.txt; do echo $f; python - "$f" <<'PY'
import json,sys
L=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')]
ep=[l for l in L if 'epoch' in l]
print(' screen', [l['screen'] for l in ep]); print(' rerank', [l['rerank'] for l in ep])
print(' total screen %.1f rerank %.1f' % (sum(l['screen'] for l in ep), sum(l['rerank'] for l in ep)), L[-1])
PY
done
