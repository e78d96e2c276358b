make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 600 python tools/screen_only.py 4 3
SOMB_TC_MULTICAST=2 timeout 300 python tools/epoch_profile.py cfg5 > gpurun_out/s_prof5_mc2.txt 2>&1
SOMB_TC_MULTICAST=2 timeout 300 python tools/epoch_profile.py cfg4 > gpurun_out/s_prof4_mc2.txt 2>&1
for f in gpurun_out/s_prof*.txt; do echo $f; python - "$f" <<'PY'
import json,sys
L=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')]
ep=[l for l in L if 'epoch' in l]
print(' screen', [l['screen'] for l in ep]); print(' rerank', [l['rerank'] for l in ep])
print(' total screen %.1f rerank %.1f' % (sum(l['screen'] for l in ep), sum(l['rerank'] for l in ep)), L[-1])
PY
done
