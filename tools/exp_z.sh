make -j16 >/dev/null 2>&1 || echo BUILD FAILED
SOMB_RERANK_PIPE=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for m in 1 2; do SOMB_RERANK_PIPE=$m timeout 300 python tools/epoch_profile.py cfg2 > gpurun_out/z_prof_$m.txt 2>&1; done
for f in gpurun_out/z_prof*.txt; do echo $f; python - "$f" <<'PY'
import json,sys
L=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')]
ep=[l for l in L if 'epoch' in l]
print(' rerank', [l['rerank'] for l in ep], sum(l['rerank'] for l in ep)); print(L[-1])
PY
done
