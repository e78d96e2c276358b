make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in cfg2 cfg5; do timeout 300 python tools/epoch_profile.py $c > gpurun_out/y_prof_$c.txt 2>&1; done
for f in gpurun_out/y_prof*.txt; do echo $f; python - "$f" <<'PY'
import json,sys
L=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')]
ep=[l for l in L if 'epoch' in l]
print(' screen', [l['screen'] for l in ep]); print(' rerank', [l['rerank'] for l in ep]); print(' update', [l['update'] for l in ep]); print(L[-1])
PY
done
timeout 1200 python tools/full_parity.py 1000000 10 > gpurun_out/y_full.txt 2>&1
cat gpurun_out/y_full.txt
