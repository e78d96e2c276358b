make -j16 >/dev/null 2>&1 || echo BUILD FAILED
# correctness first (small), with a hard timeout: the multicast variant
SOMB_TC_MULTICAST=2 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
SOMB_TC_MULTICAST=2 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
SOMB_TC_MULTICAST=2 timeout 300 python tools/epoch_profile.py cfg2 > gpurun_out/r_prof_mc2.txt 2>&1
timeout 300 python tools/epoch_profile.py cfg2 > gpurun_out/r_prof_mc1.txt 2>&1
for f in gpurun_out/r_prof*.txt; do echo $f; python - "$f" <<'PY'
import json,sys
L=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')]
ep=[l for l in L if 'epoch' in l]
print(' screen', [l['screen'] for l in ep]); print(' rerank', [l['rerank'] for l in ep])
print(' total screen %.1f rerank %.1f' % (sum(l['screen'] for l in ep), sum(l['rerank'] for l in ep)), L[-1])
PY
done
tail -3 gpurun_out/r_prof_mc2.txt
