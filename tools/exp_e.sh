make -j16 >/dev/null 2>&1 || echo BUILD FAILED
for hc in 8 16 32; do
  SOMB_HALF_CAP=$hc timeout 300 python tools/epoch_profile.py cfg2 > gpurun_out/e_prof_hc$hc.txt 2>&1
  SOMB_HALF_CAP=$hc timeout 600 python tools/trunc_check.py 9 > gpurun_out/e_trunc_hc$hc.txt 2>&1
done
SOMB_HALF_CAP=8 timeout 900 python tools/full_parity.py 1000000 10 > gpurun_out/e_full_hc8.txt 2>&1
for f in gpurun_out/e_prof_*.txt; do echo $f; python - "$f" <<'PY'
import json,sys
L=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')]
ep=[l for l in L if 'epoch' in l]
print(' screen', [l['screen'] for l in ep]); print(' rerank', [l['rerank'] for l in ep]); print(' cand', [l['cand_mean'] for l in ep], [l['trunc'] for l in ep])
print(' total screen %.1f rerank %.1f' % (sum(l['screen'] for l in ep), sum(l['rerank'] for l in ep)), L[-1])
PY
done
tail -n 12 gpurun_out/e_trunc_*.txt gpurun_out/e_full_hc8.txt
