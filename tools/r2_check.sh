make -j16 >/dev/null 2>&1 || echo BUILD FAILED
echo "== torchrun 2 ranks (gloo, one GPU) bench"
SOMB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_tr2.json 2> gpurun_out/r2_tr2.err
wc -l gpurun_out/r2_tr2.json; python -c "
import json; j=json.loads(open('gpurun_out/r2_tr2.json').read().strip().splitlines()[-1]); print(j['n_gpus'], round(j['ms_per_step'],2), j['phase_ms'], j['e2e'] and round(j['e2e']['seconds'],3))" || tail -5 gpurun_out/r2_tr2.err
echo "== reference arm under torchrun 2"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/r2_tr2_ref.json 2> gpurun_out/r2_tr2_ref.err; wc -l gpurun_out/r2_tr2_ref.json; head -c 200 gpurun_out/r2_tr2_ref.json
echo "== memcheck"
export PYTHONFAULTHANDLER=1
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests -x -q -m gpu -k "hand_cases or golden or overflow or one_call or sparse_hand or sparse_empty or auto_screen or cfg1" > gpurun_out/r2_memcheck_tests.txt 2>&1; echo "memcheck tests rc=$?"; tail -3 gpurun_out/r2_memcheck_tests.txt
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_memcheck_smoke.txt 2>&1; echo "memcheck smoke rc=$?"; tail -3 gpurun_out/r2_memcheck_smoke.txt
timeout 900 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_racecheck_smoke.txt 2>&1; echo "racecheck smoke rc=$?"; tail -4 gpurun_out/r2_racecheck_smoke.txt
