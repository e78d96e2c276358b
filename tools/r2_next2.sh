make -j16 >/dev/null 2>&1 || echo BUILD FAILED
bash tools/ab.sh ab5 cfg4 3
bash tools/ab.sh ab5 cfg2 5
SOMB_EXCHANGE=always timeout 900 python bench.py --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/nccl1_cfg2.json 2> gpurun_out/nccl1_cfg2.err
python -c "
import json; j=json.load(open('gpurun_out/nccl1_cfg2.json')); print('nccl1 cfg2', round(j['ms_per_step'],2), {k: round(v,2) for k,v in j['phase_ms'].items()})" || tail -5 gpurun_out/nccl1_cfg2.err
timeout 900 python -m pytest tests -x -q -m gpu -k "cfg1 or hand_cases or golden or overflow or one_call or dist" 2>&1 | tail -3
