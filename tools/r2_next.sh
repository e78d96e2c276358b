make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 600 python -m pytest tests -x -q -m gpu -k "grouped_rerank or overflow or hand_cases or one_call or golden or cfg1" 2>&1 | tail -2
SOMB_SCREEN_DEFER=1 timeout 900 python -m pytest tests -x -q -m gpu -k "hand_cases or golden or overflow or cfg1 or random or shape_all" 2>&1 | tail -2
bash tools/ab_env.sh df cfg5 SOMB_SCREEN_DEFER 1 0
bash tools/ab_env.sh df cfg4 SOMB_SCREEN_DEFER 1 0
bash tools/ab_env.sh df cfg2 SOMB_SCREEN_DEFER 1 0 5
CFGS="cfg2 cfg5 cfg4" bash tools/ab3.sh 2>&1 | grep group=
SOMB_EXCHANGE=always timeout 900 python bench.py --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/nccl1_cfg2.json 2> gpurun_out/nccl1_cfg2.err
python -c "
import json; j=json.load(open('gpurun_out/nccl1_cfg2.json')); print('nccl1 cfg2', round(j['ms_per_step'],2), {k: round(v,2) for k,v in j['phase_ms'].items()})" || tail -5 gpurun_out/nccl1_cfg2.err
