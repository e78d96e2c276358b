make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py --config cfg3 --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/w_cfg3.json 2> gpurun_out/w_cfg3.err
python -c "
import json; j=json.load(open('gpurun_out/w_cfg3.json')); print(j['ms_per_step'], j['phase_ms'])"
tail -3 gpurun_out/w_cfg3.err
