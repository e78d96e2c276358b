# sparse exact repair with half of the conversions off the XU pipe: parity, cfg3 e2e, ncu of the repair
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -x -q -k "sparse or cfg3" 2>&1 | tail -3
timeout 900 python bench.py --config cfg3 --steps 3 --no-cpu-baseline > gpurun_out/sprep_cfg3.json 2> gpurun_out/sprep_cfg3.err
python -c "
import json; j=json.load(open('gpurun_out/sprep_cfg3.json')); print('cfg3', round(j['ms_per_step'],2), j['e2e']['seconds'], {k: round(v,2) for k,v in j['phase_ms'].items()})" || tail -5 gpurun_out/sprep_cfg3.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sp_exact -s 1 -c 1 \
    -o gpurun_out/sprep2_ncu python tools/prof_sparse.py 500000 1 > gpurun_out/sprep2_ncu.log 2>&1
tail -1 gpurun_out/sprep2_ncu.log
