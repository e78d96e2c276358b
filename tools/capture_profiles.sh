# Round evidence: ncu full capture of the tcgen05 screen (cfg2, candidate-heavy
# epoch 4 state), the launch list of a short bench run, and bench lines for
# every config.  Outputs land in gpurun_out/ (summaries are copied to profiles/).
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 ncu --set full --import-source on --clock-control none -k regex:screen_tc -s 4 -c 1 \
    -o gpurun_out/ncu_screen_cfg2 python tools/prof_screen.py 1000000 1000 200 200 1 4 > gpurun_out/cap_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:sp_screen_ls -s 3 -c 1 \
    -o gpurun_out/ncu_sp_screen_cfg3 python tools/prof_sparse.py 500000 3 > gpurun_out/cap_ncu3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/cfg2_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
    > gpurun_out/cap_launch.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for c in cfg1 cfg4 cfg5 cfg3; do
  timeout 1200 python bench.py --config $c --steps 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
tail -2 gpurun_out/cap_ncu.log; for c in cfg1 cfg2 cfg3 cfg4 cfg5; do python -c "
import json; j=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(j['ms_per_step'],2), round(j['roofline']['frac'],3), j['e2e'] and round(j['e2e']['seconds'],3), j['cpu_baseline'] and '%.3g' % j['cpu_baseline']['value'])"; done
