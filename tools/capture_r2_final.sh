# Round-2 final evidence: bench lines for every config, ncu of the screens
# (cfg2 1-pass, cfg4 1-pass, cfg5 2-pass) and the re-rank, and the cfg2 launch list.
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 ncu --set full --import-source on --clock-control none -k regex:screen_tc -s 4 -c 1 \
    -o gpurun_out/r2f_ncu_screen_cfg2 python tools/prof_cfg.py cfg2 4 > gpurun_out/r2f_cap2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rerank -s 4 -c 1 \
    -o gpurun_out/r2f_ncu_rerank_cfg2 python tools/prof_cfg.py cfg2 4 > gpurun_out/r2f_capr.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:screen_tc -s 3 -c 1 \
    -o gpurun_out/r2f_ncu_screen_cfg4 python tools/prof_cfg.py cfg4 3 > gpurun_out/r2f_cap4.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:screen_tc -s 3 -c 1 \
    -o gpurun_out/r2f_ncu_screen_cfg5 python tools/prof_cfg.py cfg5 3 > gpurun_out/r2f_cap5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2f_cfg2_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
    > gpurun_out/r2f_cap_launch.log 2>&1
for c in cfg2 cfg1 cfg4 cfg5 cfg3; do
  timeout 1500 python bench.py --config $c > gpurun_out/r2f_bench_$c.json 2> gpurun_out/r2f_bench_$c.err
done
timeout 900 python bench.py --impl reference > gpurun_out/r2f_bench_ref_cfg2.json 2> gpurun_out/r2f_bench_ref_cfg2.err
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do python -c "
import json; j=json.load(open('gpurun_out/r2f_bench_$c.json')); print('$c', round(j['ms_per_step'],2), round(j['roofline']['frac'],3), j['e2e'] and round(j['e2e']['seconds'],3), j['cpu_baseline'] and '%.3g' % j['cpu_baseline']['value'], {k: round(v,2) for k,v in j['phase_ms'].items()})" || tail -3 gpurun_out/r2f_bench_$c.err; done
head -c 300 gpurun_out/r2f_bench_ref_cfg2.json
