make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 600 python tools/screen_only.py 3 2 cfg5 > gpurun_out/r2_screen_only_cfg5_b.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:screen_tc -c 1 \
    -o gpurun_out/r2_ncu_screen_cfg5_b python tools/prof_cfg.py cfg5 3 > gpurun_out/r2_cap5b.log 2>&1
cat gpurun_out/r2_screen_only_cfg5_b.txt; tail -1 gpurun_out/r2_cap5b.log
