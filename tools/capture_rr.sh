make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 600 ncu --set full --import-source on --clock-control none -k regex:rerank_group -s 4 -c 1 \
    -o gpurun_out/r2_ncu_rgroup_cfg2 python tools/prof_cfg.py cfg2 4 > gpurun_out/r2_caprg.log 2>&1
timeout 600 python tools/screen_only.py 3 2 cfg5 > gpurun_out/r2_screen_only_cfg5.txt 2>&1
cat gpurun_out/r2_screen_only_cfg5.txt; tail -3 gpurun_out/r2_caprg.log
