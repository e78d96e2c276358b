# ncu captures of the final kernels: the A-resident screens (cfg4 1-pass, cfg5 2-pass) and the all-F2F re-rank (cfg2)
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 ncu --set full --clock-control none -k regex:screen_tc -s 3 -c 1 \
    -o gpurun_out/r2k_ncu_screen_cfg4 python tools/prof_cfg.py cfg4 3 > gpurun_out/r2k_cap4.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:screen_tc -s 3 -c 1 \
    -o gpurun_out/r2k_ncu_screen_cfg5 python tools/prof_cfg.py cfg5 3 > gpurun_out/r2k_cap5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rerank -s 4 -c 1 \
    -o gpurun_out/r2k_ncu_rerank_cfg2 python tools/prof_cfg.py cfg2 4 > gpurun_out/r2k_capr.log 2>&1
ls gpurun_out/r2k_*
