# Round-2 evidence: ncu full captures (source-level) of the cfg5 split screen,
# the cfg2 re-rank, and the cfg2 update kernels (node sums, radix sort,
# spectral DMMA GEMMs, blend).  Outputs land in gpurun_out/.
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 ncu --set full --import-source on --clock-control none -k regex:screen_tc -c 1 \
    -o gpurun_out/r2_ncu_screen_cfg5 python tools/prof_cfg.py cfg5 3 > gpurun_out/r2_cap5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rerank -c 1 \
    -o gpurun_out/r2_ncu_rerank_cfg2 python tools/prof_cfg.py cfg2 4 > gpurun_out/r2_capr.log 2>&1
timeout 900 ncu --set full --clock-control none \
    -k "regex:seg_sum|seg_fold|seg_plan|radix|bucket|exclusive_scan|dgemm|hood|spec_|blend|occ_" -c 40 \
    -o gpurun_out/r2_ncu_update_cfg2 python tools/prof_cfg.py cfg2 1 > gpurun_out/r2_capu.log 2>&1
ls -la gpurun_out/
