make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 ncu --set full --clock-control none -k regex:dgemm_mma -s 6 -c 3 -o gpurun_out/ncu_dgemm_cfg5 python tools/epoch_profile.py cfg5 > gpurun_out/x_ncu.log 2>&1
tail -2 gpurun_out/x_ncu.log
