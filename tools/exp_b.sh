make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 300 python tools/epoch_profile.py cfg2 > gpurun_out/b_cfg2.txt 2>&1
timeout 300 python tools/epoch_profile.py cfg4 1 > gpurun_out/b_cfg4_p1.txt 2>&1
timeout 300 python tools/epoch_profile.py cfg4 3 > gpurun_out/b_cfg4_p3.txt 2>&1
timeout 300 python tools/epoch_profile.py cfg5 3 > gpurun_out/b_cfg5_p3.txt 2>&1
tail -n 11 gpurun_out/b_*.txt
