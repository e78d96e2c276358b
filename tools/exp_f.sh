make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 300 python tools/epoch_profile.py cfg2 > gpurun_out/f_prof.txt 2>&1
timeout 600 python tools/trunc_check.py 9 > gpurun_out/f_trunc.txt 2>&1
timeout 300 python tools/epoch_profile.py cfg5 > gpurun_out/f_prof5.txt 2>&1
timeout 900 python tools/full_parity.py 1000000 10 > gpurun_out/f_full.txt 2>&1
cat gpurun_out/f_prof.txt gpurun_out/f_trunc.txt gpurun_out/f_prof5.txt gpurun_out/f_full.txt
