make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rerank_vec -s 4 -c 1 -o gpurun_out/ncu_rerank_heavy python tools/prof_screen.py 1000000 1000 200 200 1 4 > gpurun_out/g_ncu.log 2>&1
tail -3 gpurun_out/g_ncu.log
for k in 8 10 12; do timeout 600 python tools/trunc_check.py 9 $k > gpurun_out/g_trunc_k$k.txt 2>&1; done
tail -n 9 gpurun_out/g_trunc_k*.txt
