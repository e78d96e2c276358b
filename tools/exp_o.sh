make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rerank_pipe -s 4 -c 1 -o gpurun_out/ncu_rerank_pipe2 python tools/prof_screen.py 1000000 1000 200 200 1 4 > gpurun_out/o_ncu.log 2>&1
tail -2 gpurun_out/o_ncu.log
