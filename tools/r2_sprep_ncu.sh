# ncu of the sparse exact repair scan (cfg3 epoch-1 state: ~270k truncated rows)
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 600 python tools/prof_sparse.py 500000 1 > gpurun_out/sprep_plain.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sp_exact -s 1 -c 1 \
    -o gpurun_out/sprep_ncu python tools/prof_sparse.py 500000 1 > gpurun_out/sprep_ncu.log 2>&1
tail -3 gpurun_out/sprep_ncu.log
