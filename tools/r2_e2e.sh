make -j16 >/dev/null 2>&1 || echo BUILD FAILED
for t in 4 8 12; do for c in 32 64; do
  SOMB_HOST_COPY_THREADS=$t SOMB_STAGE_CHUNK_MB=$c timeout 300 python tools/upload_probe.py 2>&1 | tail -1 | sed "s/^/threads $t chunk $c: /"
done; done
timeout 300 python tools/e2e_profile.py 2>&1 | tail -2
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|NUMA node"
