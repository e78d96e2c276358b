# column-block-major node sums: kernels, 2-rank gloo through CUDA, 1-rank NCCL exchange, then the full GPU suite
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "column_blocks or node_sums or sparse" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -3
SOMB_EXCHANGE=always timeout 600 python bench.py --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/cols_bench_nccl1.json 2> gpurun_out/cols_bench_nccl1.err
python -c "
import json; j=json.load(open('gpurun_out/cols_bench_nccl1.json')); print('nccl1', round(j['ms_per_step'],2), {k: round(v,2) for k,v in j['phase_ms'].items()})" || tail -5 gpurun_out/cols_bench_nccl1.err
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
