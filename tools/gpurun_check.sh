# One gpurun pass: build, -m gpu tests, smoke, cfg2 bench.  Usage: bash tools/gpurun_check.sh TAG
TAG=${1:-chk}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -40 > gpurun_out/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench_cfg2.json 2> gpurun_out/${TAG}_bench_cfg2.err
cat gpurun_out/${TAG}_pytest_gpu.txt gpurun_out/${TAG}_smoke.txt gpurun_out/${TAG}_bench_cfg2.json; tail -5 gpurun_out/${TAG}_bench_cfg2.err
