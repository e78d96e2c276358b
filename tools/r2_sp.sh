make -j16 >/dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests -x -q -m gpu -k "sparse" 2>&1 | tail -2
timeout 600 python tools/e2e_sparse_phases.py 2>&1 | tail -2
timeout 1500 python tools/parity_sweep.py cfg3 sparse 2>&1 | grep -E "SUMMARY|epoch\": 1,"
