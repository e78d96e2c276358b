make -j16 >/dev/null 2>&1 || echo BUILD FAILED
run() { timeout ${T:-900} python tools/parity_sweep.py "$@" 2>&1 | grep SUMMARY || echo "FAILED/TIMEOUT $*"; }
for f in uniform blobs dupcols onehot10 int05 offset1000 rank4; do run cfg4 $f; done
T=1500 run cfg4 nearconst 500000
timeout 900 python -m pytest tests -x -q -m gpu -k "cfg4 or extensions or hex" 2>&1 | tail -2
