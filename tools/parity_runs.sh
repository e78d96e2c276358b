# Full-scale exactness sweep (tools/parity_sweep.py) over data families and configs.
make -j16 >/dev/null 2>&1 || echo BUILD FAILED
run() { timeout ${T:-900} python tools/parity_sweep.py "$@" 2>&1 | grep SUMMARY || echo "FAILED/TIMEOUT $*"; }
for f in uniform dupcols blobs onehot10 int05 offset1000 rank4 nearconst; do run cfg2 $f; done
for f in uniform dupcols blobs onehot10 int05 offset1000 rank4; do run cfg5 $f; done
T=1500 run cfg5 nearconst 400000
for f in uniform blobs nearconst; do run cfg4 $f; done
T=1500 run cfg3 sparse
