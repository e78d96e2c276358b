make -j16 >/dev/null 2>&1 || echo BUILD FAILED
SOMB_TC_PREFERRED=1 timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
SOMB_TC_PREFERRED=1 timeout 900 python -m pytest tests -x -q -m gpu -k "random or one_call or cfg2_shape or hand_cases or overflow or golden" 2>&1 | tail -2
bash tools/ab_env.sh pf cfg2 SOMB_TC_PREFERRED 1 0 5
SOMB_TC_PREFERRED=1 timeout 300 python tools/screen_only.py 4 3 cfg2 2>&1 | tail -12
