make -j16 >/dev/null 2>&1 || echo BUILD FAILED
SOMB_A_RESIDENT=1 timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
SOMB_A_RESIDENT=1 timeout 1200 python -m pytest tests -x -q -m gpu -k "hand_cases or golden or overflow or cfg1 or random or cfg4_shape or cfg5_shape or auto_screen or one_call" 2>&1 | tail -2
bash tools/ab_env.sh ar cfg5 SOMB_A_RESIDENT 1 0
bash tools/ab_env.sh ar cfg4 SOMB_A_RESIDENT 1 0
for hc in 16; do
  SOMB_HALF_CAP=$hc bash tools/ab_env.sh arh$hc cfg5 SOMB_A_RESIDENT 1 0
  SOMB_HALF_CAP=$hc bash tools/ab_env.sh arh$hc cfg4 SOMB_A_RESIDENT 1 0
done
