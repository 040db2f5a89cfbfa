# A/B: one lockstep group vs two groups on two streams (KREG_GROUPS=2)
for g in 1 2 1 2; do
  echo "== KREG_GROUPS=$g"; KREG_GROUPS=$g STEPS=3 timeout 300 python tools/ab_step.py 2>&1 | grep "profiling=False"
done
