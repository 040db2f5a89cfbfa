# A/B: candidates in the first (gradient) line-search batch
for k in 2 1 3 2; do
  echo "== KREG_K_FIRST=$k"; KREG_K_FIRST=$k STEPS=3 timeout 300 python tools/ab_step.py 2>&1 | grep "profiling=False"
done
