# A/B: second accumulator set for the odd slot of each unit (KREG_SWEEP_ACC2)
for v in base acc2 base acc2; do
  if [ "$v" = "base" ]; then lib=""; else lib="paper_2012_03683_b200/_variants/$v.so"; fi
  echo "== $v"; KREG_LIB=$lib STEPS=3 timeout 300 python tools/ab_step.py 2>&1 | grep "profiling=False"
done
