# A/B: F-only requests in their own launch, gradient kernel at 2 or 3 CTAs/SM
for v in base split2 split3 base split3; do
  if [ "$v" = "base" ]; then lib=""; else lib="paper_2012_03683_b200/_variants/$v.so"; fi
  echo "== $v"; KREG_LIB=$lib STEPS=3 timeout 300 python tools/ab_step.py 2>&1 | grep "profiling=False"
done
