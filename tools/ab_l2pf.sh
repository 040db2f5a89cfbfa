# A/B: L2 prefetch of the sweep units KREG_L2_PREFETCH stages ahead
for v in base l2pf1 l2pf2 l2pf4 base l2pf2; do
  if [ "$v" = "base" ]; then lib=""; else lib="paper_2012_03683_b200/_variants/$v.so"; fi
  echo "== $v"; KREG_LIB=$lib STEPS=3 timeout 300 python tools/ab_step.py 2>&1 | grep "profiling=False"
done
