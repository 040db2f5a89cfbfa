for v in base nofence prefetch sepreduce all3 base; do
  if [ "$v" = "base" ]; then lib=""; else lib="paper_2012_03683_b200/_variants/$v.so"; fi
  echo "== $v"; KREG_LIB=$lib STEPS=3 timeout 300 python tools/ab_step.py 2>&1 | grep "profiling=False"
done
timeout 600 python -m pytest tests/test_facade.py -m gpu -x -q 2>&1 | tail -30
