# A/B: K4 dense target points per inner iteration (KREG_DENSE_J)
for v in base dense2 dense4 base; do
  if [ "$v" = "base" ]; then lib=""; else lib="paper_2012_03683_b200/_variants/$v.so"; fi
  echo "== $v"; KREG_LIB=$lib python tools/micro_dense.py; KREG_LIB=$lib python tools/micro_dense.py
done
