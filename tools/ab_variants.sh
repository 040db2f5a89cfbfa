#!/bin/bash
# A/B of kernel variants (paper_2012_03683_b200/_variants/*.so) on the batched benchmark workload
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=""; else lib="paper_2012_03683_b200/_variants/$v.so"; fi
  echo "== $v"
  KREG_LIB=$lib B=${B:-64} SKINS=0.25 python tools/prof_skin.py 2>&1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['reg_per_s'], d['sweep_ms'], d['s'], round(d['builds'].get('build_ms', 0), 1))"
  KREG_LIB=$lib python tools/micro_sweep.py 2>&1 | grep "M=2" | head -3
done
