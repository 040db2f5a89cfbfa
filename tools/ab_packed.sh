# A/B of the mixed slot formats (12-B packed slots for high-degree lists):
# C3 step (never packed: degree 64) vs the previous build, then the
# first-frame batch with packing on / off.
for v in prev base prev base; do
  if [ "$v" = "base" ]; then lib=""; else lib="paper_2012_03683_b200/_variants/$v.so"; fi
  echo "== $v C3"; KREG_LIB=$lib STEPS=3 timeout 300 python tools/ab_step.py 2>&1 | grep "profiling=False"
done
for d in -1 256; do
  echo "== KREG_PACKED_DEGREE=$d first"; KREG_PACKED_DEGREE=$d timeout 600 python bench.py --workload first --batch 32 --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), 'reg/s', d['config']['mean_iterations'], 'build_ms', round(d['build']['build_ms']), 'sweep_ms', round(d['sweep']['sweep_ms']), 'slots', d['sweep']['slots_streamed'], d['clocks'])"
done
