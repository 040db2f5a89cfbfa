# A/B of the candidate-list re-search threshold (KREG_SUP_SHRINK): first-frame batch and C3 step
for s in 1e9 2 1.5; do
  echo "== KREG_SUP_SHRINK=$s first"; KREG_SUP_SHRINK=$s timeout 600 python bench.py --workload first --batch 32 --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), 'reg/s', d['config']['mean_iterations'], 'build_ms', round(d['build']['build_ms']), 'sweep_ms', round(d['sweep']['sweep_ms']), d['build']['grid_why'], d['admission'])"
done
for s in 1e9 2; do
  echo "== KREG_SUP_SHRINK=$s C3"; KREG_SUP_SHRINK=$s STEPS=3 timeout 300 python tools/ab_step.py 2>&1 | grep "profiling=False"
done
