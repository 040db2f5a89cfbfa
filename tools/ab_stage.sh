# A/B: end-to-end staging workers (KREG_STAGE_WORKERS) and two-group rounds
for w in default 6 10 default; do
  if [ "$w" = "default" ]; then unset KREG_STAGE_WORKERS; else export KREG_STAGE_WORKERS=$w; fi
  echo "== workers $w"; timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), 'device', round(d['e2e']['value'],2), 'e2e')"
done
unset KREG_STAGE_WORKERS
echo "== KREG_GROUPS=2"; KREG_GROUPS=2 timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), 'device', round(d['e2e']['value'],2), 'e2e')"
