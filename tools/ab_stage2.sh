# A/B: end-to-end staging workers with the default two stream groups
for w in default 4 8 default 4 8; do
  if [ "$w" = "default" ]; then unset KREG_STAGE_WORKERS; else export KREG_STAGE_WORKERS=$w; fi
  echo "== workers $w"; timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), 'device', round(d['e2e']['value'],2), 'e2e')"
done
