# A/B of the bench (device + e2e): two vs four round groups
for g in 2 4 2 4 2 4 2 4; do
  echo "== KREG_GROUPS=$g"; KREG_GROUPS=$g timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), 'device', round(d['e2e']['value'],2), 'e2e')"
done
