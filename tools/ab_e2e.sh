# A/B of the end-to-end bench number (host staging changes) vs the previous build
for v in prev base prev base; do
  if [ "$v" = "base" ]; then lib=""; else lib="paper_2012_03683_b200/_variants/$v.so"; fi
  echo "== $v"; KREG_LIB=$lib timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), 'device', round(d['e2e']['value'],2), 'e2e')"
done
