# A/B: C5 end to end with frames staged in order vs interleaved across chains
for v in prev base; do
  if [ "$v" = "base" ]; then lib=""; else lib="paper_2012_03683_b200/_variants/$v.so"; fi
  echo "== $v"; KREG_LIB=$lib timeout 900 python bench.py --workload c5 --frames 1025 --chains 32 --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), 'device', round(d['e2e']['value'],2), 'e2e')"
done
timeout 600 python -m pytest tests/test_gpu_schedules.py -m gpu -q -k "host" 2>&1 | tail -2
