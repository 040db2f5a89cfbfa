mkdir -p gpurun_out
for lib in paper_2012_03683_b200/libkreg_b200.so paper_2012_03683_b200/_variants/${AB_GLOB:-ring_*}.so paper_2012_03683_b200/libkreg_b200.so; do
  n=$(basename $lib .so)
  KREG_LIB=$PWD/$lib timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "golden or deterministic" > gpurun_out/ab_$n.test 2>&1
  echo "$n test rc=$?" >> gpurun_out/ab_summary.txt
  KREG_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_$n.json 2> gpurun_out/ab_$n.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$n.json').read().strip().splitlines()[-1]); print('$n', round(d['value'],2), round(d['e2e']['value'],2), round(d['roofline']['frac'],3))" >> gpurun_out/ab_summary.txt 2>&1
done
cat gpurun_out/ab_summary.txt
