# Round-2 ncu evidence for the current default build (one GPU; run under gpurun):
# --set full captures of k_sweep, k_pair_pass<1> (candidate EMIT) and
# k_filter<1> (filter EMIT) inside the bench command (steady-state rounds of
# the first step), then the bench command's launch list.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 1500 -c 1 \
  -o gpurun_out/r02_sweep_full -f $B > gpurun_out/r02_sweep_full.log 2>&1
echo "sweep rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_pair_pass --launch-skip 41 -c 1 \
  -o gpurun_out/r02_pairpass_full -f $B > gpurun_out/r02_pairpass_full.log 2>&1
echo "pairpass rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_filter --launch-skip 601 -c 1 \
  -o gpurun_out/r02_filter_full -f $B > gpurun_out/r02_filter_full.log 2>&1
echo "filter rc=$?"
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
  --log-file gpurun_out/r02_launches_bench.csv $B > gpurun_out/r02_launches.log 2>&1
echo "launches rc=$?"
gzip -f gpurun_out/r02_launches_bench.csv
