# ncu evidence for the current default build (one GPU; run under gpurun):
# one --set full capture of a k_sweep launch in the bench command, then the
# bench command's launch list (first 20000 launches).
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 3000 -c 1 \
  -o gpurun_out/sweep_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_full.log 2>&1
echo "full rc=$?"
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/launches.log 2>&1
echo "launches rc=$?"
gzip -f gpurun_out/launches_bench.csv
