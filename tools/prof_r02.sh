# Round-2 ncu evidence for the current default build (one GPU; run under gpurun;
# build first: python -m paper_2012_03683_b200.build):
# --set full captures of k_sweep (bench command, steady-state round of the
# first step), k_filter<1> and the K4 dense kernel, then the bench command's
# launch list.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 1500 -c 1 \
  -o gpurun_out/r02_sweep_full -f $B > gpurun_out/r02_sweep_full.log 2>&1
echo "sweep rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_filter --launch-skip 601 -c 1 \
  -o gpurun_out/r02_filter_full -f $B > gpurun_out/r02_filter_full.log 2>&1
echo "filter rc=$?"
timeout 600 python tools/micro_dense.py > gpurun_out/r02_dense_time.txt 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:dense -c 1 \
  -o gpurun_out/r02_dense_full -f python tools/micro_dense.py > gpurun_out/r02_dense_full.log 2>&1
echo "dense rc=$?"
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
  --log-file gpurun_out/r02_launches_bench.csv $B > gpurun_out/r02_launches.log 2>&1
echo "launches rc=$?"
gzip -f gpurun_out/r02_launches_bench.csv
