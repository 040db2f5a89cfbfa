# Round-2 hand-run measurements (one GPU; run under gpurun): every bench mode
# plus the reference arm's modes, one JSON line each under gpurun_out/.
mkdir -p gpurun_out
run() { local name=$1; shift; timeout ${T:-900} python bench.py "$@" > gpurun_out/r02_$name.json 2> gpurun_out/r02_$name.err; echo "$name rc=$?"; tail -c 600 gpurun_out/r02_$name.json; echo; }
run latency --mode latency --steps 24 --warmup 3 --no-cpu-baseline
run first --workload first --batch 32 --steps 1 --warmup 1 --no-cpu-baseline
run c5 --workload c5 --frames 1025 --chains 32 --steps 1 --warmup 1 --no-cpu-baseline
timeout 900 python bench_c4.py > gpurun_out/r02_c4.json 2> gpurun_out/r02_c4.err; echo "c4 rc=$?"; tail -c 600 gpurun_out/r02_c4.json
