"""Diagnostic: reference CPU throughput modes on this host (latency vs pairs-parallel)."""
import os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import bench
from paper_2012_03683_b200 import synth
from _checkers import Reference
r = Reference()
cores = os.cpu_count()
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
Xs, Zs, inits = bench.make_workload(0, cores, 40000)
r.set_threads(cores)
t0 = time.perf_counter(); r.register_clouds(Xs[0], Zs[0], inits[0], p, cfg); t1 = time.perf_counter()
print("latency mode:", cores, "threads", 1 / (t1 - t0), "reg/s", flush=True)
t0 = time.perf_counter(); r.register_batch(Xs, Zs, inits, p, cfg); t1 = time.perf_counter()
print("throughput mode:", cores, "pairs", cores / (t1 - t0), "reg/s", flush=True)
