"""One warm B-pair batch with profiling counters: device ms of sweeps and
builds, rounds, host turnaround (no ncu)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2012_03683_b200 import api, synth
import bench
B = int(os.environ.get("B", "128"))
ctx = api.Context(0)
Xs, Zs, inits = bench.make_workload(0, B, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
dX = [api.DeviceCloud(x, ctx) for x in Xs]
dZ = [api.DeviceCloud(z, ctx) for z in Zs]
api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)
ctx.synchronize()
ctx.reset_stats()
ctx.set_profiling(True)
t = time.time()
res, st = api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)
ctx.synchronize()
dt = time.time() - t
sw = ctx.sweep_stats()
bp = ctx.build_stats()
print(f"B={B}: {dt:.3f} s  {B/dt:.1f} reg/s  sweep {sw}  build {bp}")
print("host", ctx.host_stats())
