"""Diagnostic: single-registration latency (one KITTI 40k pair at a time)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import bench
from paper_2012_03683_b200 import api, synth
ctx = api.default_context()
Xs, Zs, inits = bench.make_workload(0, 6, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
dX = [api.DeviceCloud(x, ctx) for x in Xs]; dZ = [api.DeviceCloud(z, ctx) for z in Zs]
api.register_clouds(dX[0], dZ[0], inits[0], p, cfg, ctx=ctx)
ctx.reset_stats(); ctx.set_profiling(True)
t0 = time.perf_counter(); its = 0
for k in range(1, 6):
    r = api.register_clouds(dX[k], dZ[k], inits[k], p, cfg, ctx=ctx); its += r.iterations
dt = time.perf_counter() - t0
h, s = ctx.host_stats(), ctx.sweep_stats()
print(f"latency mode: {dt / 5 * 1e3:.1f} ms per registration ({5 / dt:.1f} reg/s), {its / 5:.0f} it, rounds {h['rounds'] / 5:.0f}, "
      f"prepare {h['t_prepare_s'] / 5 * 1e3:.1f} ms, wait {h['t_wait_s'] / 5 * 1e3:.1f} ms, sweep {s['sweep_ms'] / 5:.1f} ms per registration")
