"""Diagnostic: end-to-end (host buffers) vs device-resident batch, with host phase times."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import bench
from paper_2012_03683_b200 import api, synth
B = int(os.environ.get("B", "128"))
ctx = api.default_context()
Xs, Zs, inits = bench.make_workload(0, B, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
for it in range(2):
    ctx.reset_stats(); ctx.synchronize()
    t0 = time.perf_counter()
    t_py = time.perf_counter()
    res, st = api.register_batch_host(Xs, Zs, inits, p, cfg, ctx=ctx)
    ctx.synchronize()
    dt = time.perf_counter() - t0
    h = ctx.host_stats()
    print(f"e2e B={B} {dt:.3f} s ({B / dt:.1f} reg/s) stage={h['t_sweep_prep_s']:.3f} prepare={h['t_prepare_s']:.3f} "
          f"build_prep={h['t_build_prep_s']:.3f} wait={h['t_wait_s']:.3f} solver={h['t_solver_s']:.3f} rounds={h['rounds']} "
          f"allocs={h['device_allocs']} alloc_s={h['device_alloc_s']:.3f} builds={ctx.build_stats()}", flush=True)
dX = [api.DeviceCloud(x, ctx) for x in Xs]; dZ = [api.DeviceCloud(z, ctx) for z in Zs]
api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)
ctx.reset_stats(); ctx.synchronize(); t0 = time.perf_counter()
api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx); ctx.synchronize(); dt = time.perf_counter() - t0
h = ctx.host_stats()
print(f"device B={B} {dt:.3f} s ({B / dt:.1f} reg/s) prepare={h['t_prepare_s']:.3f} wait={h['t_wait_s']:.3f} solver={h['t_solver_s']:.3f}")
