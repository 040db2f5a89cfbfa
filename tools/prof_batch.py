"""Profile one lockstep batch (host vs device time, launches)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_2012_03683_b200 import api, synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctx = api.default_context()
Xs, Zs, inits = bench.make_workload(0, B, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
dX = [api.DeviceCloud(x, ctx) for x in Xs]
dZ = [api.DeviceCloud(z, ctx) for z in Zs]
for r in range(reps):
    ctx.reset_stats()
    ctx.set_profiling(True)
    t = time.time()
    res, st = api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)
    dt = time.time() - t
    s = ctx.sweep_stats()
    h = ctx.host_stats()
    print(f"B={B} {dt:.3f}s {B / dt:.2f} reg/s rounds={h['rounds']} prep={h['t_prepare_s']:.3f} "
          f"(build {h['t_build_prep_s']:.3f} sweep {h['t_sweep_prep_s']:.3f}) solver={h['t_solver_s']:.3f} "
          f"wait={h['t_wait_s']:.3f} allocs={h['device_allocs']} ({h['device_alloc_bytes'] / 1e9:.2f} GB) "
          f"sweep_ms={s['sweep_ms']:.1f} launches={ctx.kernel_launches()} iters={[x.iterations for x in res]}", flush=True)
