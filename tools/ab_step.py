"""A/B of the device-resident bench step between library builds:
    KREG_LIB=<lib.so> python tools/ab_step.py
Prints ms per B-pair batch (warm), with and without profiling events."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
from paper_2012_03683_b200 import api, synth  # noqa: E402
import bench  # noqa: E402

B = int(os.environ.get("B", "128"))
STEPS = int(os.environ.get("STEPS", "3"))
ctx = api.Context(0)
Xs, Zs, inits = bench.make_workload(0, B, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
dX = [api.DeviceCloud(x, ctx) for x in Xs]
dZ = [api.DeviceCloud(z, ctx) for z in Zs]
for _ in range(2):
    api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)
ctx.synchronize()
for prof in (False, True):
    ctx.set_profiling(prof)
    ctx.reset_stats()
    t = time.perf_counter()
    for _ in range(STEPS):
        api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)
    ctx.synchronize()
    dt = (time.perf_counter() - t) / STEPS
    sw = ctx.sweep_stats()
    print(f"{os.path.basename(api.LIB_PATH)} profiling={prof}: {dt * 1e3:.1f} ms/step {B / dt:.1f} reg/s "
          f"sweep_ms/step {sw['sweep_ms'] / STEPS:.1f} rounds/step {sw['rounds'] / STEPS:.0f}", flush=True)
    try:
        print("  host", ctx.host_stats(), flush=True)
    except Exception as e:  # older builds
        print("  host stats n/a:", e)
