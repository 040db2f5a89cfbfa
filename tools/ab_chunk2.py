"""A/B of the sweep chunk size (units) with the default two stream groups:
    python tools/ab_chunk2.py 48 64 96"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
from paper_2012_03683_b200 import api, synth  # noqa: E402
import bench  # noqa: E402

B, STEPS = 128, 3
ctx = api.Context(0)
Xs, Zs, inits = bench.make_workload(0, B, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
dX = [api.DeviceCloud(x, ctx) for x in Xs]
dZ = [api.DeviceCloud(z, ctx) for z in Zs]
for rep in range(2):
    for cu in [int(a) for a in sys.argv[1:]]:
        ctx.set_chunk_units(cu)
        api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)  # lists rebuilt with this chunking
        ctx.synchronize()
        t = time.perf_counter()
        for _ in range(STEPS):
            api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)
        ctx.synchronize()
        dt = (time.perf_counter() - t) / STEPS
        print(f"chunk {cu}: {dt * 1e3:.1f} ms/step {B / dt:.1f} reg/s", flush=True)
