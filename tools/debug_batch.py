import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2012_03683_b200 import api, synth
import bench
B = int(os.environ.get("B", "8"))
ctx = api.Context(0)
Xs, Zs, inits = bench.make_workload(0, B, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
dX = [api.DeviceCloud(x, ctx) for x in Xs]
dZ = [api.DeviceCloud(z, ctx) for z in Zs]
for rep in range(int(os.environ.get("REPS", "2"))):
    t = time.time()
    res, st = api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)
    ctx.synchronize()
    dt = time.time() - t
    print(f"B={B} rep {rep}: {dt:.3f} s, {B/dt:.1f} reg/s, st {set(st.tolist())}, it {[r.iterations for r in res][:6]}", ctx.host_stats(), flush=True)
