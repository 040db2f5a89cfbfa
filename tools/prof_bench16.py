import os, sys
sys.path.insert(0, os.getcwd())
import bench
from paper_2012_03683_b200 import api, synth
ctx = api.default_context()
Xs, Zs, inits = bench.make_workload(0, 16, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
dX = [api.DeviceCloud(x, ctx) for x in Xs]; dZ = [api.DeviceCloud(z, ctx) for z in Zs]
res, st = api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)
print([r.iterations for r in res])
