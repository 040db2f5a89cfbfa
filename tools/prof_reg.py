import os
import sys
import time

sys.path.insert(0, os.getcwd())
from paper_2012_03683_b200 import api, synth  # noqa: E402

X, Z, Ts = synth.kitti_pair(7, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
ctx = api.default_context()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for r in range(reps):
    ctx.reset_stats()
    t = time.time()
    res = api.register_clouds(X, Z, synth.perturbed(Ts, 3), p, cfg)
    print("reg", round(time.time() - t, 4), res.iterations, res.sweeps, res.rebuilds, ctx.host_stats(), flush=True)
