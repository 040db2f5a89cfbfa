import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2012_03683_b200 import api, synth
from paper_2012_03683_b200.types import *
ctx = api.default_context()
X, Z, Ts = synth.kitti_pair(7, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
init = synth.perturbed(Ts, 3)
for rep in range(3):
    t = time.time(); res = api.register_clouds(X, Z, init, p, cfg); dt = time.time() - t
    print("single reg", dt, res.iterations, res.converged, res.sweeps, res.rebuilds, flush=True)
err = compose(inverse(res.transform), Ts); print("err", rotation_angle(err), translation_norm(err))
for B in (8, 32):
    Xs, Zs, inits = [], [], []
    for b in range(B):
        Xs.append(X); Zs.append(Z); inits.append(synth.perturbed(Ts, 100 + b))
    t = time.time(); out, st = api.register_batch(Xs, Zs, inits, p, cfg); dt = time.time() - t
    print("batch", B, dt, B / dt, "reg/s", [o.iterations for o in out][:4], flush=True)
ctx.set_profiling(True); ctx.reset_stats()
res = api.register_clouds(X, Z, init, p, cfg)
print(ctx.sweep_stats(), ctx.kernel_launches())
