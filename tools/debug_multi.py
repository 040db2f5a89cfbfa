import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2012_03683_b200 import api, synth
import bench
B = int(os.environ.get("B", "4"))
ctx = api.Context(0)
Xs, Zs, inits = bench.make_workload(0, B, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
cfg.max_iterations = int(os.environ.get("IT", "1"))
single = [api.register_clouds(Xs[k], Zs[k], inits[k], p, cfg, ctx=ctx) for k in range(B)]
for rep in range(3):
    res, st = api.register_batch(Xs, Zs, inits, p, cfg, ctx=ctx)
    for k in range(B):
        a, b = single[k].objective_trace, res[k].objective_trace
        m = min(len(a), len(b))
        d = np.nonzero(a[:m] != b[:m])[0]
        print(rep, k, "it", len(a), len(b), "first diff", d[:3], (a[d[0]], b[d[0]]) if len(d) else "", "pairs", single[k].pair_count_trace[:2], res[k].pair_count_trace[:2], flush=True)
