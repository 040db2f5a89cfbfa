"""Step-time breakdown of the batched registration for several candidate-list
skins (diagnostic; not part of the product)."""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import bench
from paper_2012_03683_b200 import api, synth

B = int(os.environ.get("B", "32"))
skins = [float(s) for s in os.environ.get("SKINS", "0,0.25,0.5,1.0").split(",")]
ctx = api.default_context()
if os.environ.get("W"):
    ctx.set_max_active(int(os.environ["W"]))
Xs, Zs, inits = bench.make_workload(0, B, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
dX = [api.DeviceCloud(x, ctx) for x in Xs]
dZ = [api.DeviceCloud(z, ctx) for z in Zs]
api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)  # warm-up / workspace growth
for skin in skins:
    ctx.set_candidate_skin(skin)
    api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)
    ctx.reset_stats()
    h0 = ctx.host_stats()
    ctx.set_profiling(True)
    ctx.synchronize()
    t0 = time.perf_counter()
    res, st = api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)
    ctx.synchronize()
    dt = time.perf_counter() - t0
    ctx.set_profiling(False)
    h, s, b = ctx.host_stats(), ctx.sweep_stats(), ctx.build_stats()
    its = [r.iterations for r in res]
    print(json.dumps({"skin": skin, "B": B, "s": round(dt, 4), "reg_per_s": round(B / dt, 2),
                      "mean_it": sum(its) / len(its), "rounds": h["rounds"], "t_prepare": round(h["t_prepare_s"], 4),
                      "t_wait": round(h["t_wait_s"], 4), "t_solver": round(h["t_solver_s"], 4),
                      "t_build_prep": round(h["t_build_prep_s"], 4), "t_sweep_prep": round(h["t_sweep_prep_s"], 4),
                      "sweep_ms": round(s["sweep_ms"], 1), "pairs_streamed": s["pairs_streamed"],
                      "slots_streamed": s["slots_streamed"], "pair_evals": s["pair_evals"], "builds": b, "allocs": h["device_allocs"] - h0["device_allocs"],
                      "alloc_s": round(h["device_alloc_s"] - h0["device_alloc_s"], 4),
                      "launches": ctx.kernel_launches()}), flush=True)
