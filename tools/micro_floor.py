"""Diagnostic: sweep time vs pair-list size (fixed per-launch cost)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
from paper_2012_03683_b200 import api, synth  # noqa: E402

ctx = api.default_context()
pk = synth.kitti_params()
X0, Z0, T0 = synth.kitti_pair(7, 40000)
warm = api.build_pairs(X0, Z0, T0, pk.with_lengthscale(0.1), 3.0, 1e-4)
t0 = time.time()
while time.time() - t0 < 1.0:
    api.eval_transforms(warm, X0, Z0, [T0], pk.with_lengthscale(0.1))
for n in (64, 1000, 5000, 20000, 40000):
    X, Z, Ts = synth.kitti_pair(7, n)
    pr = api.build_pairs(X, Z, Ts, pk.with_lengthscale(0.1), 3.0, 1e-4)
    for _ in range(3):
        api.eval_transforms(pr, X, Z, [Ts], pk.with_lengthscale(0.1))
    ctx.set_profiling(True)
    ctx.reset_stats()
    N = 50
    t1 = time.perf_counter()
    for _ in range(N):
        api.eval_transforms(pr, X, Z, [Ts], pk.with_lengthscale(0.1))
    wall = (time.perf_counter() - t1) / N * 1e6
    s = ctx.sweep_stats()
    ctx.set_profiling(False)
    print(f"n={n:6d} P={pr.size():8d} sweep {s['sweep_ms'] / N * 1e3:7.2f} us (events)  call {wall:7.1f} us wall", flush=True)
