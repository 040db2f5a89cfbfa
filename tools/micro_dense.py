"""Diagnostic: K4 dense exact cosine time at KITTI 40k (3 x 1.6e9 FP64 pair terms)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2012_03683_b200 import api, synth
X, Z, Ts = synth.kitti_pair(7, int(sys.argv[1]) if len(sys.argv) > 1 else 40000)
p = synth.kitti_params()
api.exact_cosine(X, Z, Ts, p)
t0 = time.perf_counter()
c, parts = api.exact_cosine(X, Z, Ts, p, parts=True)
dt = time.perf_counter() - t0
n = X.size() * Z.size() + X.size() ** 2 + Z.size() ** 2
print(f"n={X.size()} cosine={c:.12f} {dt * 1e3:.1f} ms  {n / dt / 1e9:.1f} G pair-terms/s (FP64)")
