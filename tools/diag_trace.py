"""Diagnostic: GPU vs reference registration traces on one KITTI pair."""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from paper_2012_03683_b200 import api, synth
from _checkers import Reference
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 7
X, Z, Ts = synth.kitti_pair(seed, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
init = synth.perturbed(Ts, 3)
g = api.register_clouds(X, Z, init, p, cfg)
r = Reference(); r.set_threads(os.cpu_count())
c = r.register_clouds(X, Z, init, p, cfg)
print("iterations gpu", g.iterations, "ref", c.iterations, "conv", g.converged, c.converged)
n = min(g.iterations, c.iterations)
ls_g, ls_c = np.array(g.lengthscale_trace), np.array(c.lengthscale_trace)
print("levels gpu", len(np.unique(ls_g)), "ref", len(np.unique(ls_c)))
for lv in sorted(set(ls_c.tolist()) | set(ls_g.tolist()), reverse=True)[:40]:
    print(f"l={lv:.6f} it gpu {np.sum(ls_g == lv):4d} ref {np.sum(ls_c == lv):4d}")
d = np.abs(np.array(g.objective_trace[:n]) - np.array(c.objective_trace[:n])) / np.abs(np.array(c.objective_trace[:n]))
k = int(np.argmax(d > 1e-6)) if np.any(d > 1e-6) else n
print("first iteration with rel F diff > 1e-6:", k)
for i in range(max(0, k - 3), min(n, k + 5)):
    print(i, g.objective_trace[i], c.objective_trace[i], g.step_trace[i], c.step_trace[i], g.rebuild_trace[i], c.rebuild_trace[i])
