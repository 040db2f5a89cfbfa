"""Diagnostic: first-frame schedule (l = 0.95) device vs reference, decision by
decision; prints the first diverging iteration and the trace context."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from _checkers import Reference  # noqa: E402
from paper_2012_03683_b200 import api, synth  # noqa: E402
from paper_2012_03683_b200.types import Isometry, compose, inverse, rotation_angle, translation_norm  # noqa: E402

n = int(os.environ.get("N", "8000"))
seq = os.environ.get("SEQ")
r = Reference()
r.set_threads(os.cpu_count())
if seq:
    frames, _ = synth.kitti_sequence(5, 6, n)
    X, Z = frames[0], frames[1]
else:
    X, Z, _ = synth.kitti_pair(7, n)
p, cfg = synth.kitti_params(), synth.kitti_first_config()
if "MAXIT" in os.environ:
    cfg.max_iterations = int(os.environ["MAXIT"])
a = r.register_clouds(X, Z, Isometry(), p, cfg)
g = api.register_clouds(X, Z, Isometry(), p, cfg)
print("iterations ref", a.iterations, "gpu", g.iterations, "conv", a.converged, g.converged)
m = min(a.iterations, g.iterations)
ls = np.nonzero(a.lengthscale_trace[:m] != g.lengthscale_trace[:m])[0]
st = np.nonzero(a.step_trace[:m] != g.step_trace[:m])[0]
rb = np.nonzero(a.rebuild_trace[:m] != g.rebuild_trace[:m])[0]
rel = np.abs(g.objective_trace[:m] - a.objective_trace[:m]) / np.abs(a.objective_trace[:m])
print("first diff: lengthscale", ls[:3], "step", st[:3], "rebuild", rb[:3])
print("max rel F diff before first step diff:", rel[: (st[0] if len(st) else m)].max())
k = st[0] if len(st) else None
if k is not None:
    lo = max(0, k - 3)
    for i in range(lo, min(m, k + 4)):
        print(i, a.lengthscale_trace[i], g.lengthscale_trace[i], a.step_trace[i], g.step_trace[i],
              a.objective_trace[i], g.objective_trace[i], a.pair_count_trace[i], g.pair_count_trace[i],
              a.rebuild_trace[i], g.rebuild_trace[i])
err = compose(inverse(g.transform), a.transform)
print("pose diff rad", rotation_angle(err), "m", translation_norm(err))
print("pairs first", a.pair_count_trace[0], g.pair_count_trace[0])
