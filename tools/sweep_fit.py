"""Per-launch sweep time vs streamed slots over one batched run (fixed cost
per launch = intercept). Diagnostic; reads KREG_TRACE_ROUNDS lines."""
import os
import re
import subprocess
import sys

import numpy as np

env = dict(os.environ, KREG_TRACE_ROUNDS="1")
code = r'''
import os, sys
sys.path.insert(0, os.getcwd())
import bench
from paper_2012_03683_b200 import api, synth
B = int(os.environ.get("B", "128"))
ctx = api.default_context()
Xs, Zs, inits = bench.make_workload(0, B, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
dX = [api.DeviceCloud(x, ctx) for x in Xs]
dZ = [api.DeviceCloud(z, ctx) for z in Zs]
api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)
ctx.set_profiling(True)
sys.stderr.write("=== timed\n")
api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)
'''
r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
lines = r.stderr.split("=== timed\n", 1)[-1].splitlines()
rows = []
for ln in lines:
    m = re.match(r"kreg-sweep ms=([\d.]+) requests=(\d+) grad=(\d+) m=(\d+) slots=(\d+) builds=(\d+)", ln)
    if m:
        rows.append([float(v) for v in m.groups()])
a = np.array(rows)
ms, req, grad, msum, slots, builds = a.T
A = np.stack([np.ones_like(ms), slots * msum / np.maximum(req, 1) / 1e9], 1)
coef, *_ = np.linalg.lstsq(A, ms, rcond=None)
print(f"launches {len(ms)}  total {ms.sum():.1f} ms  mean {ms.mean() * 1e3:.1f} us")
print(f"fit ms = {coef[0] * 1e3:.1f} us + {coef[1]:.3f} ms per 1e9 slot-candidates")
A2 = np.stack([np.ones_like(ms), slots / 1e9, req, grad, builds], 1)
c2, *_ = np.linalg.lstsq(A2, ms, rcond=None)
print(f"fit ms = {c2[0] * 1e3:.1f} us + {c2[1]:.3f} ms/Gslot + {c2[2] * 1e3:.2f} us/request"
      f" + {c2[3] * 1e3:.2f} us/grad request + {c2[4] * 1e3:.2f} us/build")
for lo, hi in ((0, 16), (16, 64), (64, 129), (129, 10000)):
    s = (req >= lo) & (req < hi)
    if s.any():
        print(f"requests [{lo},{hi}): n={s.sum():5d} mean {ms[s].mean() * 1e3:7.1f} us  slots {slots[s].mean() / 1e6:7.1f} M"
              f"  us/Mslot {(ms[s] / slots[s] * 1e9).mean():.2f}")
small = slots < np.percentile(slots, 10)
print(f"smallest 10%: mean {ms[small].mean() * 1e3:.1f} us at {slots[small].mean() / 1e6:.1f} M slots")
