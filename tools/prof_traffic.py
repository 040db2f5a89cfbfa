"""Profiling helper: one batch of B KITTI-shaped registrations with a per-round
trace (KREG_TRACE_ROUNDS=1) so ncu-captured k_sweep launches can be matched to
their algorithmic bytes (8 B per streamed pair)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_2012_03683_b200 import api, synth  # noqa: E402

B = int(os.environ.get("B", "64"))
ctx = api.default_context()
Xs, Zs, inits = bench.make_workload(0, B, 40000)
p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
dX = [api.DeviceCloud(x, ctx) for x in Xs]
dZ = [api.DeviceCloud(z, ctx) for z in Zs]
res, st = api.register_batch(dX, dZ, inits, p, cfg, ctx=ctx)
print("done", sum(r.iterations for r in res) / len(res), file=sys.stderr)
