"""Diagnostic (KREG_TIMELINE variant build): per-item and per-CTA timeline of
one sweep launch (device globaltimer records, no printf).

    python -c "from paper_2012_03683_b200.build import build_variant as b; b('tl', ['KREG_TIMELINE'])"
    KREG_LIB=paper_2012_03683_b200/_variants/tl.so python tools/timeline.py [lengthscale] [M] [B]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
from paper_2012_03683_b200 import api, synth  # noqa: E402

l = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0475
M = int(sys.argv[2]) if len(sys.argv) > 2 else 2
X, Z, Ts = synth.kitti_pair(7, 40000)
p = synth.kitti_params().with_lengthscale(l)
pr = api.build_pairs(X, Z, Ts, p, 3.0, 1e-4)
lib = api.lib()
lib.kreg_debug_timeline.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = np.zeros((1 << 16, 4), dtype=np.uint64)
get = lambda: lib.kreg_debug_timeline(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), 1 << 16)  # noqa: E731
for _ in range(3):
    api.eval_transforms(pr, X, Z, [Ts] * M, p)
ctx = api.default_context()
get()
ctx.set_profiling(True)
ctx.reset_stats()
api.eval_transforms(pr, X, Z, [Ts] * M, p)
n = get()
rec = buf[:n].astype(np.int64)
print("pairs", pr.size(), "M", M, "sweep_us (events)", round(ctx.sweep_stats()["sweep_ms"] * 1e3, 1))
cta = rec[(rec[:, 2] & 0xFFFF) == 0xFFFF]
its = rec[(rec[:, 2] & 0xFFFF) != 0xFFFF]
t0 = cta[:, 0].min()
print(f"CTAs {len(cta)}: start max {(cta[:, 0].max() - t0) / 1e3:.1f} us, end p50 {np.median(cta[:, 1] - t0) / 1e3:.1f} "
      f"max {(cta[:, 1].max() - t0) / 1e3:.1f} us")
for typ, name in ((0, "displacement"), (1, "chunk")):
    sel = its[(its[:, 3] & 1) == typ]
    if len(sel):
        d = (sel[:, 1] - sel[:, 0]) / 1e3
        s = (sel[:, 0] - t0) / 1e3
        e = (sel[:, 1] - t0) / 1e3
        print(f"{name:12s} n={len(sel):5d} dur p50 {np.median(d):.1f} p90 {np.percentile(d, 90):.1f} max {d.max():.1f} us; "
              f"start p50 {np.median(s):.1f} max {s.max():.1f}; end max {e.max():.1f} us")
order = np.argsort(-(its[:, 1] - its[:, 0]))[:6]
for k in order:
    print(f"  slow: item {its[k, 3] >> 1} type {its[k, 3] & 1} start {(its[k, 0] - t0) / 1e3:.1f} "
          f"dur {(its[k, 1] - its[k, 0]) / 1e3:.1f} us")
last = np.argsort(-its[:, 1])[:4]
for k in last:
    print(f"  last: item {its[k, 3] >> 1} type {its[k, 3] & 1} start {(its[k, 0] - t0) / 1e3:.1f} "
          f"end {(its[k, 1] - t0) / 1e3:.1f} us")
ch = its[(its[:, 3] & 1) == 1]
d = (ch[:, 1] - ch[:, 0]) / 1e3
med = np.median(d)
print(f"chunk time total {d.sum():.0f} us; excess over median {np.clip(d - med, 0, None).sum():.0f} us "
      f"({np.clip(d - med, 0, None).sum() / d.sum() * 100:.1f} %); chunks > 1.5x median: {(d > 1.5 * med).sum()}")
