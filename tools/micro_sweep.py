"""Microbenchmark: the fused sweep kernel alone (CUDA events on the engine
stream) for KITTI-shaped pair lists at several lengthscales and candidate
counts. Prints pair-evals/s and the slot padding of the sliced-ELL layout."""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_2012_03683_b200 import api, synth  # noqa: E402

X, Z, Ts = synth.kitti_pair(7, int(sys.argv[1]) if len(sys.argv) > 1 else 40000)
pk = synth.kitti_params()
ctx = api.default_context()
# bring the clocks up before measuring (idle B200s sit at ~120 MHz)
import time  # noqa: E402
_pw = api.build_pairs(X, Z, Ts, pk.with_lengthscale(0.1), 3.0, 1e-4)
_t0 = time.time()
while time.time() - _t0 < 1.5:
    api.eval_transforms(_pw, X, Z, [Ts] * 8, pk.with_lengthscale(0.1))
for l in (0.1, 0.07, 0.0475):
    pl = pk.with_lengthscale(l)
    pr = api.build_pairs(X, Z, Ts, pl, 3.0, 1e-4)
    info = pr.info()
    for M in (1, 2, 4, 8):
        Tl = [Ts] * M
        for _ in range(3):
            api.eval_transforms(pr, X, Z, Tl, pl)
        ctx.set_profiling(True)
        ctx.reset_stats()
        N = 30
        for _ in range(N):
            api.eval_transforms(pr, X, Z, Tl, pl)
        s = ctx.sweep_stats()
        ctx.set_profiling(False)
        us = s["sweep_ms"] / N * 1e3
        pe = info["pairs"] * M
        print(f"l={l:<6} P={info['pairs']:>8} slots={info['slots']:>8} (pad {info['slots'] / max(1, info['pairs']):.2f}x) "
              f"M={M} sweep {us:7.2f} us  {pe / us / 1e3:8.1f} G pair-evals/s  {info['slots'] * M / us / 1e3:8.1f} G slot-evals/s",
              flush=True)
