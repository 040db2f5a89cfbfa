"""C4 measurement: one KITTI-shaped 1M-point pair (colour +
19-class semantics), subsequent schedule, on one B200.

Reports the full registration (time, iterations, levels, pairs at the first
level, per-level iteration time) and, for the CPU comparison, both sides on a
fixed budget of iterations at the first level (the full CPU registration at
1M points takes hours). One JSON line.

    python bench_c4.py [--points 1000000] [--cpu-iterations 6] [--no-cpu]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2012_03683_b200 import api, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, default=1_000_000)
    ap.add_argument("--cpu-iterations", type=int, default=6)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    t0 = time.perf_counter()
    X, Z, Ts = synth.kitti_pair(2012036830 & 0xFFFF, args.points)
    gen_s = time.perf_counter() - t0
    init = synth.perturbed(Ts, 5)
    p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
    ctx = api.default_context()
    dX, dZ = api.DeviceCloud(X, ctx), api.DeviceCloud(Z, ctx)

    # fixed budget at the first level (GPU; warms the workspaces up)
    budget = synth.kitti_subsequent_config()
    budget.max_iterations = args.cpu_iterations
    api.register_clouds(dX, dZ, init, p, budget, ctx=ctx)
    ctx.synchronize()
    t0 = time.perf_counter()
    rb = api.register_clouds(dX, dZ, init, p, budget, ctx=ctx)
    ctx.synchronize()
    gpu_budget_s = time.perf_counter() - t0

    # full registration
    ctx.reset_stats()
    ctx.set_profiling(True)
    t0 = time.perf_counter()
    res = api.register_clouds(dX, dZ, init, p, cfg, ctx=ctx)
    ctx.synchronize()
    full_s = time.perf_counter() - t0
    ctx.set_profiling(False)
    sw = ctx.sweep_stats()
    bs = ctx.build_stats()
    ls = np.asarray(res.lengthscale_trace)
    levels = sorted(set(ls.tolist()), reverse=True)
    err = synth.pose_error(res.transform, Ts) if hasattr(synth, "pose_error") else None

    line = {
        "config": {"workload": "C4 KITTI-shaped 1M-point semantic pair, subsequent schedule l 0.1 -> 0.0475",
                   "points": args.points, "generation_s": round(gen_s, 1)},
        "gpu_full_registration": {"seconds": full_s, "iterations": res.iterations, "converged": bool(res.converged),
                                  "levels": len(levels), "pairs_first_iteration": int(res.pair_count_trace[0]),
                                  "pairs_last_iteration": int(res.pair_count_trace[-1]),
                                  "ms_per_iteration": full_s / max(1, res.iterations) * 1e3,
                                  "sweep_ms": sw["sweep_ms"], "sweep_rounds": sw["sweep_rounds"],
                                  "pair_evals_per_s": sw["pair_evals"] / (sw["sweep_ms"] * 1e-3) if sw["sweep_ms"] else None,
                                  "grid_builds": bs["grid_builds"], "filter_builds": bs["filter_builds"]},
        "budget": {"iterations": rb.iterations, "gpu_s": gpu_budget_s},
    }
    if err is not None:
        line["gpu_full_registration"]["pose_error"] = err
    if not args.no_cpu:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from _checkers import Reference, ref_available
        if ref_available():
            r = Reference()
            cores = os.cpu_count() or 1
            r.set_threads(cores)
            t0 = time.perf_counter()
            rc = r.register_clouds(X, Z, init, p, budget)
            cpu_s = time.perf_counter() - t0
            line["budget"].update({"cpu_s": cpu_s, "cpu_cores": cores, "cpu_kind": "reference",
                                   "cpu_iterations": rc.iterations, "speedup": cpu_s / gpu_budget_s,
                                   "same_trace": bool(np.allclose(rc.objective_trace, rb.objective_trace, rtol=1e-6))})
    print(json.dumps(line))


if __name__ == "__main__":
    main()
