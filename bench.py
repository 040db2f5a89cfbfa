"""Benchmark: CVO registration throughput on KITTI-shaped semantic frame pairs.

Workload (BASELINE.json configs[2], the metric's configuration): synthetic
KITTI-stereo-shaped street frames, 40 000 points each, colour (3, SE 0.15) +
19-class softmax semantics (linear), subsequent-frame schedule l = 0.1 ->
0.0475 (kitti-stereo.json), initial guess = true motion composed with a small
error (constant-velocity prior). A step = one batch of B independent frame
pairs registered to convergence on one GPU (lockstep batched host loop).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

Prints ONE JSON line (rank 0). Multi-GPU: one process per GPU (torchrun),
each rank registers its own B pairs (weak scaling, no data-path collective),
time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2012_03683_b200 import synth  # noqa: E402

METRIC = "registrations/sec (KITTI-shape 19-class pairs)"
UNIT = "registrations/s"
HBM_PEAK_FALLBACK = 6551.7


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def make_workload(rank: int, batch: int, n_points: int, seed: int = 2012036830):
    """B independent KITTI-shaped frame pairs per rank: each
    pair is its own ray-cast street, second frame 1.0 m forward + 0.5 deg yaw,
    initial guess = true motion composed with a small error."""
    Xs, Zs, inits = [], [], []
    for k in range(batch):
        s = synth.SplitMix64.derive(seed, 100003 * rank + k) & 0x7FFFFFFF
        X, Z, T = synth.kitti_pair(s, n_points, start=float(k % 7) * 9.0)
        Xs.append(X)
        Zs.append(Z)
        inits.append(synth.perturbed(T, s))
    return Xs, Zs, inits


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._thr = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([s.strip() for s in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._thr = threading.Thread(target=run, daemon=True)
        self._thr.start()

    def stop(self):
        self._stop.set()
        if self._thr:
            self._thr.join(timeout=6)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if len(s) > 3 + k and s[3 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def cloud_bytes(c) -> int:
    return c.positions.nbytes + c.features.nbytes


def cpu_reference_sample(Xs, Zs, inits, params, cfg, seconds_budget: float = 30.0):
    """The compiled reference (oracle/_ref) on the box's host cores: latency
    mode (register_clouds with OpenMP over all threads, as the CLI runs it),
    pairs registered one after another until ~seconds_budget elapsed."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _checkers import Reference, ref_available, Oracle
    cores = os.cpu_count() or 1
    if ref_available():
        r = Reference()
        r.set_threads(cores)
        kind = "reference"
        run = lambda k: r.register_clouds(Xs[k], Zs[k], inits[k], params, cfg)  # noqa: E731
    else:  # the plain-C port, single-threaded
        o = Oracle()
        kind, cores = "port", 1
        run = lambda k: o.register_clouds(Xs[k], Zs[k], inits[k], params, cfg)  # noqa: E731
    t0 = time.perf_counter()
    n = 0
    while n < len(Xs):
        run(n)
        n += 1
        if time.perf_counter() - t0 > seconds_budget:
            break
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{n} KITTI-shaped 40k-point pair(s), register_clouds with OpenMP over {cores} threads, "
                      f"{dt:.1f} s"}


def run_reference_arm(args, world, rank):
    """--impl reference: the reference CPU implementation on this box's cores."""
    if rank != 0:
        return
    params, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
    Xs, Zs, inits = make_workload(0, max(1, args.warmup + args.steps), args.points)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _checkers import Reference, ref_available
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libkreg_ref.so not built"}))
        return
    r = Reference()
    cores = os.cpu_count() or 1
    r.set_threads(cores)
    for k in range(args.warmup):
        r.register_clouds(Xs[k], Zs[k], inits[k], params, cfg)
    t0 = time.perf_counter()
    for k in range(args.warmup, args.warmup + args.steps):
        r.register_clouds(Xs[k], Zs[k], inits[k], params, cfg)
    dt = time.perf_counter() - t0
    v = args.steps / dt
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": "C3 KITTI-shaped 40k-point semantic pairs, subsequent schedule", "points": args.points,
                   "step": "one frame pair registered to convergence (latency mode)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} pairs, register_clouds with OpenMP over {cores} threads"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=128, help="frame pairs per step per GPU")
    ap.add_argument("--window", type=int, default=0, help="registrations in flight (0 = whole batch)")
    ap.add_argument("--points", type=int, default=40000)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=25.0)
    args = ap.parse_args()

    if args.impl == "reference":  # CPU only: no process group, ranks > 0 exit at once
        run_reference_arm(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")))
        return
    world, rank, local = dist_setup()

    from paper_2012_03683_b200 import api
    ctx = api.Context(local)
    ctx.set_max_active(args.window)
    params, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
    B = args.batch
    Xs, Zs, inits = make_workload(rank, B, args.points)
    dev_X = [api.DeviceCloud(x, ctx) for x in Xs]
    dev_Z = [api.DeviceCloud(z, ctx) for z in Zs]

    # warm-up (also grows the device workspaces to their steady-state size)
    for _ in range(args.warmup):
        api.register_batch(dev_X, dev_Z, inits, params, cfg, ctx=ctx)
    ctx.synchronize()

    # ---- device-resident timed region: K steps
    ctx.reset_stats()
    ctx.set_profiling(True)
    clocks = ClockSampler(local)
    clocks.start()
    barrier(world)
    ctx.synchronize()
    t0 = time.perf_counter()
    iters = []
    for _ in range(args.steps):
        res, st = api.register_batch(dev_X, dev_Z, inits, params, cfg, ctx=ctx)
        assert (np.asarray(st) == 0).all(), f"failed registrations in a timed step: {list(st)}"
        iters += [r.iterations for r in res if r is not None]
    ctx.synchronize()
    dt = time.perf_counter() - t0
    clk = clocks.stop()
    ctx.set_profiling(False)
    sweep = ctx.sweep_stats()
    host = ctx.host_stats()
    launches = ctx.kernel_launches()
    dt_max = max_over_ranks(dt, world)
    total = sum_over_ranks(B * args.steps, world)
    value = total / dt_max

    # ---- end to end through the public API with host buffers (one untimed
    # call first: it sizes the pinned staging and the device cloud arena)
    api.register_batch_host(Xs, Zs, inits, params, cfg, ctx=ctx)
    ctx.synchronize()
    ctx.reset_stats()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res_h, st_h = api.register_batch_host(Xs, Zs, inits, params, cfg, ctx=ctx)
        assert (np.asarray(st_h) == 0).all(), f"failed registrations in a timed step: {list(st_h)}"
    ctx.synchronize()
    dt_e2e = max_over_ranks(time.perf_counter() - t0, world)
    host_e2e = ctx.host_stats()
    e2e_value = sum_over_ranks(B * args.steps, world) / dt_e2e
    h2d = sum(cloud_bytes(c) for c in Xs + Zs)
    d2h = int(host_e2e["rounds"] / max(1, args.steps)) * 8 * 8 * 4  # per-round result block (<= 4 requests avg)

    # ---- roofline of the fused sweep kernel (dominant kernel)
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", HBM_PEAK_FALLBACK))
    pairs_bytes = sweep["pairs_streamed"] * 8.0
    achieved = pairs_bytes / (sweep["sweep_ms"] * 1e-3) / 1e9 if sweep["sweep_ms"] > 0 else 0.0
    # DRAM traffic per sweep launch from the committed ncu --set full capture
    # (profiles/r01_sweep_traffic.json), scaled to this run's algorithmic bytes
    # per launch by the measured traffic / algorithmic ratio
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r01_sweep_traffic.json")) as f:
            tr = json.load(f)
        if sweep["sweep_rounds"]:
            traffic = tr["traffic_over_algorithmic"] * pairs_bytes / sweep["sweep_rounds"]
    except Exception:
        tr = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic,
                "traffic_source": ("profiles/r01_sweep_traffic.json: dram__bytes_read+write per k_sweep launch = "
                                   f"{tr['traffic_over_algorithmic']:.2f} x algorithmic bytes" if tr else None),
                "algorithmic_bytes_per_launch": pairs_bytes / sweep["sweep_rounds"] if sweep["sweep_rounds"] else None,
                "kernel": "k_sweep (fused F + SE(3) gradient + displacement)",
                "algorithmic_bytes_per_pair": 8,
                "pair_evals_per_s": sweep["pair_evals"] / (sweep["sweep_ms"] * 1e-3) if sweep["sweep_ms"] else 0.0,
                "sweep_share_of_step": sweep["sweep_ms"] * 1e-3 / dt,
                "peak_source": "MEASURED_PEAKS.json" if "hbm_gbs" in peaks else "fallback"}

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_reference_sample(Xs, Zs, inits, params, cfg, args.cpu_seconds)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
            "config": {"workload": "C3 KITTI-shaped 40k-point semantic pairs (colour + 19-class), subsequent "
                                   "schedule l 0.1 -> 0.0475", "points": args.points, "pairs_per_step_per_gpu": B,
                       "parallelism": f"independent pairs x {world} GPU(s), lockstep batch per GPU",
                       "l2": "inputs larger than L2 (B pair lists > 126 MB)",
                       "mean_iterations": float(np.mean(iters)) if iters else None},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "rounds_per_step": host["rounds"] / max(1, args.steps),
            "roofline": roofline,
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
