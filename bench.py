"""Benchmark: CVO registration throughput on KITTI-shaped semantic frame pairs.

Workload (BASELINE.json configs[2], the metric's configuration): synthetic
KITTI-stereo-shaped street frames, 40 000 points each, colour (3, SE 0.15) +
19-class softmax semantics (linear), subsequent-frame schedule l = 0.1 ->
0.0475 (kitti-stereo.json), initial guess = true motion composed with a small
error (constant-velocity prior). A step = one batch of B independent frame
pairs registered to convergence on one GPU (lockstep batched host loop).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]
                    [--mode throughput|latency] [--workload c3|first|c5] [--frames F] [--chains C]

Prints ONE JSON line (rank 0). Multi-GPU: one process per GPU (torchrun),
each rank registers its own B pairs (weak scaling, no data-path collective),
time = max over ranks.

Other measurements (not the driver's line; run by hand, results under profiles/):
  --mode latency      one end-to-end kreg_register_clouds_host call per pair,
                      pairs one after another (the CLI's `kreg register` path)
  --workload first    the first-frame schedule (l 0.95 -> 0.0475) on B pairs
  --workload c5       a KITTI-shaped sequence of F frames registered as C
                      independent chains (kreg_register_sequence_chains)
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
C3_WORKLOAD = "C3 KITTI-shaped 40k-point semantic pairs (colour + 19-class), subsequent schedule l 0.1 -> 0.0475"
SEED = 2012036830
UNIT = "registrations/s"
HBM_PEAK_FALLBACK = 6551.7


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def make_workload(rank: int, batch: int, n_points: int, seed: int = SEED):
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


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_env():
    """OpenMP placement of the reference runs: one
    thread per core, packed. Must be set before the runtime starts."""
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")
    return {"cpu": cpu_model(), "omp_proc_bind": os.environ["OMP_PROC_BIND"], "omp_places": os.environ["OMP_PLACES"]}


def cpu_reference_sample(Xs, Zs, inits, params, cfg, seconds_budget: float = 30.0):
    """The compiled reference (oracle/_ref) on the box's host cores: latency
    mode (register_clouds with OpenMP over all threads, as the CLI runs it),
    pairs registered one after another until ~seconds_budget elapsed."""
    env = reference_env()
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
                      f"{dt:.1f} s", **env}


# Per pair evaluation k_sweep issues 17 FP32 flops (3 sub, |d|^2 as 1 mul +
# 2 FMA, the exponent FMA, W +=, 3 FMA into S) and one MUFU ex2. Nominal issue
# rates on sm_100: 128 FP32 lanes (2 flops per FMA) and 16 MUFU lanes per SM
# per clock.
SWEEP_FLOPS_PER_PAIR = 17
SM_COUNT = 148


def issue_fractions(sweep, clk):
    """FP32 and MUFU throughput of the sweep as fractions of nominal at the
    measured SM clock: how close the pair loop is to its issue bound."""
    if not sweep.get("sweep_ms"):
        return {}
    mhz = (clk or {}).get("sm_mhz") or 1965.0
    pe = sweep["pair_evals"] / (sweep["sweep_ms"] * 1e-3)
    fp32_peak = SM_COUNT * 128 * 2 * mhz * 1e6
    mufu_peak = SM_COUNT * 16 * mhz * 1e6
    return {"fp32_tflops": pe * SWEEP_FLOPS_PER_PAIR / 1e12,
            "fp32_frac_of_nominal": pe * SWEEP_FLOPS_PER_PAIR / fp32_peak,
            "mufu_frac_of_nominal": pe / mufu_peak,
            "nominal_at_mhz": mhz}


def run_other(args, world, rank, local):
    """The hand-run measurements (module docstring). Prints one JSON line."""
    from paper_2012_03683_b200 import api
    ctx = api.Context(local)
    if args.chunk_units > 0:
        ctx.set_chunk_units(args.chunk_units)
    params = synth.kitti_params()
    clocks = ClockSampler(local)
    if args.workload == "c5":
        cfg = synth.kitti_subsequent_config()
        t0 = time.perf_counter()
        frames, _ = synth.kitti_sequence(1000 + rank, args.frames, args.points)
        gen_s = time.perf_counter() - t0
        for _ in range(args.warmup):
            api.register_sequence(frames, params, cfg, ctx=ctx, chains=args.chains)
        ctx.synchronize()
        clocks.start()
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.steps):  # frames resident on the device (uploaded by the warm-up)
            seq = api.register_sequence(frames, params, cfg, ctx=ctx, chains=args.chains)
        ctx.synchronize()
        dt = max_over_ranks(time.perf_counter() - t0, world)
        clk = clocks.stop()
        # end to end: host frames in, every frame uploaded inside the timed call
        ctx.reset_stats()
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            seq = api.register_sequence_host(frames, params, cfg, ctx=ctx, chains=args.chains)
        ctx.synchronize()
        dt_e2e = max_over_ranks(time.perf_counter() - t0, world)
        io = ctx.io_stats()
        n = sum_over_ranks((args.frames - 1) * args.steps, world)
        line = {"metric": METRIC, "value": n / dt, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
                "scaling": "weak", "dtype": "f32+f64", "data": "synthetic", "mode": "sequence",
                "config": {"workload": f"C5 KITTI-shaped sequence, {args.frames} frames of {args.points} points, "
                                       f"{args.chains} chains (kreg_register_sequence_chains)",
                           "frame_generation_s": gen_s, "mean_iterations": float(np.mean(seq.iterations)),
                           "fallbacks": int(np.sum(seq.fallback))},
                "e2e": {"value": n / dt_e2e, "unit": UNIT, "h2d_bytes_per_step": io["h2d_bytes"] // args.steps,
                        "d2h_bytes_per_step": io["d2h_bytes"] // args.steps},
                "gpu_launches": ctx.kernel_launches(), "clocks": clk, "admission": ctx.admission_stats()}
    else:
        cfg = synth.kitti_first_config() if args.workload == "first" else synth.kitti_subsequent_config()
        B = args.batch
        Xs, Zs, inits = make_workload(rank, B, args.points)
        if args.mode == "latency":
            # one pair per call, host clouds in, results out: `kreg register`
            n_pairs = max(1, args.steps)
            for k in range(args.warmup):
                api.register_clouds_host(Xs[k % B], Zs[k % B], inits[k % B], params, cfg, ctx=ctx)
            ctx.synchronize()
            ctx.reset_stats()
            clocks.start()
            barrier(world)
            lat, its = [], []
            for k in range(n_pairs):
                t0 = time.perf_counter()
                r = api.register_clouds_host(Xs[k % B], Zs[k % B], inits[k % B], params, cfg, ctx=ctx)
                lat.append(time.perf_counter() - t0)
                its.append(r.iterations)
            clk = clocks.stop()
            dt = max_over_ranks(sum(lat), world)
            io = ctx.io_stats()
            n = sum_over_ranks(n_pairs, world)
            line = {"metric": METRIC, "value": n / dt, "unit": UNIT, "n_gpus": world, "steps": n_pairs,
                    "warmup": args.warmup, "ms_per_step": dt / n_pairs * 1e3, "higher_is_better": True,
                    "scaling": "weak", "dtype": "f32+f64", "data": "synthetic", "mode": "latency",
                    "config": {"workload": f"{args.workload.upper()} KITTI-shaped {args.points}-point pairs, one "
                                           "kreg_register_clouds_host call per pair",
                               "mean_iterations": float(np.mean(its)),
                               "latency_ms": {"p50": float(np.percentile(lat, 50) * 1e3),
                                              "p90": float(np.percentile(lat, 90) * 1e3),
                                              "max": float(np.max(lat) * 1e3)}},
                    "e2e": {"value": n / dt, "unit": UNIT, "h2d_bytes_per_step": io["h2d_bytes"] // n_pairs,
                            "d2h_bytes_per_step": io["d2h_bytes"] // n_pairs},
                    "gpu_launches": ctx.kernel_launches(), "clocks": clk}
        else:  # throughput, first-frame schedule
            dev_X = [api.DeviceCloud(x, ctx) for x in Xs]
            dev_Z = [api.DeviceCloud(z, ctx) for z in Zs]
            for _ in range(args.warmup):
                api.register_batch(dev_X, dev_Z, inits, params, cfg, ctx=ctx)
            ctx.synchronize()
            ctx.reset_stats()
            ctx.set_profiling(True)
            clocks.start()
            barrier(world)
            t0 = time.perf_counter()
            its = []
            for _ in range(args.steps):
                res, st = api.register_batch(dev_X, dev_Z, inits, params, cfg, ctx=ctx)
                assert (np.asarray(st) == 0).all(), f"failed registrations in a timed step: {list(st)}"
                its += [r.iterations for r in res]
            ctx.synchronize()
            dt = max_over_ranks(time.perf_counter() - t0, world)
            clk = clocks.stop()
            ctx.set_profiling(False)
            sweep, build = ctx.sweep_stats(), ctx.build_stats()
            n = sum_over_ranks(B * args.steps, world)
            line = {"metric": METRIC, "value": n / dt, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                    "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
                    "scaling": "weak", "dtype": "f32+f64", "data": "synthetic", "mode": "throughput",
                    "config": {"workload": f"first-frame schedule (l 0.95 -> 0.0475) on {B} KITTI-shaped "
                                           f"{args.points}-point pairs", "mean_iterations": float(np.mean(its))},
                    "gpu_launches": ctx.kernel_launches(), "clocks": clk,
                    "sweep": {**sweep, **issue_fractions(sweep, clk)}, "build": build,
                    "admission": ctx.admission_stats()}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_reference_arm(args, world, rank):
    """--impl reference: the reference CPU implementation on this box's cores,
    in both of its modes: latency (register_clouds with
    OpenMP inside, one pair after another, as `kreg register` runs it: the
    timed steps) and throughput (OpenMP over independent pairs, one thread each,
    as synth_bench does, eval.cpp:323: one batch of `cores` pairs, reported
    beside it). `value` is the better of the two."""
    if rank != 0:
        return
    env = reference_env()
    params, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _checkers import Reference, ref_available
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libkreg_ref.so not built"}))
        return
    r = Reference()
    cores = os.cpu_count() or 1
    n_lat = max(1, args.warmup + args.steps)
    Xs, Zs, inits = make_workload(0, n_lat + cores, args.points)
    r.set_threads(cores)
    for k in range(args.warmup):
        r.register_clouds(Xs[k], Zs[k], inits[k], params, cfg)
    t0 = time.perf_counter()
    iters = []
    for k in range(args.warmup, args.warmup + args.steps):
        iters.append(r.register_clouds(Xs[k], Zs[k], inits[k], params, cfg).iterations)
    dt = time.perf_counter() - t0
    v_lat = args.steps / dt
    # throughput mode: one thread per pair, `cores` pairs at once
    res, st, secs = r.register_batch(Xs[n_lat:n_lat + cores], Zs[n_lat:n_lat + cores], inits[n_lat:n_lat + cores],
                                     params, cfg)
    v_thr = cores / secs if secs > 0 else 0.0
    it_thr = [x.iterations for x in res if x is not None]
    v = max(v_lat, v_thr)
    mode = "latency" if v_lat >= v_thr else "throughput"
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": C3_WORKLOAD, "points": args.points, "seed": SEED},
        "execution": {"step": "one frame pair registered to convergence (latency mode)",
                      "pairs": "make_workload(rank 0): the first steps + warmup pairs of the GPU arm's batch"},
        "mean_iterations": float(np.mean(iters)),
        "cpu_modes": {"latency": {"value": v_lat, "pairs": args.steps, "threads_per_pair": cores,
                                  "mean_iterations": float(np.mean(iters))},
                      "throughput": {"value": v_thr, "pairs": cores, "threads_per_pair": 1, "seconds": secs,
                                     "mean_iterations": float(np.mean(it_thr)) if it_thr else None},
                      "reported": mode},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"better of latency ({args.steps} pairs, OpenMP over {cores} threads) and "
                                   f"throughput ({cores} pairs, one thread each)", **env},
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
    ap.add_argument("--mode", default="throughput", choices=["throughput", "latency"])
    ap.add_argument("--chunk-units", type=int, default=0,
                    help="sweep chunk size of new pair lists (0 = engine default, 48; ~12 suits one registration at a time)")
    ap.add_argument("--workload", default="c3", choices=["c3", "first", "c5"])
    ap.add_argument("--frames", type=int, default=257, help="c5: frames in the sequence")
    ap.add_argument("--chains", type=int, default=16, help="c5: independent chains")
    args = ap.parse_args()

    if args.impl == "reference":  # CPU only: no process group, ranks > 0 exit at once
        run_reference_arm(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")))
        return
    world, rank, local = dist_setup()

    from paper_2012_03683_b200 import api
    if args.mode != "throughput" or args.workload != "c3":
        return run_other(args, world, rank, local)
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

    # ---- device-resident timed region: K steps (the engine's default: the
    # batch's rounds alternate between two groups on two streams)
    ctx.reset_stats()
    clocks = ClockSampler(local)
    clocks.start()
    barrier(world)
    ctx.synchronize()
    # device time of the K steps: CUDA events on the engine's stream (every
    # step's host loop runs between them, it is part of the step)
    ctx.timer_mark(0)
    t0 = time.perf_counter()
    iters = []
    for _ in range(args.steps):
        res, st = api.register_batch(dev_X, dev_Z, inits, params, cfg, ctx=ctx)
        assert (np.asarray(st) == 0).all(), f"failed registrations in a timed step: {list(st)}"
        iters += [r.iterations for r in res if r is not None]
    ctx.timer_mark(1)
    ctx.synchronize()
    wall = time.perf_counter() - t0
    dt = ctx.timer_ms() * 1e-3
    clk = clocks.stop()
    host = ctx.host_stats()
    launches = ctx.kernel_launches()
    dt_max = max_over_ranks(dt, world)
    total = sum_over_ranks(B * args.steps, world)
    value = total / dt_max

    # ---- kernel roofline: one more step with the rounds on ONE stream and
    # per-launch CUDA events (with two streams a launch's events would also
    # span the other stream's concurrent kernels); not part of `value`
    prev_groups = os.environ.get("KREG_GROUPS")
    os.environ["KREG_GROUPS"] = "1"
    try:
        ctx.reset_stats()
        ctx.set_profiling(True)
        ctx.timer_mark(0)
        api.register_batch(dev_X, dev_Z, inits, params, cfg, ctx=ctx)
        ctx.timer_mark(1)
        ctx.synchronize()
        dt_prof = ctx.timer_ms() * 1e-3
        ctx.set_profiling(False)
        sweep = ctx.sweep_stats()
    finally:
        if prev_groups is None:
            del os.environ["KREG_GROUPS"]
        else:
            os.environ["KREG_GROUPS"] = prev_groups

    # ---- end to end through the public API with host buffers (one untimed
    # call first: it sizes the pinned staging and the device cloud arena)
    api.register_batch_host(Xs, Zs, inits, params, cfg, ctx=ctx)
    ctx.synchronize()
    ctx.reset_stats()
    barrier(world)
    ctx.timer_mark(0)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res_h, st_h = api.register_batch_host(Xs, Zs, inits, params, cfg, ctx=ctx)
        assert (np.asarray(st_h) == 0).all(), f"failed registrations in a timed step: {list(st_h)}"
    ctx.timer_mark(1)
    ctx.synchronize()
    wall_e2e = time.perf_counter() - t0
    dt_e2e = max_over_ranks(ctx.timer_ms() * 1e-3, world)
    host_e2e = ctx.host_stats()
    e2e_value = sum_over_ranks(B * args.steps, world) / dt_e2e
    io = ctx.io_stats()  # bytes the engine copied host->device / read back, counted in the library
    h2d = io["h2d_bytes"] // args.steps
    d2h = io["d2h_bytes"] // args.steps

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
                "sweep_share_of_step": sweep["sweep_ms"] * 1e-3 / dt_prof,
                "measured_in": "one extra step after the timed region with the rounds on one stream (per-launch "
                               "CUDA events around the sweep launches on that stream)",
                **issue_fractions(sweep, clk),
                "peak_source": "MEASURED_PEAKS.json" if "hbm_gbs" in peaks else "fallback"}

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_reference_sample(Xs, Zs, inits, params, cfg, args.cpu_seconds)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
            # config: identical in both arms (same generator, same pairs);
            # how each arm runs them is in "execution"
            "config": {"workload": C3_WORKLOAD, "points": args.points, "seed": SEED},
            "execution": {"pairs_per_step_per_gpu": B,
                          "parallelism": f"independent pairs x {world} GPU(s), lockstep batch per GPU",
                          "l2": "inputs larger than L2 (B pair lists > 126 MB)"},
            "mean_iterations": float(np.mean(iters)) if iters else None,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "rounds_per_step": host["rounds"] / max(1, args.steps),
            "roofline": roofline,
            "clocks": clk,
            "timing": {"method": "CUDA events on the engine stream around the K steps (max over ranks)",
                       "device_s": dt_max, "wall_s": wall, "e2e_device_s": dt_e2e, "e2e_wall_s": wall_e2e},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
