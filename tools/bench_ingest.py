"""Frame ingest measurement: KITTI-sized frames (1241 x
376, 19 classes) -> FAST-selected semantic clouds, frames/s end to end through
the public API (host images in, host cloud out) on the B200, vs the compiled
reference (oracle/_ref, single-threaded: its selector is serial) on the host.
One JSON line.

    python tools/bench_ingest.py [--frames 50]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2012_03683_b200 import api, synth  # noqa: E402
from paper_2012_03683_b200.types import SelectorConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=50)
    ap.add_argument("--cpu-frames", type=int, default=3)
    args = ap.parse_args()
    frames = [synth.kitti_frame(s) for s in range(4)]
    sel = SelectorConfig()
    ctx = api.default_context()
    for f in frames:  # warm-up
        api.depth_rgb_to_cloud(*f[:3], f[3], sel, ctx=ctx)
    ctx.synchronize()
    t0 = time.perf_counter()
    sizes = []
    for k in range(args.frames):
        d, rgb, sem, intr = frames[k % len(frames)]
        sizes.append(api.depth_rgb_to_cloud(d, rgb, sem, intr, sel, ctx=ctx).size())
    gpu_s = (time.perf_counter() - t0) / args.frames
    line = {"metric": "frames/s (KITTI-size depth+RGB+19-class frame -> FAST-selected cloud)",
            "config": {"workload": "1241x376 frame, 19 classes, default SelectorConfig", "frames": args.frames,
                       "mean_points": float(np.mean(sizes))},
            "gpu": {"frames_per_s": 1.0 / gpu_s, "ms_per_frame": gpu_s * 1e3,
                    "note": "end to end: host images -> device -> host cloud rows, one ABI call per frame"}}
    from _checkers import Reference, ref_available
    if ref_available():
        r = Reference()
        t0 = time.perf_counter()
        for k in range(args.cpu_frames):
            d, rgb, sem, intr = frames[k % len(frames)]
            r.depth_rgb_to_cloud(d, rgb, sem, intr, sel)
        cpu_s = (time.perf_counter() - t0) / args.cpu_frames
        line["cpu_baseline"] = {"frames_per_s": 1.0 / cpu_s, "ms_per_frame": cpu_s * 1e3, "cores": 1,
                                "kind": "reference", "sample": f"{args.cpu_frames} frames"}
        line["speedup"] = cpu_s / gpu_s
    print(json.dumps(line))


if __name__ == "__main__":
    main()
