"""Diagnostic (KREG_TIMELINE variant): per-CTA start / last item / end of one single-request sweep."""
import os, re, subprocess, sys
sys.path.insert(0, os.getcwd())
if os.environ.get("TL_CHILD") != "1":
    env = dict(os.environ, TL_CHILD="1", KREG_LIB="paper_2012_03683_b200/_variants/tl.so")
    out = subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, capture_output=True, text=True).stdout
    rows = [tuple(map(int, m.groups())) for m in re.finditer(r"TL cta (\d+) sm \d+ start (\d+) last_item (\d+) end (\d+) items (\d+)", out)]
    # the last launch: rows whose start lies within 5 ms of the latest start
    tmax = max(r[1] for r in rows)
    rows = [r for r in rows if r[1] > tmax - 5_000_000]
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/timeline_rows.txt", "w") as f:
        for r in sorted(rows, key=lambda r: r[1]):
            f.write(" ".join(map(str, r)) + "\n")
    t0 = min(r[1] for r in rows)
    starts = sorted((r[1] - t0) / 1e3 for r in rows)
    ends = sorted((r[3] - t0) / 1e3 for r in rows)
    lasts = sorted((r[2] - t0) / 1e3 for r in rows if r[4] > 0)
    items = sum(r[4] for r in rows)
    print(f"CTAs {len(rows)} items {items}; start us: min 0 p50 {starts[len(starts)//2]:.1f} max {starts[-1]:.1f}; "
          f"last item us: p50 {lasts[len(lasts)//2]:.1f} max {lasts[-1]:.1f}; end us: p50 {ends[len(ends)//2]:.1f} max {ends[-1]:.1f}")
    print(out.strip().splitlines()[-1])
    sys.exit(0)
from paper_2012_03683_b200 import api, synth
X, Z, Ts = synth.kitti_pair(7, 40000)
l = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0475
p = synth.kitti_params().with_lengthscale(l)
pr = api.build_pairs(X, Z, Ts, p, 3.0, 1e-4)
for _ in range(3):
    api.eval_transforms(pr, X, Z, [Ts, Ts], p)
print("pairs", pr.size())
ctx = api.default_context()
ctx.set_profiling(True)
ctx.reset_stats()
api.eval_transforms(pr, X, Z, [Ts, Ts], p)
print("pairs", pr.size(), "sweep_us", round(ctx.sweep_stats()["sweep_ms"] * 1e3, 1))
