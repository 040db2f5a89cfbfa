"""Build profiles/<round>_sweep_traffic.json from an ncu --set full capture of
k_sweep launches plus the engine's KREG_TRACE_ROUNDS trace of the same run
(exact launch matching through the trace's launch index). Run on the GPU box:

    KREG_TRACE_ROUNDS=1 B=64 ncu --set full --clock-control none -k regex:^k_sweep$ \\
        --launch-skip 300 -c 4 -o gpurun_out/sweep_full python tools/prof_traffic.py \\
        2> gpurun_out/sweep_trace.txt
    python tools/make_traffic.py gpurun_out/sweep_full.ncu-rep gpurun_out/sweep_trace.txt 300 out.json
"""
import csv
import io
import json
import re
import subprocess
import sys

rep, trace, skip, out = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]


def val(d, k):
    v = float(d[k].replace(",", ""))
    u = units[hdr.index(k)]
    return v * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e3, "msecond": 1e6,
                "nsecond": 1.0, "us": 1e3, "ms": 1e6, "ns": 1.0}.get(u, 1.0)


launches = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    launches.append({"duration_ns": val(d, "gpu__time_duration.sum"), "dram_read_bytes": val(d, "dram__bytes_read.sum"),
                     "dram_write_bytes": val(d, "dram__bytes_write.sum")})
by_launch = {}
for ln in open(trace):
    m = re.search(r"kreg-round sweeps=\d+ launch=(\d+) requests=(\d+) launches=\d+ pairs=(\d+) slots=(\d+)", ln)
    if m:
        by_launch[int(m.group(1))] = (int(m.group(2)), int(m.group(3)), int(m.group(4)))
for k, L in enumerate(launches):
    req, pairs, slots = by_launch[skip + k]
    L.update({"launch_index": skip + k, "requests": req, "pairs": pairs, "slots": slots,
              "algorithmic_bytes": 8 * pairs, "slot_bytes": 16 * slots})
n = len(launches)
dram = sum(L["dram_read_bytes"] + L["dram_write_bytes"] for L in launches) / n
alg = sum(L["algorithmic_bytes"] for L in launches) / n
slot = sum(L["slot_bytes"] for L in launches) / n
dur = sum(L["duration_ns"] for L in launches) / n
json.dump({"kernel": "k_sweep (fused F + SE(3) gradient + displacement)",
           "command": "KREG_TRACE_ROUNDS=1 B=64 ncu --set full --clock-control none -k regex:^k_sweep$ "
                      f"--launch-skip {skip} -c {n} python tools/prof_traffic.py; tools/make_traffic.py",
           "launches": launches, "mean_dram_bytes_per_launch": dram, "mean_algorithmic_bytes_per_launch": alg,
           "mean_streamed_slot_bytes_per_launch": slot, "traffic_over_algorithmic": dram / alg,
           "traffic_over_slot_bytes": dram / slot, "mean_duration_us": dur / 1e3,
           "dram_rate_TBps": dram / dur / 1e3, "algorithmic_rate_TBps": alg / dur / 1e3,
           "note": "algorithmic bytes = 8 B x pairs of the launch's round (reference pair list {i, c}); slots = "
                   "16-B sweep-list slots incl. tile padding (x_i - Ts z_j travels inline instead of being "
                   "gathered, hence ~2x); DRAM rate under ncu replay (cold L2, serialised)."},
          open(out, "w"), indent=1)
print(open(out).read()[-600:])
