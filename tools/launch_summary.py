"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import sys
from collections import defaultdict

tot = defaultdict(float)
cnt = defaultdict(int)
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for row in csv.DictReader(lines):
    if row.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = row["Kernel Name"].split("(")[0].replace("kreg_dev::", "").replace("<unnamed>::", "")
    v = float(row["Metric Value"].replace(",", ""))
    unit = row.get("Metric Unit", "ns")
    v *= {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:40s} {cnt[k]:7d} launches {tot[k] / 1e3:10.2f} ms {100 * tot[k] / T:6.1f} %  avg {tot[k] / cnt[k]:9.1f} us")
print(f"total {T / 1e3:.2f} ms")
