"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys


def summarise(path, top=20):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hdr]
    ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split('(')[0].replace('kreg_dev::', '').replace('(anonymous namespace)::', '').replace('void ', '').replace('<unnamed>::', '')
        v = float(r[vi].replace(',', ''))
        v *= {'nsecond': 1e-3, 'usecond': 1.0, 'msecond': 1e3, 'ns': 1e-3, 'us': 1.0, 'ms': 1e3}.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    out = []
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{k[:48]:48s} n={n:5d} total={t / 1e3:8.3f} ms avg={t / n:8.2f} us share={t / tot * 100:5.1f}%")
    out.append(f"total {tot / 1e3:.3f} ms over {sum(a[0] for a in agg.values())} launches")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
