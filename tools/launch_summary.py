"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per-kernel
count, total and mean device time, share of the captured launches.

usage: python tools/launch_summary.py launches.csv [steps]
"""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"<.*", "", name) if not name.startswith("void c3d") else name
    return name.replace("void ", "")[:70]


def main():
    path = sys.argv[1]
    steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
        rows.append((r["Kernel Name"], r.get("Grid Size", ""), r.get("Block Size", ""), us))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, g, b, us in rows:
        k = short(name)
        agg[k][0] += 1
        agg[k][1] += us
    total = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {total:.1f} us total ({total / steps:.1f} us per step)")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{t / steps:9.1f} us/step {100 * t / total:5.1f}%  n/step={n / steps:5.1f}  "
              f"mean={t / n:7.1f} us  {k}")


if __name__ == "__main__":
    main()
