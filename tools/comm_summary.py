"""Summarise C3D_PROF_DUMP collective records (stderr of a bench run).

usage: python tools/comm_summary.py LOG [ranks] [steps]
"""
import collections
import re
import sys

NAMES = ["bcast", "AG", "RS", "AR", "barrier", "enter", "GEMM+RS", "AG+GEMM+RS", "finish"]


def main():
    path = sys.argv[1]
    ranks = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    d = collections.defaultdict(lambda: [0, 0.0])
    for line in open(path):
        m = re.search(r"kind=(\d+) bytes=(\d+) us=([\d.]+)", line)
        if m:
            k = (int(m[1]), int(m[2]))
            d[k][0] += 1
            d[k][1] += float(m[3])
    tot = 0.0
    div = ranks * steps
    for k, (n, t) in sorted(d.items(), key=lambda kv: -kv[1][1]):
        print(f"  {NAMES[k[0]]:6s} {k[1] / 1e6:9.3f} MB  calls/step={n / div:5.1f}  "
              f"avg_us={t / n:7.1f}  us/step={t / div:8.1f}")
        tot += t / div
    print(f"  total collective us/step/rank = {tot:.1f}")


if __name__ == "__main__":
    main()
