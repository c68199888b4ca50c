"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel:
launches, total device time and share.  Usage: python scripts/launch_share.py launches.csv"""
import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    m = re.search(r"(\w+_kernel|\w+Kernel)\b", name)
    return m.group(1) if m else name[:60]


def main(path):
    rows = [r for r in csv.DictReader(l for l in open(path) if not l.startswith("=="))]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        v = float(r["Metric Value"])
        unit = r["Metric Unit"]
        v = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v   # -> us
        agg[k][0] += 1
        agg[k][1] += v
    total = sum(v for _, v in agg.values())
    print(f"{'kernel':40s} {'launches':>9s} {'total_us':>12s} {'share':>7s}")
    for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {c:9d} {v:12.1f} {100 * v / total:6.2f}%")
    print(f"{'TOTAL':40s} {sum(c for c, _ in agg.values()):9d} {total:12.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
