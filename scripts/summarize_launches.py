"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list by kernel."""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(anonymous namespace\)::", "", name)
    name = re.sub(r"dart::", "", name)
    return name[:90]


def main(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "ns")
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
            rows.append((short(r["Kernel Name"]), v * scale))
    agg = defaultdict(lambda: [0, 0.0])
    for n, t in rows:
        agg[n][0] += 1
        agg[n][1] += t
    total = sum(t for _, t in rows)
    print(f"{len(rows)} launches, {total/1000:.3f} ms total (serialised, cold cache)")
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{t/1000:9.3f} ms {100*t/total:5.1f}% {c:5d}x  {n}")


if __name__ == "__main__":
    main(sys.argv[1])
