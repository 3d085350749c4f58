"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv
import statistics
import sys
from collections import defaultdict


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)  # -> us
        rows.append((r["Kernel Name"], r.get("Grid Size", ""), v))
    return rows


def main(path, by_grid=False):
    rows = load(path)
    g = defaultdict(list)
    for name, grid, us in rows:
        short = name.replace("(anonymous namespace)::", "").replace("void ", "").replace("dpk::", "")
        short = short.split("(")[0]
        g[(short, grid) if by_grid else short].append(us)
    total = sum(us for _, _, us in rows)
    print(f"{len(rows)} launches, {total / 1000:.3f} ms total")
    for k, v in sorted(g.items(), key=lambda kv: -sum(kv[1])):
        print(f"{sum(v) / 1000:9.3f} ms {100 * sum(v) / total:5.1f}%  n={len(v):4d}  median {statistics.median(v):8.1f} us  max {max(v):8.1f} us  {k}")


if __name__ == "__main__":
    main(sys.argv[1], "--grid" in sys.argv)
