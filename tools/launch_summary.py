"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel name, launches,
mean duration and share of the total device time."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        agg[r[ki].split("(")[0]].append(v * scale)
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:40]:40s} n={len(v):4d} mean={sum(v) / len(v):9.1f}us share={sum(v) / tot:.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
