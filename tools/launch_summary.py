#!/usr/bin/env python3
"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes])
per kernel: count, total/avg time, share, DRAM bytes and achieved GB/s."""
import collections
import csv
import sys

# time -> microseconds, bytes -> bytes
UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
        "second": 1e6, "s": 1e6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, top=40, steps=None):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    per = collections.defaultdict(dict)
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        per[(d["ID"], d["Kernel Name"])][d["Metric Name"]] = v
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), m in per.items():
        a = agg[name.split("(")[0][:70]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'us':>9} {'share':>6} {'n':>4} {'avg_us':>8} {'GB/s':>7}  kernel   (launches={len(per)}, total {tot:.0f} us)")
    if steps:
        print(f"  (per step over {steps} profiled steps: {tot / steps:.0f} us)")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{t:9.1f} {100*t/tot:5.1f}% {n:4d} {t/n:8.2f} {b/t/1e3 if t else 0:7.0f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], steps=int(sys.argv[2]) if len(sys.argv) > 2 else None)
