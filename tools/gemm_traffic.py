#!/usr/bin/env python3
"""profiles/gemm_traffic.json from ncu launch lists that carry
dram__bytes_read.sum / dram__bytes_write.sum: DRAM bytes per GEMM launch
(gemm_tc_kernel*), cold (ncu's default cache flush between replays) and warm
(--cache-control none, the in-step-like case).

  python tools/gemm_traffic.py COLD.csv WARM.csv OUT.json [note]"""
import collections
import csv
import json
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
        "msecond": 1e3}


def per_launch(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    per = collections.defaultdict(dict)
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        if not d["Kernel Name"].startswith("void tc::gemm_tc_kernel"):
            continue
        per[d["ID"]][d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
    n = len(per)
    by = sum(m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0) for m in per.values())
    us = sum(m.get("gpu__time_duration.sum", 0.0) for m in per.values())
    return n, by, us


def main():
    cold, warm, out = sys.argv[1:4]
    note = sys.argv[4] if len(sys.argv) > 4 else ""
    nc, bc, uc = per_launch(cold)
    nw, bw, uw = per_launch(warm)
    res = {"kernel": "gemm_tc_kernel (all GEMM launches of the C2 step)",
           "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                     f"--clock-control none on bench.py (C2); cold = default cache control ({cold}), "
                     f"warm = --cache-control none ({warm})",
           "launches": nc, "dram_bytes_total": bc, "dram_bytes_per_launch": bc / nc if nc else None,
           "warm": {"launches": nw, "dram_bytes_per_launch": bw / nw if nw else None,
                    "us_per_launch": uw / nw if nw else None},
           "cold_us_per_launch": uc / nc if nc else None,
           "note": note or "dram_bytes_per_launch (the bench's roofline.traffic) is the cold-cache "
                           "figure: an upper bound on the in-step traffic, where activations and "
                           "weights are often L2-resident (the warm figure)"}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
