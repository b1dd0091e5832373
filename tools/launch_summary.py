"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import csv
import sys

for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr, data = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = d["Kernel Name"].split("(")[0][-40:]
            data.setdefault((d["ID"], k), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    print(f)
    agg = {}
    for (i, k), m in data.items():
        agg.setdefault(k, []).append(m)
    for k, l in agg.items():
        t = sum(x["gpu__time_duration.sum"] for x in l) / len(l)
        by = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in l) / len(l)
        print(f"  {k:40s} n={len(l):3d} avg {t / 1000:.2f} us  {by / 1e6:.1f} MB  {by / t:.0f} GB/s")
