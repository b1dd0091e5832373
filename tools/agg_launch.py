"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name.
usage: python tools/agg_launch.py file.csv [skip_first_n_launches]"""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, mi = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Name')
data = [(r[ki], float(r[vi].replace(',', ''))) for r in rows[1:] if r[mi] == 'gpu__time_duration.sum']
data = data[int(sys.argv[2]) if len(sys.argv) > 2 else 0:]
agg = collections.defaultdict(lambda: [0, 0.0])
for n, v in data:
    agg[n[:90]][0] += 1
    agg[n[:90]][1] += v
print(f"total {sum(v for _, v in data) / 1e6:.3f} ms over {len(data)} launches")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 20]:
    print(f"{v / 1e6:9.3f} ms {c:6d}  {n}")
