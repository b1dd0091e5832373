"""Summarise an `ncu --csv --metrics gpu__time_duration.sum[,dram__bytes_*]` launch list
into per-kernel shares (JSON on stdout or into a file).

usage: python tools/ncu_summary.py launches.csv [out.json] [--command "..."]
"""
import argparse
import collections
import csv
import json
import re


def summarise(path, from_kernel=None, launches=None):
    """Per-kernel shares.  from_kernel / launches: keep only the `launches`
    launches that start at the first launch whose name contains `from_kernel`
    (e.g. the decode steps after the engine's cuBLASLt tuning)."""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    idx = {h: i for i, h in enumerate(hdr)}
    body = [r for r in rows[hi + 1:] if len(r) >= len(hdr)]
    if from_kernel:
        ids = []
        for r in body:
            if r[idx["ID"]] not in ids:
                ids.append(r[idx["ID"]])
        names = {r[idx["ID"]]: r[idx["Kernel Name"]] for r in body}
        start = next(i for i, k in enumerate(ids) if from_kernel in names[k])
        keep = set(ids[start:start + launches] if launches else ids[start:])
        body = [r for r in body if r[idx["ID"]] in keep]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in body:
        name = re.sub(r"\(.*", "", r[idx["Kernel Name"]]).strip()[:80]
        metric, val = r[idx["Metric Name"]], float(r[idx["Metric Value"]].replace(",", ""))
        if metric == "gpu__time_duration.sum":
            agg[name][0] += 1
            agg[name][1] += val
        elif metric in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            agg[name][2] += val
    total = sum(v[1] for v in agg.values())
    out = []
    for k, (n, ns, dram) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append({"kernel": k, "launches": n, "share": round(ns / total, 4), "total_ms": round(ns / 1e6, 3),
                    "avg_us": round(ns / n / 1e3, 2), "dram_bytes_per_launch": dram / n if dram else None})
    return {"total_ms": total / 1e6, "kernels": out}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("out", nargs="?")
    ap.add_argument("--command", default=None)
    ap.add_argument("--from-kernel", default=None)
    ap.add_argument("--launches", type=int, default=None)
    a = ap.parse_args()
    s = summarise(a.csv, a.from_kernel, a.launches)
    s["command"] = a.command
    s["note"] = "ncu per-launch times are cold-cache and serialised: compare shares, not absolutes"
    text = json.dumps(s, indent=1)
    if a.out:
        open(a.out, "w").write(text)
    for k in s["kernels"][:20]:
        print(f"{100 * k['share']:5.1f}% n={k['launches']:5d} avg_us={k['avg_us']:9.2f}  {k['kernel']}")
