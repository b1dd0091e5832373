"""profiles/ncu_attention_c2.json from the att_tail ncu CSV of tools/r2_prof_att.sh: per-kernel serialised
time and DRAM bytes of qdots / core / vsum at the bench's final tail (320 rows), averaged over the 32 layers.

usage: python tools/att_tail_json.py gpurun_out/r2/att_tail_T.csv profiles/ncu_attention_c2.json
"""
import collections
import csv
import json
import sys

ALG = 235290624  # algorithmic bytes of one C2 layer (16 instances) at tail 320, DESIGN.md §3
PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]


def main(src, dst):
    rows = [r for r in csv.reader(open(src)) if r]
    hi = [i for i, r in enumerate(rows) if r[0] == "ID"][0]
    idx = {h: i for i, h in enumerate(rows[hi])}
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    names = {}
    for r in rows[hi + 1:]:
        if len(r) < len(idx):
            continue
        k = r[idx["Kernel Name"]]
        if not any(x in k for x in ("qdots", "core_kernel", "vsum")):
            continue
        short = k.split("::")[-1].split("(")[0]
        names[r[idx["ID"]]] = short
        v = float(r[idx["Metric Value"]].replace(",", ""))
        per[r[idx["ID"]]][r[idx["Metric Name"]]] = v
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for i, m in per.items():
        for k, v in m.items():
            agg[names[i]][k].append(v)
    kernels, tot_t, tot_b = {}, 0.0, 0.0
    for k, m in agg.items():
        t = sum(m["gpu__time_duration.sum"]) / len(m["gpu__time_duration.sum"]) / 1e3
        b = (sum(m["dram__bytes_read.sum"]) + sum(m["dram__bytes_write.sum"])) / len(m["dram__bytes_read.sum"])
        kernels[k] = {"launches": len(m["gpu__time_duration.sum"]), "us_per_launch": round(t, 2),
                      "dram_bytes_per_launch": int(b), "dram_GBps": round(b / t / 1e3, 1),
                      "frac_of_hbm_peak": round(b / t / 1e3 / PEAK, 3)}
        tot_t += t
        tot_b += b
    out = {"round": 2, "config": "c2", "tail_tokens": 320, "source": "ncu --profile-from-start off --metrics "
           "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none python "
           "tools/ncu_tail.py c2 256 (tools/r2_prof_att.sh)", "note": "one decode-attention layer (16 instances) = "
           "qdots + core (split mode) + vsum at tail 320; cold-cache serialised replay (no PDL overlap), averaged "
           "over the 32 layers", "peak_gbs": PEAK, "algorithmic_bytes_per_layer": ALG,
           "dram_bytes_per_layer": int(tot_b), "traffic_over_algorithmic": round(tot_b / ALG, 4),
           "serialised_us_per_layer": round(tot_t, 2), "kernels": kernels}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:3])
