"""Summarize an ncu launch list (gpu__time_duration + dram bytes, --csv) into
per-kernel means: launch_summary.json and traffic.json (the per-launch DRAM
bytes of the step's dominant kernels, read by bench.py as roofline.traffic).

    python tools/summarize_launches.py gpurun_out/launches_<tag>.csv profiles/r1
"""
import collections
import csv
import json
import os
import sys


def main(src, outdir):
    rows = list(csv.reader(open(src)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            h, start = r, i + 1
            break
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit")
    per = collections.defaultdict(lambda: collections.defaultdict(list))
    scale = {"ns": 1, "us": 1e3, "ms": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows[start:]:
        if len(r) <= vi or r[ki].startswith("void at::") or r[ki].startswith("at::"):
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("sk::", "")
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        per[name][r[mi]].append(v)
    summ = {}
    for k, m in per.items():
        summ[k] = {"ns": sum(m["gpu__time_duration.sum"]) / len(m["gpu__time_duration.sum"]),
                   "n": len(m["gpu__time_duration.sum"])}
        for key, met in (("dram_read", "dram__bytes_read.sum"), ("dram_write", "dram__bytes_write.sum")):
            if m.get(met):
                summ[k][key] = sum(m[met]) / len(m[met])
    os.makedirs(outdir, exist_ok=True)
    json.dump(summ, open(os.path.join(outdir, "launch_summary.json"), "w"), indent=1)
    traffic = {}
    for k, v in summ.items():
        base = k.split("<")[0]
        if base in ("score_kernel", "score_reg_kernel", "decode_mma_kernel", "topk_cluster_kernel", "prologue_kernel") and "dram_read" in v:
            traffic[base] = v["dram_read"] + v.get("dram_write", 0.0)
    json.dump(traffic, open(os.path.join(outdir, "traffic.json"), "w"), indent=1)
    for k, v in summ.items():
        print(f"{k:40s} n={v['n']:2d} {v['ns'] / 1e3:9.1f} us  read {v.get('dram_read', 0) / 1e6:9.1f} MB"
              f"  write {v.get('dram_write', 0) / 1e6:8.1f} MB")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
