"""Per-phase DRAM traffic of one coloring from an ncu CSV
(--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum).

  python tools/ncu_traffic.py CONFIG NODES_WITH_SPMM launches.csv [profiles/ncu_traffic.json]

Kernels are grouped into the SpMM phase (bucket_*, rooted_*, spmm_*: every
kernel that produces a P'), the eMA phase (ema_*, root_reduce) and the rest
(coloring).  `dram_bytes_per_launch` is the SpMM phase's DRAM bytes divided by
the number of node-level SpMMs (bench.py's roofline `launches` unit)."""
import csv
import json
import sys
from collections import defaultdict


def phase(name):
    if name.startswith(("bucket_", "rooted_", "spmm_", "lspmm", "color_bucket", "pair_expand", "seg_")):
        return "spmm"
    if name.startswith(("ema_", "root_reduce")):
        return "ema"
    return "other"


def main():
    cfg, nodes, path = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    out = sys.argv[4] if len(sys.argv) > 4 else None
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, ii, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}
    per = defaultdict(lambda: {"name": "", "read": 0.0, "write": 0.0, "time": 0.0})
    for r in rows[1:]:
        d = per[r[ii]]
        d["name"] = r[ki].split("(")[0].strip().replace("void ", "").replace("tcg::dev::", "").replace("tcg::", "")
        val = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        if r[mi] == "dram__bytes_read.sum":
            d["read"] = val
        elif r[mi] == "dram__bytes_write.sum":
            d["write"] = val
        elif r[mi] == "gpu__time_duration.sum":
            d["time"] = val
    agg = defaultdict(lambda: defaultdict(float))
    kern = defaultdict(lambda: defaultdict(float))
    for d in per.values():
        p = phase(d["name"].split("<")[0])
        for key in ("read", "write", "time"):
            agg[p][key] += d[key]
            kern[d["name"]][key] += d[key]
        kern[d["name"]]["launches"] += 1
    spmm = agg["spmm"]
    res = {
        "dram_bytes_per_launch": (spmm["read"] + spmm["write"]) / max(nodes, 1),
        "unit": "bytes per node-level SpMM (all SpMM-phase kernels of one coloring / SpMM nodes)",
        "spmm_nodes": nodes,
        "phases": {p: {"dram_read": v["read"], "dram_write": v["write"], "ms": v["time"] * 1e3} for p, v in agg.items()},
        "kernels": {k: {"launches": int(v["launches"]), "dram_read": v["read"], "dram_write": v["write"],
                        "ms": v["time"] * 1e3} for k, v in sorted(kern.items(), key=lambda x: -x[1]["time"])},
        "source": path,
    }
    print(json.dumps({cfg: res}, indent=1))
    if out:
        try:
            allr = json.load(open(out))
        except (OSError, ValueError):
            allr = {}
        allr[cfg] = res
        json.dump(allr, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
