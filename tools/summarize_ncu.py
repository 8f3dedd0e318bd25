"""Summarize ncu artefacts into the text files committed under profiles/.

  python tools/summarize_ncu.py report.ncu-rep [...]      -> key metrics per kernel launch
  python tools/summarize_ncu.py --launches launches.csv    -> per-kernel share of one coloring
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
       "l1tex__m_xbar2l1tex_read_bytes.sum", "smsp__inst_executed.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarize(rep):
    lines = [f"# {rep}"]
    rows = ncu_csv(rep, "details")
    hdr = rows[0]
    ni, vi, ui, ki, ii = (hdr.index(x) for x in ("Metric Name", "Metric Value", "Metric Unit", "Kernel Name", "ID"))
    last = None
    for r in rows[1:]:
        if r[ii] != last:
            lines.append(f"## launch {r[ii]}: {r[ki][:110]}")
            last = r[ii]
        if r[ni] in KEYS:
            lines.append(f"  {r[ni]:38s} {r[vi]:>14s} {r[ui]}")
    raw = ncu_csv(rep, "raw")
    hdr, units = raw[0], raw[1]
    for vals in raw[2:]:
        lines.append("  -- raw")
        for name in RAW:
            if name in hdr:
                i = hdr.index(name)
                lines.append(f"  {name:55s} {vals[i]:>18s} {units[i]}")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st.append((float(vals[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1.0
        lines.append("  stall samples: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:6]))
    return "\n".join(lines)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    agg = {}
    for r in rows[1:]:
        ms = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        name = r[ki].split("(")[0].strip()
        a = agg.setdefault(name, [0.0, 0])
        a[0] += ms
        a[1] += 1
    tot = sum(a[0] for a in agg.values())
    out = [f"# {path}: {sum(a[1] for a in agg.values())} launches, {tot:.3f} ms (ncu, serialized, cold caches)"]
    for name, (ms, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        out.append(f"  {ms:10.3f} ms {100 * ms / tot:5.1f}%  {c:5d} x  {name}")
    return "\n".join(out)


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--launches":
        for p in args[1:]:
            print(launches(p))
    else:
        for p in args:
            print(summarize(p))
