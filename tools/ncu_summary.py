"""Summarise ncu captures into profiles/ (run here, on the .ncu-rep / csv from gpurun_out).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep gpurun_out/launches.csv profiles/rNN_ncu.md
Writes the markdown summary and updates profiles/ncu_traffic.json (dram bytes per
launch of each profiled kernel, used by bench.py as roofline.traffic).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__t_requests_srcunit_tex.sum", "L2 requests (SM)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("smsp__average_warp_latency_issue_stalled_barrier", "stall barrier"),
]


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("void ", "").replace("dbl::", "")


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    return float(v) * scale.get(unit, 1)


def to_us(v, unit):
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3,
             "second": 1e6, "s": 1e6}
    return float(v) * scale.get(unit, 1)


def main(rep, launches, out_md):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    col = {m: h.index(m) for m, _ in METRICS if m in h}
    kn = h.index("Kernel Name")
    lines = ["| kernel | " + " | ".join(lbl for m, lbl in METRICS if m in col) + " |",
             "|---|" + "---|" * len(col)]
    traffic, l2req = {}, {}
    for r in rows[2:]:
        cells = []
        for m, _ in METRICS:
            if m not in col:
                continue
            cells.append(f"{r[col[m]]} {units[col[m]]}".strip())
        lines.append(f"| `{short(r[kn])}` | " + " | ".join(cells) + " |")
        rb = to_bytes(r[col["dram__bytes_read.sum"]].replace(",", ""), units[col["dram__bytes_read.sum"]])
        wb = to_bytes(r[col["dram__bytes_write.sum"]].replace(",", ""), units[col["dram__bytes_write.sum"]])
        key = short(r[kn]).split("<")[0]
        traffic.setdefault(key, []).append(rb + wb)
        if "lts__t_requests_srcunit_tex.sum" in col:
            l2req.setdefault(key, []).append(float(r[col["lts__t_requests_srcunit_tex.sum"]].replace(",", "")))
    # launch list shares
    share = defaultdict(float)
    total = 0.0
    if launches and os.path.exists(launches):
        lr = list(csv.reader(open(launches)))
        hi = [i for i, r in enumerate(lr) if "Kernel Name" in r][0]
        H = lr[hi]
        ki, mi, ui = H.index("Kernel Name"), H.index("Metric Value"), H.index("Metric Unit")
        for r in lr[hi + 1:]:
            if len(r) <= mi:
                continue
            t = to_us(r[mi].replace(",", ""), r[ui])
            share[short(r[ki]).split("<")[0]] += t
            total += t
    md = [f"# ncu summary ({os.path.basename(rep)})", "",
          "Full-set captures (`ncu --set full --clock-control none`, cold caches, serialised):", ""]
    md += lines
    if total:
        md += ["", "Launch list (`--metrics gpu__time_duration.sum`), total device time per kernel:", "",
               "| kernel | total us | share |", "|---|---|---|"]
        for k, t in sorted(share.items(), key=lambda kv: -kv[1]):
            md.append(f"| `{k}` | {t:.1f} | {100 * t / total:.1f}% |")
    open(out_md, "w").write("\n".join(md) + "\n")
    tj = os.path.join(os.path.dirname(out_md), "ncu_traffic.json")
    old = json.load(open(tj)) if os.path.exists(tj) else {}
    for k, v in traffic.items():
        old[k] = sum(v) / len(v)
    json.dump(old, open(tj, "w"), indent=1, sort_keys=True)
    lj = os.path.join(os.path.dirname(out_md), "ncu_l2req.json")
    old = json.load(open(lj)) if os.path.exists(lj) else {}
    for k, v in l2req.items():
        old[k] = sum(v) / len(v)
    json.dump(old, open(lj, "w"), indent=1, sort_keys=True)
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 3 else None, sys.argv[-1])
