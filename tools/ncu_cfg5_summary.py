"""Markdown table of the key ncu metrics of a capture (used for the cfg5 kernels).

    python tools/ncu_cfg5_summary.py gpurun_out/prof_cfg5_r01.ncu-rep profiles/r01_ncu_cfg5.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("lts__t_requests_srcunit_tex_op_read.sum", "L2 read requests"),
    ("lts__t_sector_op_read_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
]


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(m for m, _ in METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu summary ({rep.split('/')[-1]})", "",
             "cfg5: R-MAT 2^26, d = 16 (1.06 B edges), k = 256, k' = 64; 64M-query batch.  "
             "`ncu --set full --clock-control none`, cold caches, serialised.", "",
             "| kernel | " + " | ".join(name for _, name in METRICS) + " |",
             "|---|" + "---|" * len(METRICS)]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("dbl::", "")
        cells = [f"{d.get(m, '')} {u.get(m, '')}".strip() for m, _ in METRICS]
        lines.append(f"| `{name}` | " + " | ".join(cells) + " |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
