"""Markdown summary of an ncu report (one section per captured kernel) plus
the launch-list shares of a `--metrics gpu__time_duration.sum` CSV.

usage: python tools/ncu_summary.py REPORT.ncu-rep [LAUNCHES.csv]
"""

import collections
import csv
import io
import re
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__inst_executed.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def kernels(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(head, r))
        yield d["Kernel Name"], [(m, d.get(m, ""), units[head.index(m)] if m in head else "") for m in METRICS]


def launches(path):
    tot = collections.OrderedDict()
    with open(path) as fh:
        text = "".join(l for l in fh if not l.startswith("=="))
    for r in csv.DictReader(io.StringIO(text)):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"[<(].*", "", r["Kernel Name"]).replace("void ", "").replace("hcnn::", "")
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(
            r.get("Metric Unit", "ns"), 1e-6)
        c, t = tot.get(name, (0, 0.0))
        tot[name] = (c + 1, t + float(r["Metric Value"].replace(",", "")) * scale)
    return tot


if __name__ == "__main__":
    for name, ms in kernels(sys.argv[1]):
        print(f"## {name[:90]}\n")
        for m, v, u in ms:
            print(f"- `{m}`: {v} {u}")
        print()
    if len(sys.argv) > 2:
        tot = launches(sys.argv[2])
        all_ms = sum(t for _, t in tot.values())
        print("## Launch-list shares (one `--profile-only` step incl. setup kernels)\n")
        print("| kernel | launches | ms (cold, serialised) | share |\n|---|---|---|---|")
        for name, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
            print(f"| {name} | {c} | {t:.3f} | {t / all_ms:.3f} |")
