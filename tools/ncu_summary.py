"""Summarises ncu output brought back in gpurun_out/ into profiles/.

    python tools/ncu_summary.py launches <launches.csv> <out.md>
    python tools/ncu_summary.py full <report.ncu-rep> <out.md> [--json out.json --cells N --workload c3]
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def launches(path, out):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = defaultdict(list)
    for r in rows[1:]:
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue  # (lists captured with extra metrics)
        name = r[ki].split("(")[0].replace("mas::<unnamed>::", "")
        v = float(r[vi].replace(",", ""))
        agg[name].append(v / 1000.0 if r[ui] == "ns" else v)
    tot = sum(sum(v) for v in agg.values())
    lines = ["| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v)/len(v):.1f} | {sum(v):.1f} | {100*sum(v)/tot:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out, js=None, cells=None, workload=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")].split("(")[0].replace("mas::<unnamed>::", "")}
        for k in KEYS:
            if k in h:
                d[k] = (v[h.index(k)], u[h.index(k)])
        stalls = []
        for i, n in enumerate(h):
            if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued"):
                try:
                    stalls.append((float(v[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(x for x, _ in stalls) or 1
        d["stalls"] = [(n, round(100 * x / tot, 1)) for x, n in sorted(stalls, reverse=True)[:8]]
        res.append(d)
    lines = []
    for d in res:
        lines.append(f"### {d['kernel']}\n")
        lines.append("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in d:
                lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
        lines.append("\nwarp stall samples (share of all samples): " +
                     ", ".join(f"{n} {p}%" for n, p in d["stalls"]) + "\n")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if js:
        d = res[0]

        def num(k, scale):
            val, unit = d[k]
            val = float(val.replace(",", ""))
            return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6,
                          "ms": 1e-3, "ns": 1e-9}.get(unit, 1) / scale

        traffic = num("dram__bytes_read.sum", 1) + num("dram__bytes_write.sum", 1)
        rec = {"kernel": d["kernel"], "workload": workload, "report": rep,
               "dram_bytes_per_launch": traffic,
               "duration_s": num("gpu__time_duration.sum", 1)}
        if cells:
            rec["algorithmic_bytes_per_launch"] = 5.125 * cells
            rec["traffic_over_algorithmic"] = traffic / (5.125 * cells)
        json.dump(rec, open(js, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        args = sys.argv[2:]
        js = cells = wl = None
        if "--json" in args:
            js = args[args.index("--json") + 1]
        if "--cells" in args:
            cells = int(args[args.index("--cells") + 1])
        if "--workload" in args:
            wl = args[args.index("--workload") + 1]
        full(args[0], args[1], js, cells, wl)
