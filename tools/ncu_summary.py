#!/usr/bin/env python3
"""Summarise an ncu report (.ncu-rep) or a launch-list CSV into profiles/.

    python tools/ncu_summary.py full  gpurun_out/prof.ncu-rep  profiles/<name>.md [--traffic profiles/traffic_<w>.json]
    python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/<name>.md
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_int8_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "smsp__cycles_active.avg", "sm__cycles_elapsed.avg.per_second", "gpc__cycles_elapsed.max",
    "dram__cycles_elapsed.avg.per_second",
]


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def full(rep, dst, traffic=None):
    hdr, units, data = raw(rep)
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --set full summary: `{rep}`", ""]
    for r in data:
        name = r[idx.get("Kernel Name", 0)]
        lines.append(f"## {name[:160]}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k in KEYS:
            if k in idx:
                lines.append(f"| {k} | {r[idx[k]]} | {units[idx[k]]} |")
        # stall reasons
        st = [(h, r[i]) for h, i in idx.items() if h.startswith("smsp__average_warp_latency_issue_stalled")
              or (h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"))]
        vals = []
        for h, v in st:
            try:
                vals.append((float(v.replace(",", "")), h))
            except ValueError:
                pass
        vals.sort(reverse=True)
        if vals:
            lines.append("")
            lines.append("top stall reasons (pc sampling):")
            for v, h in vals[:8]:
                lines.append(f"- {h}: {v}")
        lines.append("")
        if traffic:
            def num(k):
                return float(r[idx[k]].replace(",", "")) * (1e9 if units[idx[k]] == "Gbyte" else
                                                            1e6 if units[idx[k]] == "Mbyte" else
                                                            1e3 if units[idx[k]] == "Kbyte" else 1)
            t = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
            json.dump({"dram_bytes_per_launch": t, "kernel": name, "source": rep}, open(traffic, "w"))
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def launches(src, dst):
    txt = open(src).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = r[idx["Kernel Name"]].split("(")[0]
        v = float(r[idx["Metric Value"]].replace(",", ""))
        unit = r[idx["Metric Unit"]]
        v = v / 1e3 if unit in ("nsecond", "ns") else v * 1e3 if unit in ("msecond", "ms") else v
        tot[k] += v
        cnt[k] += 1
    allt = sum(tot.values())
    lines = [f"# ncu launch list: `{src}`", "", "| kernel | launches | total us | mean us | share |",
             "|---|---|---|---|---|"]
    for k in sorted(tot, key=lambda x: -tot[x]):
        lines.append(f"| {k[:90]} | {cnt[k]} | {tot[k]:.1f} | {tot[k] / cnt[k]:.2f} | {tot[k] / allt:.3f} |")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    tr = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    full(src, dst, tr) if mode == "full" else launches(src, dst)
