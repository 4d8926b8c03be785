#!/usr/bin/env python3
"""Per-source-line instruction and stall-sample shares of one kernel in an
.ncu-rep (ncu --import-source on), plus the headline issue / pipe metrics.

    python tools/ncu_lines.py report.ncu-rep [top_n]
"""
import collections
import csv
import io
import subprocess
import sys


def _csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, top=30):
    raw = _csv(rep, "--page", "raw")
    keys = ("gpu__time_duration.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__inst_issued.avg.per_cycle_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sass__inst_executed_per_opcode", "sass__inst_executed_shared_loads",
            "sass__inst_executed_shared_stores", "launch__registers_per_thread",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
    for k, v in zip(raw[0], raw[2]):
        if k in keys:
            print(f"{k} {v}")
    rows = _csv(rep, "--page", "source", "--print-source", "cuda,sass")
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    text, cur = {}, None
    for r in rows:
        if len(r) < 8 or r[0] == "Line No":
            continue
        if r[0]:
            cur = r[0]
            text[cur] = r[1]
        try:
            agg[cur][0] += float(r[7] or 0)
            agg[cur][1] += float(r[4] or 0)
        except ValueError:
            pass
    tot = sum(v[0] for v in agg.values()) or 1
    tots = sum(v[1] for v in agg.values()) or 1
    print("inst%  stall%  line")
    for ln, (n, s) in sorted(agg.items(), key=lambda t: -t[1][0])[:top]:
        print(f"{n / tot * 100:5.1f} {s / tots * 100:6.1f}  L{ln}: {text.get(ln, '')[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
