#!/usr/bin/env python3
"""Tuning sweep: run bench.py per (workload, env override) and print one line each.

    python tools/sweep.py c2 QPIR_GEMV_U=1,2,4 QPIR_GEMV_UNROLL=4,8 [-- extra bench args]
"""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    args = sys.argv[1:]
    extra = []
    if "--" in args:
        i = args.index("--")
        args, extra = args[:i], args[i + 1:]
    wl, specs = args[0], args[1:]
    keys = [s.split("=")[0] for s in specs]
    vals = [s.split("=")[1].split(",") for s in specs]
    for combo in itertools.product(*vals) if specs else [()]:
        env = dict(os.environ)
        env.update(dict(zip(keys, combo)))
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", wl,
               "--no-cpu-baseline", "--no-e2e", *extra]
        p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
        line = [l for l in p.stdout.splitlines() if l.startswith("{")]
        tag = " ".join(f"{k}={v}" for k, v in zip(keys, combo))
        if not line:
            print(f"{wl} {tag}: FAILED rc={p.returncode} {p.stderr[-400:]}", flush=True)
            continue
        j = json.loads(line[-1])
        r = j["roofline"]
        print(f"{wl} {tag}: value={j['value']} {j['unit']} ms/step={j['ms_per_step']} "
              f"roof={r['achieved']} frac={r['frac']} clk={j['clocks'].get('sm_mhz')} "
              f"reasons={j['clocks'].get('reasons')}", flush=True)


if __name__ == "__main__":
    main()
