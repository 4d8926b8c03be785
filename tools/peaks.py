#!/usr/bin/env python3
"""Context roofs on this box (not the bench denominators, which come from
MEASURED_PEAKS.json): a read-only HBM stream and cuBLASLt int8 GEMM throughput
(torch._int_mm), each timed back to back for ~2 s with clocks sampled."""
import json
import subprocess
import time

import torch


def clocks_during(fn, seconds=2.0):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                          "--format=csv,noheader,nounits", "-lms", "100"],
                         stdout=subprocess.PIPE, text=True)
    t0 = time.time()
    n = 0
    while time.time() - t0 < seconds:
        fn()
        n += 1
    torch.cuda.synchronize()
    p.terminate()
    out = p.communicate()[0].strip().splitlines()
    sm = sorted(float(l.split(",")[0]) for l in out if l.strip())
    return n, (sm[len(sm) // 2] if sm else None)


def timed(fn, iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    res = {}
    # read-only stream: int64 sum over 4 GiB (result is one scalar)
    x = torch.randint(0, 1 << 30, (1 << 29,), dtype=torch.int64, device="cuda")
    f = lambda: x.sum()
    for _ in range(5):
        f()
    ms = timed(f, 50)
    _, clk = clocks_during(f, 1.0)
    res["hbm_read_only_gbs"] = round(x.numel() * 8 / (ms / 1e3) / 1e9, 1)
    res["hbm_read_only_clk"] = clk
    del x
    # cuBLASLt int8 GEMM, C4-like shape: (M x K) @ (K x N), int32 accumulate
    for (M, K, N) in [(8192, 65536, 256), (8192, 65536, 1024), (16384, 16384, 4096)]:
        a = torch.randint(-128, 127, (M, K), dtype=torch.int8, device="cuda")
        b = torch.randint(-128, 127, (K, N), dtype=torch.int8, device="cuda")
        g = lambda: torch._int_mm(a, b)
        for _ in range(3):
            g()
        ms = timed(g, 20)
        n, clk = clocks_during(g, 2.0)
        res[f"int_mm_{M}x{K}x{N}_tops"] = round(2.0 * M * K * N / (ms / 1e3) / 1e12, 1)
        res[f"int_mm_{M}x{K}x{N}_sustained_clk"] = clk
        del a, b
    print(json.dumps(res))


if __name__ == "__main__":
    main()
