#!/usr/bin/env python3
"""Benchmark of the LWE-PIR answer path (BASELINE.json metric:
"PIR answer DB-scan GB/s and queries/sec per GPU at 1/2/4/8 B200 vs HBM roof").

    python bench.py [--gpus N] [--steps K] [--warmup W]
                    [--workload c1|c2|c3|c4-64|c4-256|c5|ens-c2|ens-c2-b128|ftr-c2-b128|oop-c2|
                                bind-c2|bind-c2-unsigned]
                    [--impl ours|reference] [--no-cpu-baseline] [--no-e2e] [--graph 0|1]
    torchrun --nproc-per-node N bench.py --gpus N ...   (plain `--gpus N` re-runs itself
                                                        under torchrun on 127.0.0.1)

A step = one pass of the whole hot path over one batch of synthetic input:
  c2 (default)  single query on the regional 1.007 GB DB (BASELINE.json configs[1]):
                GEMV kernel (query ingest + scan + reduction fused) [+ NCCL gather, N>1]
  c3            single query on the 32.2 GB nationwide DB row-sharded over N GPUs
  c4-64/256     batch of 64/256 queries on the 8.05 GB DB (limb split + tcgen05 GEMM)
  c5            hint H = D.A (n = 1024) for one rank's shard of the 32 GB DB
  ens-c2 / ens-c2-b128 / ftr-c2-b128 / oop-c2   the NEXT rows (Chor XOR PIR: 1 and 128
                shares; Goldberg PIR over F_65537, 128 queries; CIP-PIR online answer)
  bind-c2       Puzzle.Bind of every C2 record: HCT puzzle + ML-DSA-44 signature on the
                GPU, packed into D (bind-c2-unsigned: the packing alone)
At N > 1, c2 is weak scaling (each rank holds a 40-channel 1.007 GB slice; the
DB grows with N), c3 is strong scaling (fixed 32.2 GB).
value = DB bytes scanned by all ranks / max-over-ranks device time.
"""
from __future__ import annotations

import os

# The CPU oracle (cpu_baseline / --impl reference) uses OpenMP; with torch's
# own OpenMP threads spin-waiting in the same process its parallel regions
# slow down by orders of magnitude.  Passive waiting must be set before any
# OpenMP runtime starts, i.e. before torch is imported.
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")

import argparse
import json
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PIR answer DB-scan GB/s and queries/sec per GPU at 1/2/4/8 B200 vs HBM roof"
FALLBACK_HBM_GBS = 6650.0
FALLBACK_BF16_TFLOPS = 1590.0

WORKLOADS = {
    "c1": dict(name="tiny SAS DB 1024 cells x 16 ch x 8 B (BASELINE configs[0])",
               n_cells=1024, n_ch=16, d=8, kind="answer"),
    "c2": dict(name="regional SAS DB 8192 cells x 40 ch x 3072 B = 1.007 GB, single query "
                    "(BASELINE configs[1])", n_cells=8192, n_ch=40, d=3072, kind="answer"),
    "c3": dict(name="nationwide SAS DB 262144 cells x 40 ch x 3072 B = 32.2 GB row-sharded, "
                    "single query + NCCL gather (BASELINE configs[2])",
               n_cells=262144, n_ch=40, d=3072, kind="answer"),
    "c4-64": dict(name="8.05 GB DB (65536 cells x 40 ch x 3072 B), batch of 64 queries "
                       "(BASELINE configs[3])", n_cells=65536, n_ch=40, d=3072, kind="batch", B=64),
    "c4-256": dict(name="8.05 GB DB (65536 cells x 40 ch x 3072 B), batch of 256 queries "
                        "(BASELINE configs[3])", n_cells=65536, n_ch=40, d=3072, kind="batch", B=256),
    "ens-c2": dict(name="QPADL-ENS (Chor XOR PIR, NEXT-1): 327680 paper-shaped 3 KB records "
                        "= 1.007 GB, one uniform r-bit share", n_cells=8192, n_ch=40, d=3072,
                   kind="ens"),
    "oop-c2": dict(name="QPADL-OOP (CIP-PIR, NEXT-3) online answer of one of n = 4 servers on "
                        "1.007 GB (touches its 1/4 flip chunk) + offline queue of 128 (S, A)",
                   n_cells=8192, n_ch=40, d=3072, kind="oop", n_chunks=4),
    "ens-c2-b128": dict(name="QPADL-ENS multi-request (Alg. 3): 1.007 GB, 128 shares",
                        n_cells=8192, n_ch=40, d=3072, kind="ens_batch", B=128),
    "ftr-c2-b128": dict(name="QPADL-FTR (Goldberg PIR over F_65537, NEXT-2; Alg. 4): 327680 "
                             "paper-shaped 3 KB records = 1.007 GB, 128 Shamir-share queries",
                        n_cells=327680, n_ch=1, d=3072, kind="batch", B=128, modp=65537),
    "bind-c2": dict(name="NEXT-4 PSD.Puzzle.Bind (Alg. 1 step 1): all 327680 records of the "
                         "1.007 GB regional DB built on the GPU (560 B spectrum + 37 B HCT puzzle "
                         "+ 2420 B ML-DSA-44 signature of the puzzle) straight into the D panels",
                    n_cells=8192, n_ch=40, d=3072, kind="bind", sign=True),
    "bind-c2-unsigned": dict(name="NEXT-4 Puzzle.Bind without the signatures (spectrum + HCT "
                                  "puzzle + zero slot): the packing alone", n_cells=8192, n_ch=40,
                             d=3072, kind="bind", sign=False),
    "c5": dict(name="hint D.A, n=1024, one rank's shard of the 32.2 GB DB at G=8 "
                    "(BASELINE configs[4])", n_cells=262144, n_ch=40, d=3072, kind="hint", n=1024,
               shard_of=8),
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return j.get("hbm_gbs", FALLBACK_HBM_GBS), j.get("bf16_tflops", FALLBACK_BF16_TFLOPS), \
            j.get("bf16_tflops_sustained"), "measured"
    return FALLBACK_HBM_GBS, FALLBACK_BF16_TFLOPS, None, "fallback"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index: int):
        self.samples = []
        self.marks = [None, None]
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(gpu_index), "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.samples.append((time.time(), line.strip()))

    def start(self):
        self.marks[0] = time.time()

    def stop(self):
        self.marks[1] = time.time()
        if self.p:
            time.sleep(0.12)
            self.p.terminate()
            try:
                self.p.wait(timeout=2)
            except Exception:
                self.p.kill()

    def summary(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t0, t1 = self.marks
        rows = [s for (t, s) in self.samples if t0 - 0.06 <= t <= t1 + 0.06] or \
               [s for (_, s) in self.samples[-3:]]
        sm, mx, pw, reasons = [], [], [], set()
        for r in rows:
            f = [x.strip() for x in r.split(",")]
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except (ValueError, IndexError):
                continue
            try:
                pw.append(float(f[2]))
            except (ValueError, IndexError):
                pass
            for name, v in zip(self.NAMES, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": statistics.median(pw) if pw else None}


# ---------------------------------------------------------------- helpers
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def physical_gpu(local: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [x for x in vis.split(",") if x.strip()]
        if local < len(ids) and ids[local].strip().isdigit():
            return int(ids[local])
    return local


def build_db(P, wl, n_ch_total, row_begin, row_end, seed, device, lwe_n=1024):
    """Setup (untimed): stream synthetic records, generated on the device in
    256 MB theta-ordered chunks, into this rank's shard (rows outside the shard
    are skipped by the pack kernel)."""
    import synth
    n_cells, d = wl["n_cells"], wl["d"]
    s = P.PirServer(n_cells, n_ch_total, d, lwe_n=lwe_n, seed_A=0x5EED, row_begin=row_begin,
                    row_end=row_end, device=device, stable_inputs=True)
    # stable_inputs: the timed loops answer device queries written (and
    # synchronised) before the loop, never by the kernel right before an answer
    # call, so the scan may start before griddepcontrol.wait (include/qpir.h)
    n_rec = n_cells * n_ch_total
    chunk = max(1, (256 << 20) // d)
    for t0 in range(0, n_rec, chunk):
        n = min(chunk, n_rec - t0)
        rec = synth.records(seed, t0, n, d, n_ch_total, device=f"cuda:{device}")
        s.db_write(t0, rec)
    torch.cuda.synchronize(device)
    return s


def _host_cpu():
    """The host CPU the oracle runs on (record the model)."""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return f"{ln.split(':', 1)[1].strip()}, {os.cpu_count()} logical CPUs"
    except OSError:
        pass
    return f"{os.cpu_count()} logical CPUs"


def _warm_oracle(fn, seconds):
    """Untimed oracle calls for `seconds`: on the GPU box's host the oracle's
    speed rises over the first seconds of a process (13 -> 18+ GB/s,
    tools/baseline_state_probe.py), so every oracle timing starts warm."""
    t0 = time.perf_counter()
    fn()
    while time.perf_counter() - t0 < seconds:
        fn()


def cpu_baseline_answer(wl, seed, budget_s=12.0):
    """The oracle as it stands, on a bounded sample: the first 4 channels of the
    same DB (4 * d rows x n_cells columns), repeated for ~budget_s seconds."""
    import synth
    from oracle import oracle as O
    O.set_num_threads(os.cpu_count() or 1)  # torchrun defaults OMP_NUM_THREADS to 1
    n_cells, d = wl["n_cells"], wl["d"]
    n_ch_s = min(4, wl["n_ch"])
    # theta = cell * n_ch + ch with the FULL n_ch: gather the first n_ch_s channels
    theta = (torch.arange(n_cells).unsqueeze(1) * wl["n_ch"] + torch.arange(n_ch_s)).reshape(-1)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    rec = synth.records_at(seed, theta.to(dev), d, wl["n_ch"], 512).cpu().numpy()
    D = O.pack(rec, n_cells, n_ch_s, d, n_cells)
    qu = synth.uniform_u32_np(seed + 1, (n_cells,))
    _warm_oracle(lambda: O.answer(D, qu), 4.0)
    t0 = time.perf_counter()
    reps = 0
    while True:
        O.answer(D, qu)
        reps += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    gbs = reps * D.nbytes / dt / 1e9
    return {"value": round(gbs, 3), "unit": "GB/s", "cores": O.num_threads(), "kind": "oracle",
            "host": _host_cpu(),
            "sample": f"oracle answer over rows of the first {n_ch_s} channels "
                      f"({D.shape[0]} rows x {D.shape[1]} cells = {D.nbytes / 1e6:.1f} MB), "
                      f"{reps} repetitions in {dt:.1f} s"}


def cpu_baseline_gemm(wl, seed, kind, budget_s=10.0):
    """Oracle batch / hint on a bounded sample (a few rows of the same DB, all
    queries / hint columns), all host cores; the full-size time is reported as an
    explicit extrapolation from the measured rate."""
    import synth
    from oracle import oracle as O
    O.set_num_threads(os.cpu_count() or 1)
    n_cells, n_ch, d = wl["n_cells"], wl["n_ch"], wl["d"]
    rows = 8
    cells = torch.arange(n_cells, dtype=torch.int64)
    Dr = np.stack([synth.byte_column(seed, cells * n_ch + (r // d), r % d, d, n_ch).numpy()
                   for r in range(rows)])
    if kind == "batch":
        B = wl["B"]
        R = synth.uniform_u32_np(seed + 5, (B, n_cells))
        fn = (lambda: O.ftr_respond_batch(np.ascontiguousarray(Dr.T), R, wl["modp"])) \
            if wl.get("modp") else (lambda: O.answer_batch(Dr, R))
        macs = rows * n_cells * B
        full = wl.get("ell_total", n_ch * d) * n_cells * B
    else:
        A = O.expand_A(0x5EED, n_cells, wl["n"])
        fn = lambda: O.hint(Dr, A)
        macs = rows * n_cells * wl["n"]
        full = (n_ch * d // wl.get("shard_of", 1)) * n_cells * wl["n"]
    _warm_oracle(fn, 2.0)
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < budget_s:
        fn()
        reps += 1
    dt = (time.perf_counter() - t0) / reps
    rate = macs / dt
    return {"value": round(rate / 1e9, 3), "unit": "G u32-MAC/s", "cores": O.num_threads(),
            "kind": "oracle", "host": _host_cpu(),
            "sample": f"{rows} rows of the same DB x all {n_cells} cells x all "
                      f"{'queries' if kind == 'batch' else 'hint columns'}, {reps} repetitions",
            "extrapolated_full_step_s": round(full / rate, 1)}


def cpu_baseline_ens(wl, seed, kind, B=1, n_chunks=4, budget_s=8.0):
    """Oracle ENS answer / batch or OOP online answer on a bounded sample: the first
    32768 records (100.7 MB) of the same DB, all host cores, in the line's unit."""
    import synth
    from oracle import oracle as O
    O.set_num_threads(os.cpu_count() or 1)
    d, n_ch = wl["d"], wl["n_ch"]
    rs = 32768
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    rec = synth.records(seed, 0, rs, d, n_ch, device=dev).cpu().numpy()
    nbs = rs // 8
    if kind == "oop":
        k = rs // n_chunks
        q = synth.uniform_u8_np(seed + 3, (k // 8,))
        A = O.oop_preprocess(rec, n_chunks, 0, 7919)
        fn = lambda: O.oop_respond(rec, n_chunks, 0, q, A)  # noqa: E731
        per_call = rs * d  # whole-DB equivalent, as the line
    elif B == 1:
        q = synth.uniform_u8_np(seed + 7, (nbs,))
        fn = lambda: O.ens_respond(rec, q)  # noqa: E731
        per_call = rs * d
    else:
        Q = synth.uniform_u8_np(seed + 7, (B, nbs))
        fn = lambda: O.ens_respond_batch(rec, Q)  # noqa: E731
        per_call = B * rs * d  # query-equivalent, as the line
    _warm_oracle(fn, 2.0)
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < budget_s:
        fn()
        reps += 1
    dt = time.perf_counter() - t0
    what = ("OOP online answer (n = 4)" if kind == "oop" else
            "ENS answer" if B == 1 else f"ENS batch of {B} shares")
    return {"value": round(reps * per_call / dt / 1e9, 3),
            "unit": "GB/s" + ("" if B == 1 else " (query-equivalent)"),
            "cores": O.num_threads(), "kind": "oracle", "host": _host_cpu(),
            "sample": f"oracle {what} over the first {rs} records ({rs * d / 1e6:.1f} MB) of "
                      f"the same DB, {reps} repetitions in {dt:.1f} s"}


# ---------------------------------------------------------------- reference arm
def run_reference(args, wl, world, rank):
    if rank != 0:
        return
    import synth  # noqa: F401
    from oracle import oracle as O
    O.set_num_threads(os.cpu_count() or 1)  # torchrun defaults OMP_NUM_THREADS to 1
    cb = None
    # each step = oracle answer over a bounded sample (first 4 channels)
    n_cells, d = wl["n_cells"], wl["d"]
    n_ch_s = min(4, wl["n_ch"])
    import synth as S
    theta = (torch.arange(n_cells).unsqueeze(1) * wl["n_ch"] + torch.arange(n_ch_s)).reshape(-1)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    rec = S.records_at(args.seed, theta.to(dev), d, wl["n_ch"], 512).cpu().numpy()
    D = O.pack(rec, n_cells, n_ch_s, d, n_cells)
    qu = S.uniform_u32_np(args.seed + 1, (n_cells,))
    for _ in range(args.warmup):
        O.answer(D, qu)
    _warm_oracle(lambda: O.answer(D, qu), 4.0)  # extra untimed warm-up (see _warm_oracle)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.answer(D, qu)
    dt = time.perf_counter() - t0
    gbs = args.steps * D.nbytes / dt / 1e9
    sample = (f"oracle answer over rows of the first {n_ch_s} channels ({D.shape[0]} rows x "
              f"{D.shape[1]} cells = {D.nbytes / 1e6:.1f} MB) per step")
    cb = {"value": round(gbs, 3), "unit": "GB/s", "cores": O.num_threads(), "kind": "oracle",
          "host": _host_cpu(),
          "sample": sample}
    line = {"impl": "reference", "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt / args.steps * 1e3, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8xu32->u32 (mod 2^32)",
            "data": "synthetic", "config": {"workload": wl["name"], "sample": sample},
            "cpu_baseline": cb,
            "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _pipelined_e2e(call, stream, dev, out_bytes, n):
    """Device-timed e2e loop: call(b, dev_out) enqueues one answer from a pinned
    host input into device buffer b; its bytes are copied back to pinned host on
    a side stream while the next answer runs.  Returns ms per step."""
    copy = torch.cuda.Stream(dev)
    d_outs = [torch.empty(out_bytes, dtype=torch.uint8, device=dev) for _ in range(2)]
    h_outs = [torch.empty(out_bytes, dtype=torch.uint8).pin_memory() for _ in range(2)]
    k_ev = [torch.cuda.Event() for _ in range(2)]
    c_ev = [torch.cuda.Event() for _ in range(2)]
    used = [False, False]

    def one(i):
        b = i % 2
        if used[b]:
            stream.wait_event(c_ev[b])
        call(b, d_outs[b])
        k_ev[b].record(stream)
        copy.wait_event(k_ev[b])
        with torch.cuda.stream(copy):
            h_outs[b].copy_(d_outs[b], non_blocking=True)
            c_ev[b].record(copy)
        used[b] = True

    for i in range(3):
        one(i)
    torch.cuda.synchronize(dev)
    a0 = torch.cuda.Event(enable_timing=True)
    a1 = torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for i in range(n):
        one(i)
    stream.wait_stream(copy)
    a1.record(stream)
    torch.cuda.synchronize(dev)
    return a0.elapsed_time(a1) / n


# ---------------------------------------------------------------- ENS (NEXT-1)
def run_ens(args, wl, world, rank, local):
    """QPADL-ENS single / multi-request scan.  Every rank runs an independent
    replica (no data-path collective; weak scaling)."""
    import synth
    import paper_2510_03631_b200 as P
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    n_cells, n_ch, d = wl["n_cells"], wl["n_ch"], wl["d"]
    r = n_cells * n_ch
    t0 = time.time()
    srv = P.EnsServer(r, d, device=local, stable_inputs=True)
    chunk = max(1, (256 << 20) // d)
    for a in range(0, r, chunk):
        srv.db_write(a, synth.records(args.seed, a, min(chunk, r - a), d, n_ch, device=dev))
    torch.cuda.synchronize(dev)
    setup_s = time.time() - t0
    nb = (r + 7) // 8
    B = wl.get("B", 1)
    shares = [(synth.uniform_u32(args.seed + 7 + i, ((B * nb + 3) // 4,), device=dev)
               .view(torch.uint8)[: B * nb].reshape(B, nb).contiguous()) for i in range(4)]
    out = torch.empty((B, d), dtype=torch.uint8, device=dev)

    def step(i):
        if B == 1:
            srv.answer(shares[i % 4][0], out=out[0], stream=stream)
        else:
            srv.answer_batch(shares[i % 4], out=out, stream=stream)

    sampler = ClockSampler(physical_gpu(local))
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    time.sleep(0.3)
    l0 = srv.kernel_launches
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    sampler.start()
    e0.record(stream)
    for i in range(args.steps):
        step(i)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    launches = srv.kernel_launches - l0
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = tt.item()
    # e2e: share from pinned host, response back to pinned host, every step.
    # One share: the library stages the host share on its copy stream; the
    # response D2H runs on a side stream (double-buffered), device-timed.
    # Batches: synchronous calls with host in/out, host wall clock.
    h_in = torch.empty((B, nb), dtype=torch.uint8).pin_memory()
    h_in.copy_(shares[0].cpu())
    h_out = torch.empty((B, d), dtype=torch.uint8).pin_memory()
    n_e2e = max(3, min(args.steps, 200 if B == 1 else 100))
    if B == 1:
        h_ins = [h_in[0], torch.empty(nb, dtype=torch.uint8).pin_memory()]
        h_ins[1].copy_(shares[1][0].cpu())
        te = _pipelined_e2e(lambda b, o: srv.answer(h_ins[b], out=o, stream=stream),
                            stream, dev, d, n_e2e)
        e2e_timing = "device events; H2D on the library's copy stream, D2H on a side stream"
    else:
        h_ins = [h_in, torch.empty((B, nb), dtype=torch.uint8).pin_memory()]
        h_ins[1].copy_(shares[1].cpu())
        te = _pipelined_e2e(lambda b, o: srv.answer_batch(h_ins[b], out=o.view(B, d),
                                                          stream=stream),
                            stream, dev, B * d, n_e2e)
        e2e_timing = "device events; H2D on the library's copy stream, D2H on a side stream"
    if rank != 0:
        return
    hbm, _, _, peak_src = peaks()
    db = r * d
    value = world * db * B / (ms / 1e3) / 1e9
    nnz_frac = float(np.unpackbits(shares[0].cpu().numpy().reshape(-1)[: nb]).mean())
    touched = nnz_frac * db  # rows actually read (Alg. 3 step 9 skips unselected rows)
    achieved = (touched + nb + d) / (ms / 1e3) / 1e9 if B == 1 else None
    tc_used = B > 1 and srv.last_path == "tensor"  # the library reports the path it took
    if tc_used:
        # Work of the method: B x r x 8d GF(2) bit-products; on tcgen05 each
        # is one u8 x u8 MAC of the weighted bit-row operand (ens_mma.cuh), so the
        # tensor roof counts 2 ops per bit-product at the int8 peak; the HBM roof
        # counts the method's bytes (records once + shares + responses, Alg. 3).
        t_peak = 2.0 * peaks()[1]  # int8 dense = 2 x the measured bf16 (nominal ratio)
        ops = 2.0 * B * r * 8 * d
        meth_bytes = db + B * nb + B * d
        t_tensor = ops / (t_peak * 1e12) * 1e3
        t_hbm = meth_bytes / (hbm * 1e9) * 1e3
        ach_t = ops / (ms / 1e3) / 1e12
        ach_h = meth_bytes / (ms / 1e3) / 1e9
        if t_tensor >= t_hbm:
            roof_tc = {"bound": "tensor", "achieved": round(ach_t, 1), "peak": round(t_peak, 1),
                       "unit": "TOPS", "frac": round(ach_t / t_peak, 4),
                       "hbm_frac": round(ach_h / hbm, 4)}
        else:
            roof_tc = {"bound": "hbm", "achieved": round(ach_h, 1), "peak": hbm, "unit": "GB/s",
                       "frac": round(ach_h / hbm, 4), "tensor_frac": round(ach_t / t_peak, 4)}
        roof_tc.update({"traffic": _traffic(args.workload),
                        "kernel": "ens_share_pack_kernel + qpir_ens_mma_ts_kernel (shares in TMEM)",
                        "kernel_ms": round(ms, 5),
                        "peak_source": f"{peak_src} (int8 = 2 x bf16 burst)",
                        "algorithmic_bytes_per_launch": meth_bytes,
                        "algorithmic_ops_per_launch": ops,
                        "note": "GF(2) product on tcgen05 kind::i8: records read once in "
                                "place, expanded on chip to bit-rows weighted 2^i"})
    roof = (roof_tc if tc_used else
            {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
             "frac": round(achieved / hbm, 4), "traffic": _traffic(args.workload),
             "kernel": "ens_scan_wide_kernel",
             "kernel_ms": round(ms, 5), "peak_source": f"{peak_src} hbm_gbs",
             "algorithmic_bytes_per_launch": touched + nb + d,
             "note": "selected rows only (nnz(q) * d), P:968; back-to-back answers overlap "
                     "through programmatic dependent launch (one kernel alone under ncu: "
                     "profiles/r01_ens_scan_pdl_ncu_full.md)"} if B == 1 else
            {"bound": "alu", "achieved": round(B * r * d / 4 / (ms / 1e3) / 1e12, 3),
             "unit": "T word-XOR/s", "peak": round(148 * 64 * 1.965e9 / 1e12, 2),
             "frac": round(B * r * d / 4 / (ms / 1e3) / (148 * 64 * 1.965e9), 4),
             "traffic": None, "kernel": "ens_transpose_bits_kernel + ens_batch_kernel",
             "kernel_ms": round(ms, 5),
             "peak_source": "148 SMs x 64 LOP3 lanes/clk x 1965 MHz (guide unit counts)"})
    line = {"metric": METRIC, "value": round(value, 2),
            "unit": "GB/s" if B == 1 else "GB/s (query-equivalent)", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8 (GF(2) XOR)", "data": "synthetic",
            "config": {"workload": wl["name"], "n_records": r, "rec_bytes": d,
                       "queries_per_step": B, "selected_row_fraction": round(nnz_frac, 4),
                       "setup_s": round(setup_s, 1),
                       "l2": "inputs larger than L2 (1.007 GB records)"},
            "queries_per_s": round(world * B / (ms / 1e3), 1), "roofline": roof,
            "cpu_baseline": (cpu_baseline_ens(wl, args.seed, "ens", B)
                             if world == 1 and not args.no_cpu_baseline else None),
            "e2e": {"value": round(world * db * B / (te / 1e3) / 1e9, 2), "unit": "GB/s",
                    "h2d_bytes_per_step": B * nb, "d2h_bytes_per_step": B * d,
                    "ms_per_step": round(te, 4), "timing": e2e_timing},
            "gpu_launches": launches, "clocks": sampler.summary()}
    print(json.dumps(line), flush=True)


def _max_over_ranks(ms, world, dev):
    if world <= 1:
        return ms
    t = torch.tensor([ms], device=dev if torch.distributed.get_backend() == "nccl" else "cpu",
                     dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return t.item()


def run_oop(args, wl, rank, local, world=1):
    """QPADL-OOP: online answer (1/n of the DB) timed per step; the offline
    preprocessing of a 128-entry (S, A) queue timed once and reported beside it."""
    import synth
    import paper_2510_03631_b200 as P
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    n_cells, n_ch, d, n = wl["n_cells"], wl["n_ch"], wl["d"], wl["n_chunks"]
    r = n_cells * n_ch
    srv = P.EnsServer(r, d, device=local, stable_inputs=True)
    chunk = max(1, (256 << 20) // d)
    for a in range(0, r, chunk):
        srv.db_write(a, synth.records(args.seed, a, min(chunk, r - a), d, n_ch, device=dev))
    k = r // n
    kb = (k + 7) // 8
    seeds = torch.arange(1, 129, dtype=torch.int64, device=dev) * 7919
    # offline queue (timed once, after a warm-up call of the same size and path)
    srv.oop_preprocess(n, 0, seeds, stream=stream)
    o0 = torch.cuda.Event(enable_timing=True)
    o1 = torch.cuda.Event(enable_timing=True)
    o0.record(stream)
    A = srv.oop_preprocess(n, 0, seeds, stream=stream)
    o1.record(stream)
    torch.cuda.synchronize(dev)
    off_ms = o0.elapsed_time(o1)
    qs = [synth.uniform_u32(args.seed + 3 + i, ((kb + 3) // 4,), device=dev).view(torch.uint8)[:kb]
          .contiguous() for i in range(4)]
    out = torch.empty(d, dtype=torch.uint8, device=dev)
    sampler = ClockSampler(physical_gpu(local))
    for i in range(args.warmup):
        srv.oop_answer(n, 0, qs[i % 4], A[i % 128], out=out, stream=stream)
    torch.cuda.synchronize(dev)
    time.sleep(0.3)
    l0 = srv.kernel_launches
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    sampler.start()
    e0.record(stream)
    for i in range(args.steps):
        srv.oop_answer(n, 0, qs[i % 4], A[i % 128], out=out, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    sampler.stop()
    launches_oop = srv.kernel_launches - l0
    ms = _max_over_ranks(e0.elapsed_time(e1) / args.steps, world, dev)
    # e2e: the online query q_i and the precomputed A_i from pinned host, R_i
    # back to pinned host, every step (A_i lives with the client-facing server
    # state; staging it from host is the pessimistic case)
    h_q = [torch.empty(kb, dtype=torch.uint8).pin_memory() for _ in range(2)]
    h_A = [torch.empty(d, dtype=torch.uint8).pin_memory() for _ in range(2)]
    for b in range(2):
        h_q[b].copy_(qs[b].cpu())
        h_A[b].copy_(A[b].cpu())
    n_e2e = max(3, min(args.steps, 200))
    te = _pipelined_e2e(lambda b, o: srv.oop_answer(n, 0, h_q[b], h_A[b], out=o, stream=stream),
                        stream, dev, d, n_e2e)
    if rank != 0:
        return
    hbm, _, _, peak_src = peaks()
    touched = 0.5 * k * d
    achieved = (touched + kb + 2 * d) / (ms / 1e3) / 1e9
    line = {"metric": METRIC, "value": round(world * r * d / (ms / 1e3) / 1e9, 2),
            "unit": "GB/s (whole-DB equivalent: the online step reads 1/n of it)", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8 (GF(2) XOR)", "data": "synthetic",
            "config": {"workload": wl["name"], "n_records": r, "rec_bytes": d, "n_chunks": n,
                       "offline_queue": 128, "offline_ms_for_128": round(off_ms, 3),
                       "offline_ms_per_pair": round(off_ms / 128, 4),
                       "offline_gbs_db_equivalent": round(128 * (n - 1) / n * r * d / (off_ms / 1e3) / 1e9, 1),
                       "offline_path": srv.last_path},
            "queries_per_s": round(1e3 / ms, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(achieved / hbm, 4), "traffic": _traffic(args.workload),
                         "kernel": "ens_scan_wide_kernel (flip chunk)", "kernel_ms": round(ms, 5),
                         "peak_source": f"{peak_src} hbm_gbs",
                         "note": "back-to-back online answers overlap through programmatic "
                                 "dependent launch (one kernel alone under ncu: "
                                 "profiles/r01_oop_scan_ncu_full.md)"},
            "cpu_baseline": (cpu_baseline_ens(wl, args.seed, "oop", n_chunks=n)
                             if not args.no_cpu_baseline else None),
            "e2e": {"value": round(r * d / (te / 1e3) / 1e9, 2), "unit": "GB/s",
                    "h2d_bytes_per_step": kb + d, "d2h_bytes_per_step": d,
                    "ms_per_step": round(te, 4),
                    "timing": "device events; H2D on the library's copy stream, D2H on a "
                              "side stream"},
            "gpu_launches": launches_oop, "clocks": sampler.summary()}
    print(json.dumps(line), flush=True)


def run_bind(args, wl, rank, local, world=1):
    """NEXT-4: one step = Puzzle.Bind of every record of the DB on the GPU (HCT
    puzzle generation fused into the pack into the D panels), the spectrum data
    resident in HBM.  Replicas only (every rank binds its own copy)."""
    import synth
    import paper_2510_03631_b200 as P
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    n_cells, n_ch, d = wl["n_cells"], wl["n_ch"], wl["d"]
    r = n_cells * n_ch
    spec = synth.uniform_u32(args.seed, (r, 140), device=dev).view(torch.uint8).contiguous()  # 560 B rows
    srv = P.PirServer(n_cells, n_ch, d, lwe_n=4, device=local)
    seed_psd = 0x5D5EED
    xi = bytes(range(32)) if wl.get("sign") else None  # the PSD's ML-DSA-44 key seed
    for _ in range(args.warmup):
        srv.puzzle_bind_hct(0, spec, seed_psd, 20, 3, mldsa_seed=xi, stream=stream)
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(physical_gpu(local))
    l0 = srv.kernel_launches
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    sampler.start()
    e0.record(stream)
    for _ in range(args.steps):
        srv.puzzle_bind_hct(0, spec, seed_psd, 20, 3, mldsa_seed=xi, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    sampler.stop()
    launches = srv.kernel_launches - l0
    ms = _max_over_ranks(e0.elapsed_time(e1) / args.steps, world, dev)
    # e2e: the spectrum from pinned host memory every step (staged by the library)
    h_spec = spec.cpu().pin_memory()
    n_e2e = max(3, min(args.steps, 20))
    srv.puzzle_bind_hct(0, h_spec, seed_psd, 20, 3, mldsa_seed=xi, stream=stream)
    torch.cuda.synchronize(dev)
    a0 = torch.cuda.Event(enable_timing=True)
    a1 = torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for _ in range(n_e2e):
        srv.puzzle_bind_hct(0, h_spec, seed_psd, 20, 3, mldsa_seed=xi, stream=stream)
    a1.record(stream)
    torch.cuda.synchronize(dev)
    te = a0.elapsed_time(a1) / n_e2e
    srv.close()
    if rank != 0:
        return
    hbm, _, _, peak_src = peaks()
    db = r * d
    alg = r * 560 + db  # spectrum read + D written (the bound records)
    achieved = alg / (ms / 1e3) / 1e9
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import oracle as O
        O.set_num_threads(os.cpu_count() or 1)
        ns = (200 if not xi else 2) * n_ch  # records (whole cells), oracle bind (+ sign) + pack
        sp = spec[:ns].cpu().numpy()
        if xi:
            fn = lambda: O.pack(O.puzzle_bind_hct_signed(sp, 0, seed_psd, 20, 3, d, xi),  # noqa: E731
                                ns // n_ch, n_ch, d, ns // n_ch)
        else:
            fn = lambda: O.pack(O.puzzle_bind_hct(sp, 0, seed_psd, 20, 3, d), ns // n_ch, n_ch, d,  # noqa: E731
                                ns // n_ch)
        _warm_oracle(fn, 1.0)
        t0 = time.perf_counter()
        reps = 0
        while time.perf_counter() - t0 < 8.0:
            fn()
            reps += 1
        el = time.perf_counter() - t0
        cpu = {"value": round(reps * ns * d / el / 1e9, 6), "unit": "GB/s", "cores": 1 if xi else os.cpu_count(),
               "kind": "oracle", "sample": f"{ns} records ({ns * d / 1e6:.2f} MB), oracle "
                                           f"{'puzzle_bind_hct_signed (Python ML-DSA-44)' if xi else 'qo_puzzle_bind_hct'}"
                                           f" + qo_pack, {reps} repetitions",
               "records_per_s": round(reps * ns / el, 2)}
    roof_sig = None
    if xi:
        # ALU bound of the signing: Keccak-f[1600] work per ML-DSA-44
        # signature ~ 125 permutations (4.25 expected rejection-loop iterations x
        # (4 x 5 mask + 7 challenge + 2 SampleInBall) + mu, rho'') x ~7200 32-bit
        # lane-instructions, against 148 SMs x 128 INT lanes x the sampled SM clock
        sm = (sampler.summary() or {}).get("sm_mhz") or 1965.0
        sig_s = r / (ms / 1e3)
        peak_sig = 148 * 128 * sm * 1e6 / (125 * 7200)
        roof_sig = {"bound": "alu", "achieved": round(sig_s, 1), "peak": round(peak_sig, 1),
                    "unit": "signatures/s", "frac": round(sig_s / peak_sig, 5), "traffic": None,
                    "kernel": "mldsa_sign_kernel (+ pack_bind_tile_kernel)", "kernel_ms": round(ms, 5),
                    "peak_source": "Keccak-f[1600] issue bound: 148 SMs x 128 lanes x SM clock / "
                                   "(125 permutations x 7200 lane-instructions per signature)"}
    line = {"metric": METRIC, "value": round(world * db / (ms / 1e3) / 1e9, 2),
            "unit": "GB/s (bound DB bytes built per second)", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": wl["name"], "n_records": r, "rec_bytes": d,
                       "records_per_s": round(r / (ms / 1e3), 1),
                       "signature": ("ML-DSA-44 (FIPS 204, deterministic variant) of every puzzle, "
                                     "signed on the GPU" if xi else "none (zero slot)"),
                       "paper_context": "Table 1 (P:1448): PSD-HCT Puzzle.Bind on GPU 346 ms for 2^12 "
                                        "records, 21825 ms for 2^18 (RTX 3060 + CPU signing)"},
            "roofline": (roof_sig if xi else
                         {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                          "frac": round(achieved / hbm, 4), "traffic": _traffic(args.workload),
                          "kernel": "pack_bind_tile_kernel", "kernel_ms": round(ms, 5),
                          "algorithmic_bytes_per_launch": alg, "peak_source": f"{peak_src} hbm_gbs"}),
            "cpu_baseline": cpu,
            "e2e": {"value": round(db / (te / 1e3) / 1e9, 2), "unit": "GB/s",
                    "h2d_bytes_per_step": r * 560, "d2h_bytes_per_step": 0, "ms_per_step": round(te, 4),
                    "timing": "device events; pinned host spectrum staged by the library each step"},
            "gpu_launches": launches, "clocks": sampler.summary()}
    print(json.dumps(line), flush=True)


# The default run (c2) also measures the other hot-path rows in child processes on
# the same GPU, after its own timed region, and attaches a compact summary of each
# line ("secondary"), so every row has numbers from the driver's own run; the
# headline fields above are the c2 measurement alone.
SECONDARY = [("c4-64", []), ("c4-256", []), ("c5", []), ("ens-c2", []), ("ens-c2-b128", []),
             ("ftr-c2-b128", []), ("oop-c2", []), ("bind-c2", ["--steps", "8"])]


def _secondary_workloads():
    out = []
    for w, extra in SECONDARY:
        cmd = [sys.executable, os.path.abspath(__file__), "--workload", w, "--no-cpu-baseline",
               "--no-e2e", *extra]
        try:
            p = subprocess.run(cmd, capture_output=True, text=True, timeout=240)
            d = json.loads(p.stdout.strip().splitlines()[-1])
            r = d.get("roofline") or {}
            c = d.get("clocks") or {}
            out.append({"workload": w, "value": d.get("value"), "unit": d.get("unit"),
                        "ms_per_step": d.get("ms_per_step"), "steps": d.get("steps"),
                        "queries_per_s": d.get("queries_per_s"), "bound": r.get("bound"),
                        "frac": r.get("frac"), "gpu_launches": d.get("gpu_launches"),
                        "sm_mhz": c.get("sm_mhz"), "reasons": c.get("reasons")})
        except Exception as e:  # a failed child is reported, never hidden
            out.append({"workload": w, "error": f"{type(e).__name__}: {str(e)[:200]}"})
    return out


def _traffic(workload):
    """DRAM bytes per launch of the dominant kernel from a committed ncu --set full
    summary (profiles/traffic_<workload>.json), else None."""
    prof = os.path.join(ROOT, "profiles", f"traffic_{workload}.json")
    try:
        return json.load(open(prof)).get("dram_bytes_per_launch")
    except Exception:
        return None


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=2025)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="default run only: skip the summaries of the other workloads")
    ap.add_argument("--graph", type=int, default=None,
                    help="1: capture the K timed steps into one CUDA graph and replay it "
                         "(N = 1; default on for the launch-bound c1 workload only)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo + --device-override: functional multi-rank test on one GPU")
    ap.add_argument("--device-override", type=int, default=None,
                    help="put every rank on this CUDA device (functional tests only)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without a launcher: re-run under torchrun,
        # one rank per GPU, rendezvous on 127.0.0.1
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                                  "--master-port", str(port), os.path.abspath(__file__)]
                 + sys.argv[1:])
    wl = dict(WORKLOADS[args.workload])
    world, rank, local = dist_env()
    if args.impl == "reference":
        args.steps = args.steps or 20
        args.warmup = args.warmup if args.warmup is not None else 3
        return run_reference(args, wl, world, rank)

    if wl["kind"] in ("bind", "oop"):
        # independent replicas per rank (no data-path collective): the process
        # group only takes the max of the per-rank device times
        if wl["kind"] == "bind":
            args.steps = args.steps or 50
            args.warmup = max(3, args.warmup if args.warmup is not None else 3)
        else:
            args.steps = args.steps or 1000
            args.warmup = max(3, args.warmup if args.warmup is not None else 5)
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group(args.backend)
        fn = run_bind if wl["kind"] == "bind" else run_oop
        return fn(args, wl, rank, local if args.device_override is None else args.device_override,
                  world)
    if wl["kind"] in ("ens", "ens_batch"):
        args.steps = args.steps or (1000 if wl["kind"] == "ens" else 50)
        args.warmup = max(3, args.warmup if args.warmup is not None else 5)
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group(args.backend)
        return run_ens(args, wl, world, rank,
                       local if args.device_override is None else args.device_override)
    default_steps = {"answer": 2000, "batch": 300, "hint": 40}[wl["kind"]]
    if args.workload == "c3":
        default_steps = 200
    args.steps = args.steps or default_steps
    args.warmup = max(3, args.warmup if args.warmup is not None else 10)

    if args.device_override is not None:
        local = args.device_override
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    import paper_2510_03631_b200 as P
    from paper_2510_03631_b200.dist import gather_answer, shard_rows

    hbm, bf16, bf16_sus, peak_src = peaks()
    n_cells, d = wl["n_cells"], wl["d"]
    kind = wl["kind"]
    # geometry per rank
    if args.workload in ("c1", "c2", "c4-64", "c4-256") and world > 1:
        n_ch_total = wl["n_ch"] * world  # weak scaling: 40-channel slice per rank
        scaling = "weak"
    else:
        n_ch_total = wl["n_ch"]
        scaling = "weak" if world == 1 else "strong"
    if kind == "hint":
        shard_world = wl.get("shard_of", 1)
        r0, r1 = shard_rows(n_cells, n_ch_total, d, n_cells, shard_world, rank % shard_world)
        scaling = "weak"
    else:
        r0, r1 = shard_rows(n_cells, n_ch_total, d, n_cells, world, rank)
    sizes = [b - a for a, b in (shard_rows(n_cells, n_ch_total, d, n_cells, world, r)
                                for r in range(world))] if kind != "hint" else None

    t_setup = time.time()
    srv = build_db(P, wl, n_ch_total, r0, r1, args.seed, local, lwe_n=wl.get("n", 1024))
    setup_s = time.time() - t_setup
    ell_local = srv.ell_local
    db_bytes_local = ell_local * n_cells
    import synth
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    B = wl.get("B", 1)
    if kind == "answer":
        qs = [synth.uniform_u32(args.seed + 100 + i, (n_cells,), device=dev) for i in range(16)]
        out = torch.empty(ell_local, dtype=torch.int32, device=dev)
    elif kind == "batch":
        qs = [synth.uniform_u32(args.seed + 100 + i, (B, n_cells), device=dev) for i in range(2)]
        out = torch.empty((B, ell_local), dtype=torch.int32, device=dev)
    else:
        qs = [None]
        out = torch.empty((ell_local, wl["n"]), dtype=torch.int32, device=dev)

    # N > 1: the NCCL gather of query i runs on a side stream, overlapped with the
    # scan of query i + 1 (double-buffered answer slices); device-side ordering
    # only, no host syncs inside the timed region.
    pipelined = world > 1 and kind != "hint"
    comm = torch.cuda.Stream(dev) if pipelined else None
    outs = [out, torch.empty_like(out)] if pipelined else [out]
    kdone = [torch.cuda.Event() for _ in outs]
    gdone = [torch.cuda.Event() for _ in outs]
    used = [False for _ in outs]

    def step(i, evs=None):
        b = i % len(outs)
        if pipelined and used[b]:
            stream.wait_event(gdone[b])  # slice b's previous gather has read it
        if evs is not None:
            evs[0].record(stream)
        if kind == "answer":
            srv.answer(qs[i % len(qs)], out=outs[b], stream=stream)
        elif kind == "batch" and wl.get("modp"):
            srv.answer_batch_modp(qs[i % len(qs)], wl["modp"], out=outs[b], stream=stream)
        elif kind == "batch":
            srv.answer_batch(qs[i % len(qs)], out=outs[b], stream=stream)
        else:
            srv.hint(out=outs[b], stream=stream)
        if evs is not None:
            evs[1].record(stream)
        if pipelined:
            kdone[b].record(stream)
            comm.wait_event(kdone[b])
            with torch.cuda.stream(comm):
                gather_answer(outs[b], sizes)
                gdone[b].record(comm)
            used[b] = True

    def drain():
        if pipelined:
            stream.wait_stream(comm)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    # CUDA-graph mode (launch-bound configs): the K steps are captured once and
    # replayed as one graph, so the device time is not the host's call rate
    use_graph = (args.graph if args.graph is not None else args.workload == "c1") and world == 1
    if use_graph:
        stream = torch.cuda.Stream(dev)  # capture needs a non-default stream
    sampler = ClockSampler(physical_gpu(local))
    for i in range(args.warmup):
        step(i)
    drain()
    barrier()
    graph = None
    if use_graph:
        l0 = srv.kernel_launches
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream, capture_error_mode="relaxed"):
            for i in range(args.steps):
                step(i)
        launches = srv.kernel_launches - l0  # launches recorded into the graph
        with torch.cuda.stream(stream):
            graph.replay()  # untimed warm replay
        barrier()
    time.sleep(0.3)  # let the clock sampler come up
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l0 = srv.kernel_launches
    barrier()
    sampler.start()
    e0.record(stream)
    # per-step kernel events only when the step has a side-stream gather (N > 1):
    # an event record between two launches also cuts the programmatic dependent
    # launch overlap of back-to-back GEMVs, so at N = 1 the step time is the
    # kernel time
    per_step_events = world > 1
    if use_graph:
        with torch.cuda.stream(stream):
            graph.replay()
    else:
        for i in range(args.steps):
            step(i, kev[i] if per_step_events else None)
    drain()
    e1.record(stream)
    barrier()
    sampler.stop()
    t_ms = e0.elapsed_time(e1)
    if use_graph:
        k_ms = t_ms / args.steps  # the replay holds only the captured steps
    else:
        launches = srv.kernel_launches - l0
        k_ms = (sum(a.elapsed_time(b) for a, b in kev) / args.steps if per_step_events
                else t_ms / args.steps)  # N = 1: only our kernels are in the step
    if world > 1:
        tt = torch.tensor([t_ms, k_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_ms, k_ms = tt.tolist()
    ms_per_step = t_ms / args.steps

    # ---------------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e and kind in ("answer", "batch"):
        if kind == "answer":
            h_in = torch.empty(n_cells, dtype=torch.int32).pin_memory()
            h_in.copy_(qs[0].cpu())
            h_out = torch.empty(srv.ell if world > 1 else ell_local, dtype=torch.int32).pin_memory()
        else:
            h_in = torch.empty((B, n_cells), dtype=torch.int32).pin_memory()
            h_in.copy_(qs[0].cpu())
            h_out = torch.empty((B, srv.ell if world > 1 else ell_local), dtype=torch.int32).pin_memory()
        # as many steps as the device-timed loop (up to 200), so both run in the
        # same power / clock state (batches are power-capped in steady state)
        e2e_steps = max(3, min(args.steps, 200))
        dev_out = out
        two = world == 1  # answers and batches: D2H overlapped on a copy stream
        if two:
            # every step: pinned-host query (batch) -> H2D (inside the C call) ->
            # kernels on the compute stream (kept serialised) -> answer D2H to
            # pinned host on a copy stream, overlapping the next step's kernels
            copy_stream = torch.cuda.Stream(dev)
            h_ins = [h_in, torch.empty_like(h_in).pin_memory()]
            h_ins[1].copy_(qs[1].cpu())
            h_outs = [h_out, torch.empty_like(h_out).pin_memory()]
            d_outs = [dev_out, torch.empty_like(dev_out)]
            k_ev = [torch.cuda.Event(), torch.cuda.Event()]
            c_ev = [torch.cuda.Event(), torch.cuda.Event()]
            c_used = [False, False]

        def e2e_step(i=0):
            if two:
                b = i % 2
                if c_used[b]:
                    stream.wait_event(c_ev[b])  # slot's previous D2H has read it
                if kind == "answer":
                    srv.answer(h_ins[b], out=d_outs[b], stream=stream)
                elif wl.get("modp"):
                    srv.answer_batch_modp(h_ins[b], wl["modp"], out=d_outs[b], stream=stream)
                else:
                    srv.answer_batch(h_ins[b], out=d_outs[b], stream=stream)
                k_ev[b].record(stream)
                copy_stream.wait_event(k_ev[b])
                with torch.cuda.stream(copy_stream):
                    h_outs[b].copy_(d_outs[b], non_blocking=True)
                    c_ev[b].record(copy_stream)
                c_used[b] = True
                return
            if kind == "answer":
                srv.answer(h_in, out=dev_out, stream=stream)  # H2D of qu inside the C call
            elif wl.get("modp"):
                srv.answer_batch_modp(h_in, wl["modp"], out=dev_out, stream=stream)
            else:
                srv.answer_batch(h_in, out=dev_out, stream=stream)
            full = gather_answer(dev_out, sizes) if world > 1 else dev_out
            h_out.copy_(full, non_blocking=True)
            stream.synchronize()

        for i in range(3):
            e2e_step(i)
        torch.cuda.synchronize(dev)
        barrier()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for i in range(e2e_steps):
            e2e_step(i)
        if two:
            stream.wait_stream(copy_stream)
        a1.record(stream)
        barrier()
        te = a0.elapsed_time(a1)
        if world > 1:
            tt = torch.tensor([te], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te = tt.item()
        scanned = db_bytes_local * world * B
        e2e = {"value": round(scanned / (te / e2e_steps / 1e3) / 1e9, 2), "unit": "GB/s",
               "h2d_bytes_per_step": int(h_in.numel() * 4),
               "d2h_bytes_per_step": int(h_out.numel() * 4), "steps": e2e_steps,
               "ms_per_step": round(te / e2e_steps, 4),
               "path": ("D2H overlapped with the next kernel on a copy stream: "
                        if world == 1 else "")
                       + "qpir_answer with pinned host query (H2D inside the C call) "
                       + ("+ NCCL all-gather " if world > 1 else "") + "+ D2H of the answer "
                       "to pinned host, every step"}

    # ---------------------------------------------------------------- line
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    clocks = sampler.summary()
    if kind == "answer":
        scanned = db_bytes_local * world
        value = scanned / (ms_per_step / 1e3) / 1e9
        alg_bytes = db_bytes_local + 4 * n_cells + 4 * ell_local
        achieved = alg_bytes / (k_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": None,
                "kernel": "gemv_u8_u32_kernel", "kernel_ms": round(k_ms, 5),
                "peak_source": f"{peak_src} hbm_gbs (copy, read+write)",
                "algorithmic_bytes_per_launch": alg_bytes}
        qps = world / (ms_per_step / 1e3)
        unit = "GB/s"
    elif kind == "batch":
        scanned = db_bytes_local * world * B
        value = scanned / (ms_per_step / 1e3) / 1e9
        mp = wl.get("modp") or 0
        if mp and mp <= 65537 and os.environ.get("QPIR_MODP2", "1") != "0":
            limbs = 2
        elif mp and mp <= (1 << 24) and os.environ.get("QPIR_MODP3", "1") != "0":
            limbs = 3
        else:
            limbs = 4
        ops = 2.0 * ell_local * n_cells * limbs * B  # int8 tensor ops actually executed
        # the step is bound by whichever roof takes longer: streaming D (+ Q in,
        # ANS out) from HBM once, or the executed int8 MMAs
        alg_bytes = db_bytes_local + 4 * n_cells * B + 4 * ell_local * B
        pk = 2.0 * bf16
        t_hbm = alg_bytes / (hbm * 1e9)
        t_tc = ops / (pk * 1e12)
        achieved_tc = ops / (k_ms / 1e3) / 1e12
        achieved_hbm = alg_bytes / (k_ms / 1e3) / 1e9
        common = {"traffic": None,
                  "kernel": ("mma_u8_limb_kernel with the fused 2-limb split + modp_fixup_kernel "
                             "(step time, upper bound)" if limbs == 2 and os.environ.get("QPIR_FTR_FUSE", "1") != "0"
                             else "limb_split_kernel + mma_u8_limb_kernel (step time, upper bound)"),
                  "limbs_per_query": limbs, "kernel_ms": round(k_ms, 5),
                  "algorithmic_ops_per_launch": ops, "algorithmic_bytes_per_launch": alg_bytes,
                  "roof_ms": {"hbm": round(t_hbm * 1e3, 5), "tensor": round(t_tc * 1e3, 5)}}
        if t_hbm > t_tc:
            roof = {"bound": "hbm", "achieved": round(achieved_hbm, 1), "peak": hbm,
                    "unit": "GB/s", "frac": round(achieved_hbm / hbm, 4), **common,
                    "peak_source": f"{peak_src} hbm_gbs (copy, read+write)",
                    "tensor_frac": round(achieved_tc / pk, 4)}
        else:
            roof = {"bound": "tensor", "achieved": round(achieved_tc, 1), "peak": pk,
                    "unit": "TFLOP/s", "frac": round(achieved_tc / pk, 4), **common,
                    "peak_source": f"{peak_src} bf16_tflops x 2 (nominal int8/bf16 ratio), int8 TOPS",
                    "hbm_frac": round(achieved_hbm / hbm, 4)}
            if bf16_sus:
                roof["peak_sustained"] = 2.0 * bf16_sus
                roof["frac_sustained"] = round(achieved_tc / (2.0 * bf16_sus), 4)
        qps = B * world / (ms_per_step / 1e3)
        unit = "GB/s (query-equivalent)"
    else:
        ops = 2.0 * ell_local * n_cells * 4 * wl["n"]
        value = ops / (ms_per_step / 1e3) / 1e12
        achieved = value
        pk = 2.0 * bf16
        roof = {"bound": "tensor", "achieved": round(achieved, 1), "peak": pk, "unit": "TFLOP/s",
                "frac": round(achieved / pk, 4), "traffic": None,
                "kernel": "expand_A_limbs_kernel + mma_u8_limb_kernel (step time)",
                "kernel_ms": round(k_ms, 5),
                "peak_source": f"{peak_src} bf16_tflops x 2 (nominal int8/bf16 ratio), int8 TOPS"}
        if bf16_sus:
            roof["peak_sustained"] = 2.0 * bf16_sus
            roof["frac_sustained"] = round(achieved / (2.0 * bf16_sus), 4)
        qps = None
        unit = "TOPS (int8)"
    ctx_peaks = os.path.join(ROOT, "profiles", "r01_context_peaks.json")
    if os.path.exists(ctx_peaks) and roof.get("bound") in ("hbm", "tensor"):
        try:
            cp = json.load(open(ctx_peaks))
            if roof["bound"] == "hbm":
                roof["context_read_only_stream_gbs"] = cp.get("hbm_read_only_gbs")
            else:
                roof["context_cublaslt_int8_tops"] = {k: v for k, v in cp.items()
                                                      if k.startswith("int_mm") and k.endswith("tops")}
        except Exception:
            pass
    prof = os.path.join(ROOT, "profiles", f"traffic_{args.workload}.json")
    if os.path.exists(prof):
        try:
            roof["traffic"] = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            pass
    cpu_base = None
    if not args.no_cpu_baseline and world == 1 and kind == "answer":
        cpu_base = cpu_baseline_answer(wl, args.seed)
    elif not args.no_cpu_baseline and world == 1 and kind in ("batch", "hint"):
        cpu_base = cpu_baseline_gemm(wl, args.seed, kind)
    cfg = {"workload": wl["name"], "n_cells": n_cells, "n_ch": n_ch_total, "rec_bytes": d,
           "ell_local": ell_local, "db_bytes_per_gpu": db_bytes_local,
           "queries_per_step": B if kind != "hint" else 0,
           "l2": "inputs larger than L2: D slice per GPU >> 126 MB, no flush needed"
                 if db_bytes_local > 512e6 else "D slice fits in L2 (latency config)",
           "setup_s": round(setup_s, 1), "parallelism": f"row-shard x{world}",
           "backend": args.backend if world > 1 else None,
           "launch": "K steps replayed from one CUDA graph" if use_graph
                     else "eager C-ABI calls from Python"}
    line = {"metric": METRIC, "value": round(value, 2), "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "u8xu32->u32 (mod 2^32)", "data": "synthetic", "config": cfg,
            "queries_per_s": round(qps, 1) if qps else None,
            "roofline": roof, "cpu_baseline": cpu_base, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks}
    srv.close()
    if world == 1 and args.workload == "c2" and not args.no_secondary:
        line["secondary"] = _secondary_workloads()
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
