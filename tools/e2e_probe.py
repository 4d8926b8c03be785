"""Probe: end-to-end C2 answer loop variants (pinned host query in, answer out)."""
import sys
import torch
import numpy as np
sys.path.insert(0, '.')
import paper_2510_03631_b200 as P
import synth

n_cells, n_ch, d = 8192, 40, 3072


def make(seed):
    s = P.PirServer(n_cells, n_ch, d, lwe_n=1024, device=0)
    chunk = 16384
    for t0 in range(0, n_cells * n_ch, chunk):
        n = min(chunk, n_cells * n_ch - t0)
        s.db_write(t0, synth.records(seed, t0, n, d, n_ch, device='cuda:0'))
    torch.cuda.synchronize()
    return s


srv = make(7)
srv2 = make(8)  # a second 1 GB DB: alternating them rules out L2 reuse across steps
L = srv.ell_local
K = 200
main = torch.cuda.Stream()
h2d = torch.cuda.Stream()
d2h = torch.cuda.Stream()
h_in = [torch.from_numpy(synth.uniform_u32_np(i, (n_cells,)).view(np.int32)).pin_memory() for i in range(2)]
h_out = [torch.empty(L, dtype=torch.int32).pin_memory() for _ in range(2)]
d_in = [torch.empty(n_cells, dtype=torch.int32, device='cuda') for _ in range(2)]
d_out = [torch.empty(L, dtype=torch.int32, device='cuda') for _ in range(2)]


def run(variant):
    in_ev = [torch.cuda.Event() for _ in range(2)]
    used_in = [torch.cuda.Event() for _ in range(2)]
    k_ev = [torch.cuda.Event() for _ in range(2)]
    c_ev = [torch.cuda.Event() for _ in range(2)]
    used = [False, False]

    def step(i):
        b = i % 2
        if variant == "lib_h2d":
            if used[b]:
                main.wait_event(c_ev[b])
            srv.answer(h_in[b], out=d_out[b], stream=main)
        elif variant in ("user_h2d", "user_h2d_nod2h"):
            if used[b]:
                h2d.wait_event(used_in[b])  # GEMV that read d_in[b] done
            with torch.cuda.stream(h2d):
                d_in[b].copy_(h_in[b], non_blocking=True)
                in_ev[b].record(h2d)
            main.wait_event(in_ev[b])
            if used[b] and variant == "user_h2d":
                main.wait_event(c_ev[b])
            srv.answer(d_in[b], out=d_out[b], stream=main)
            used_in[b].record(main)
        elif variant == "kernel_only":
            srv.answer(d_in[b], out=d_out[b], stream=main)
            used[b] = True
            return
        elif variant == "kernel_only_2db":
            (srv if b == 0 else srv2).answer(d_in[b], out=d_out[b], stream=main)
            used[b] = True
            return
        if variant != "user_h2d_nod2h":
            k_ev[b].record(main)
            d2h.wait_event(k_ev[b])
            with torch.cuda.stream(d2h):
                h_out[b].copy_(d_out[b], non_blocking=True)
                c_ev[b].record(d2h)
        used[b] = True

    for i in range(10):
        step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for i in range(K):
        step(i)
    main.wait_stream(d2h)
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    print(f"{variant:16s} {ms*1e3:7.1f} us/query  {L*n_cells/ms/1e6:7.0f} GB/s", flush=True)


for v in ["kernel_only", "kernel_only_2db", "lib_h2d", "user_h2d", "user_h2d_nod2h",
          "kernel_only", "kernel_only_2db"]:
    run(v)
