"""Probe: C2 (1.007 GB) answers per second vs batch size -- single-query GEMV
(B = 1) against the tcgen05 batch path for B = 2..256 (D streamed once per batch)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_03631_b200 as P  # noqa: E402
import synth  # noqa: E402

n_cells, n_ch, d = 8192, 40, 3072
srv = P.PirServer(n_cells, n_ch, d, lwe_n=1024, device=0)
for t0 in range(0, n_cells * n_ch, 16384):
    n = min(16384, n_cells * n_ch - t0)
    srv.db_write(t0, synth.records(7, t0, n, d, n_ch, device="cuda:0"))
torch.cuda.synchronize()
db = srv.ell_local * n_cells


def timeit(fn, k):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


q = synth.uniform_u32(1, (n_cells,), device="cuda")
o = torch.empty(srv.ell_local, dtype=torch.int32, device="cuda")
ms = timeit(lambda: srv.answer(q, out=o), 200)
print(f"B=1 GEMV      {ms * 1e3:8.1f} us/batch  {1e3 / ms:9.0f} q/s  D at {db / ms / 1e6:6.0f} GB/s")
for B in (2, 4, 8, 16, 32, 64, 128, 256):
    Q = synth.uniform_u32(2, (B, n_cells), device="cuda")
    O = torch.empty((B, srv.ell_local), dtype=torch.int32, device="cuda")
    ms = timeit(lambda: srv.answer_batch(Q, out=O), 50)
    print(f"B={B:<4d} tcgen05 {ms * 1e3:8.1f} us/batch  {B * 1e3 / ms:9.0f} q/s  "
          f"D at {db / ms / 1e6:6.0f} GB/s", flush=True)
