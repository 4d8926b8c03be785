"""Probe: oracle answer timing on the host under different process states
(plain numpy process vs after torch/CUDA init), to explain baseline spread."""
import os
import sys
import time
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")
sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import synth as S  # noqa: E402
from oracle import oracle as O  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "plain"
if mode in ("torch", "cuda"):
    import torch
    if mode == "cuda":
        torch.zeros(1, device="cuda")
        torch.cuda.synchronize()
O.set_num_threads(os.cpu_count())
n_cells, d, n_ch = 8192, 3072, 40
rec = S.records_np(2025, n_cells * 4, d, n_ch)
D = O.pack(rec, n_cells, 4, d, n_cells)
qu = S.uniform_u32_np(1, (n_cells,))
ts = []
for i in range(40):
    t0 = time.perf_counter()
    O.answer(D, qu)
    ts.append((time.perf_counter() - t0) * 1e3)
ts2 = []
for i in range(40):
    t0 = time.perf_counter()
    O.answer(D, qu)
    ts2.append((time.perf_counter() - t0) * 1e3)
    time.sleep(0.002)
print(mode, "threads", O.num_threads(), "median ms back-to-back %.2f, with 2 ms gaps %.2f"
      % (np.median(ts), np.median(ts2)), "GB/s %.1f" % (D.nbytes / np.median(ts) / 1e6))
