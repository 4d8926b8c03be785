"""Probe: hint (C5 shard shape) DRAM traffic vs the D/A' panel stride.
Usage: python tools/hint_stride_probe.py N_CELLS  (262144 = power-of-two panel stride)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_03631_b200 as P  # noqa: E402

n_cells = int(sys.argv[1])
srv = P.PirServer(n_cells, 40, 3072, lwe_n=1024, seed_A=7, row_begin=0, row_end=15360, device=0)
out = torch.empty((srv.ell_local, 1024), dtype=torch.int32, device="cuda")
for _ in range(2):
    srv.hint(out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    srv.hint(out=out)
e1.record()
torch.cuda.synchronize()
print(f"n_cells={n_cells} hint {e0.elapsed_time(e1) / 5:.2f} ms", flush=True)
