"""Probe: does the oracle baseline's speed depend on what the process did before
(fresh vs after the GPU bench)?"""
import os
import sys
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")
sys.path.insert(0, ".")
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2510_03631_b200 as P  # noqa: E402

wl = bench.WORKLOADS["c2"]
print("fresh", bench.cpu_baseline_answer(wl, 2025, 4.0)["value"], flush=True)
srv = bench.build_db(P, wl, wl["n_ch"], 0, 0, 2025, 0)
import synth  # noqa: E402
q = synth.uniform_u32(5, (wl["n_cells"],), device="cuda")
out = torch.empty(srv.ell_local, dtype=torch.int32, device="cuda")
print("after build_db", bench.cpu_baseline_answer(wl, 2025, 4.0)["value"], flush=True)
for _ in range(2000):
    srv.answer(q, out=out)
torch.cuda.synchronize()
print("after 2000 GEMVs", bench.cpu_baseline_answer(wl, 2025, 4.0)["value"], flush=True)
srv.close()
print("after close", bench.cpu_baseline_answer(wl, 2025, 4.0)["value"], flush=True)
