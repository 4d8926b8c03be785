"""Probe: C2 GEMV per-query time vs query rotation / output reuse and nvidia-smi polling
(all within box-to-box noise: 0.136-0.157 ms)."""
import sys, subprocess, time
sys.path.insert(0, '.')
import torch, numpy as np
import paper_2510_03631_b200 as P
import synth
n_cells, n_ch, d = 8192, 40, 3072
srv = P.PirServer(n_cells, n_ch, d, lwe_n=1024, device=0)
for t0 in range(0, n_cells * n_ch, 16384):
    n = min(16384, n_cells * n_ch - t0)
    srv.db_write(t0, synth.records(7, t0, n, d, n_ch, device='cuda:0'))
torch.cuda.synchronize()
qs16 = [synth.uniform_u32(100 + i, (n_cells,), device='cuda') for i in range(16)]
outs = [torch.empty(srv.ell_local, dtype=torch.int32, device='cuda') for _ in range(2)]
st = torch.cuda.current_stream()
def run(nq, nout, K=2000):
    for i in range(10): srv.answer(qs16[i % nq], out=outs[i % nout], stream=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(K): srv.answer(qs16[i % nq], out=outs[i % nout], stream=st)
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3
for rep in range(2):
    print("q16 out1", round(run(16, 1), 1), "q2 out2", round(run(2, 2), 1), "q16 out2", round(run(16, 2), 1), "q2 out1", round(run(2, 1), 1))
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-i", "0", "-lms", "50"], stdout=subprocess.DEVNULL)
time.sleep(0.3)
print("with nvidia-smi 50ms polling: q16 out1", round(run(16, 1), 1))
p.terminate()
