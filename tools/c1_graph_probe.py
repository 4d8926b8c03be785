"""Probe: C1 (tiny, launch-bound) answers eager vs captured in a CUDA graph."""
import sys, torch, numpy as np, time
sys.path.insert(0, '.')
import paper_2510_03631_b200 as P
import synth
n_cells, n_ch, d = 1024, 16, 8
rec = torch.from_numpy(synth.records_np(1, n_cells * n_ch, d, n_ch)).cuda()
srv = P.PirServer(n_cells, n_ch, d, lwe_n=256, device=0, records=rec)
qs = [torch.from_numpy(synth.uniform_u32_np(i, (n_cells,)).view(np.int32)).cuda() for i in range(4)]
out = torch.empty(srv.ell_local, dtype=torch.int32, device='cuda')
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for i in range(20): srv.answer(qs[i % 4], out=out, stream=st.cuda_stream)
st.synchronize()
K = 200
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for i in range(K): srv.answer(qs[i % 4], out=out, stream=st.cuda_stream)
e1.record(st); st.synchronize()
print("eager us/query", e0.elapsed_time(e1) / K * 1e3)
t0 = time.perf_counter()
for i in range(K): srv.answer(qs[i % 4], out=out, stream=st.cuda_stream)
st.synchronize()
print("host us/call", (time.perf_counter() - t0) / K * 1e6)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st, capture_error_mode="relaxed"):
    for i in range(K): srv.answer(qs[i % 4], out=out, stream=st.cuda_stream)
st.synchronize()
with torch.cuda.stream(st):
    g.replay()
    st.synchronize()
    e0.record(st); g.replay(); e1.record(st)
st.synchronize()
print("graph us/query", e0.elapsed_time(e1) / K * 1e3)
import oracle.oracle as O
D = O.pack(rec.cpu().numpy(), n_cells, n_ch, d, n_cells)
print("parity", (P.u32(out) == O.answer(D, qs[(K - 1) % 4].cpu().numpy().view(np.uint32))).all())
