"""Probe: A/B the K-split count of the tcgen05 batch in one process (servers
created under different QPIR_MMA_SPLIT, timed alternately).
Usage: split_ab_probe.py SPLITS BATCHES [N_CELLS]  (8192 = C2, 65536 = C4)."""
import os
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_03631_b200 as P  # noqa: E402
import synth  # noqa: E402

n_ch, d = 40, 3072
splits = [int(x) for x in sys.argv[1].split(",")]
Bs = [int(x) for x in sys.argv[2].split(",")]
n_cells = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
srvs = []
for s in splits:
    os.environ["QPIR_MMA_SPLIT"] = str(s)
    v = P.PirServer(n_cells, n_ch, d, lwe_n=1024, device=0)
    for t0 in range(0, n_cells * n_ch, 16384):
        n = min(16384, n_cells * n_ch - t0)
        v.db_write(t0, synth.records(7, t0, n, d, n_ch, device="cuda:0"))
    srvs.append(v)
torch.cuda.synchronize()


def timeit(fn, k=40 if n_cells <= 8192 else 8):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3


for B in Bs:
    Q = synth.uniform_u32(2, (B, n_cells), device="cuda")
    O = torch.empty((B, srvs[0].ell_local), dtype=torch.int32, device="cuda")
    res = {s: [] for s in splits}
    for rep in range(4):
        for s, v in zip(splits, srvs):
            res[s].append(timeit(lambda: v.answer_batch(Q, out=O)))
    print(f"B={B}: " + "  ".join(f"split {s}: {min(r):.1f}/{sorted(r)[len(r)//2]:.1f} us"
                                  for s, r in res.items()), flush=True)
