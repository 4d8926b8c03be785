import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2510_03631_b200 as P
for d, r in [(64, 1 << 23), (512, 1 << 20), (1024, 1 << 19), (3072, 327680)]:
    rec = torch.randint(0, 256, (r, d), dtype=torch.uint8, device='cuda')
    srv = P.EnsServer(r, d, records=rec)
    share = torch.randint(0, 256, ((r + 7) // 8,), dtype=torch.uint8, device='cuda')
    out = torch.empty(d, dtype=torch.uint8, device='cuda')
    for _ in range(5): srv.answer(share, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(200): srv.answer(share, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 200
    gb = r * d / 2 / 1e9
    print(f"d={d} r={r} {ms*1e3:.1f} us  {gb/ms*1e3:.0f} GB/s selected  frac={gb/ms*1e3/6454.3:.3f}", flush=True)
    srv.close(); del rec
