"""Signed Puzzle.Bind of 16384 records (one mldsa_sign_kernel launch) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2510_03631_b200 as P
import synth

n_cells, n_ch, d = 8192, 2, 3072
spec = synth.uniform_u32(1, (n_cells * n_ch, 140), device="cuda").view(torch.uint8).contiguous()
with P.PirServer(n_cells, n_ch, d, lwe_n=4) as s:
    for _ in range(2):
        s.puzzle_bind_hct(0, spec, 5, 20, 3, mldsa_seed=bytes(range(32)))
    torch.cuda.synchronize()
print("ok")
