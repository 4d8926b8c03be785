"""Exact products over Z_{2^32} for the full-size Freivalds checks (test
infrastructure).

The oracle's C loops (oracle/qpir_oracle.c) are the reference for every
element-by-element parity test, but a Freivalds right side at C4 / C5 size is
~10^12 multiply-adds -- too slow for plain loops.  This module computes the
same product with a library primitive (float64 BLAS matmul via torch CPU),
independently of both the oracle and the CUDA path: every u32 operand is split
into 16-bit limbs (u8 operands stay whole), and a limb product summed over K
terms is at most K * (2^16 - 1)^2, exact in float64 while that is < 2^53
(K < 2.1e6; K < 5.4e8 when one side is u8).  The limb
products are reduced mod 2^32 before they are shifted and summed, so the int64
combination never overflows.  Pinned against the oracle on small inputs and
against a closed form in tests/test_exact_helper.py.
"""
from __future__ import annotations

import numpy as np
import torch

_M32 = (1 << 32) - 1


def _limbs(x: np.ndarray):
    """(limbs, width): a u8 array whole, a u32 array as two 16-bit limbs, as
    float64 tensors."""
    if x.dtype == np.uint8:
        return [torch.from_numpy(np.ascontiguousarray(x)).to(torch.float64)], 8
    t = torch.from_numpy(np.ascontiguousarray(x).astype(np.int64))
    return [(t & 0xFFFF).to(torch.float64), (t >> 16).to(torch.float64)], 16


def matmul_mod32(A: np.ndarray, B: np.ndarray, row_chunk: int = 256) -> np.ndarray:
    """(A @ B) mod 2^32 for unsigned integer A (M, K) and B (K, N), A of dtype
    uint8 or uint32, B of dtype uint8 or uint32.  Returns uint32 (M, N)."""
    assert A.ndim == 2 and B.ndim == 2 and A.shape[1] == B.shape[0]
    K = A.shape[1]
    assert A.dtype in (np.uint8, np.uint32) and B.dtype in (np.uint8, np.uint32)
    Bl, wb = _limbs(B)
    wa = 8 if A.dtype == np.uint8 else 16
    assert K * ((1 << wa) - 1) * ((1 << wb) - 1) < (1 << 53), "K too large for exact float64 sums"
    M, N = A.shape[0], B.shape[1]
    out = np.empty((M, N), np.uint32)
    for r0 in range(0, M, row_chunk):
        Al, _ = _limbs(A[r0:r0 + row_chunk])
        acc = torch.zeros((Al[0].shape[0], N), dtype=torch.int64)
        for i in range(len(Al)):
            for j in range(len(Bl)):
                s = wa * i + wb * j
                if s >= 32:
                    continue
                p = torch.matmul(Al[i], Bl[j]).to(torch.int64) & _M32
                acc = (acc + ((p << s) & _M32)) & _M32
        out[r0:r0 + row_chunk] = acc.numpy().astype(np.uint32)
    return out
