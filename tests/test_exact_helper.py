"""Pins for tests/_exact.py (the float64-limb product used by the full-size
Freivalds checks): oracle parity on small inputs, a closed form at the largest
K it is used at, and the wrap behaviour."""
import numpy as np
import pytest

import synth
from oracle import oracle as O
from _exact import matmul_mod32


@pytest.mark.parametrize("rows,K,n", [(1, 1, 1), (37, 300, 5), (130, 4097, 40)])
def test_u8_times_u32_matches_oracle(rows, K, n):
    D = synth.uniform_u8_np(rows + K, (rows, K))
    V = synth.uniform_u32_np(n + K, (n, K))
    want = O.answer_batch(D, V)                       # (n, rows): D . v for each v
    got = matmul_mod32(D, np.ascontiguousarray(V.T), row_chunk=64).T
    assert (got == want).all()


def test_u32_times_u32_matches_brute_force():
    A = synth.uniform_u32_np(5, (19, 211))
    B = synth.uniform_u32_np(6, (211, 7))
    want = np.array([[sum(int(A[i, k]) * int(B[k, j]) for k in range(211)) % (1 << 32)
                      for j in range(7)] for i in range(19)], np.uint32)
    assert (matmul_mod32(A, B, row_chunk=8) == want).all()


def test_closed_form_at_c5_depth():
    """All-255 D against all-(2^32 - 1) v over K = 262144 (the C5 depth):
    sum = K * 255 * (2^32 - 1) == -255 K (mod 2^32)."""
    K = 262144
    D = np.full((3, K), 255, np.uint8)
    V = np.full((K, 2), 0xFFFFFFFF, np.uint32)
    want = (-255 * K) % (1 << 32)
    assert (matmul_mod32(D, V) == want).all()
