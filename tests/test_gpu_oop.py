"""GPU parity for QPADL-OOP (CIP-PIR offline-online, NEXT-3) against the oracle."""
import numpy as np
import pytest
import torch

import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _P():
    import paper_2510_03631_b200 as P
    return P


@pytest.mark.parametrize("B,d,n", [(96, 20, 2), (4096, 64, 4), (1000, 3072, 5), (30000, 16, 3)])
def test_oop_preprocess_and_answer_match_oracle(cuda_ok, B, d, n):
    P = _P()
    rec = synth.uniform_u8_np(B + d + n, (B, d))
    seeds = np.array([11, 22, 33, 44, 55, 66][:n], np.uint64)
    with P.EnsServer(B, d, records=rec) as s:
        for i in range(n):
            A = s.oop_preprocess(n, i, torch.from_numpy(seeds.view(np.int64)).cuda()).cpu().numpy()
            for j in range(n):
                assert (A[j] == O.oop_preprocess(rec, n, i, int(seeds[j]))).all(), (i, j)
        theta = B // 3
        q = O.oop_query(theta, B, n, seeds)
        resp = []
        for i in range(n):
            A_i = O.oop_preprocess(rec, n, i, int(seeds[i]))
            r_gpu = s.oop_answer(n, i, q[i], A_i).cpu().numpy()
            assert (r_gpu == O.oop_respond(rec, n, i, q[i], A_i)).all()
            resp.append(r_gpu)
        assert (np.bitwise_xor.reduce(np.stack(resp), axis=0) == rec[theta]).all()


def test_oop_end_to_end_all_gpu(cuda_ok):
    """Offline A_i and online R_i both from the GPU; every block of a small DB."""
    P = _P()
    B, d, n = 256, 48, 4
    rec = synth.uniform_u8_np(77, (B, d))
    with P.EnsServer(B, d, records=torch.from_numpy(rec).cuda()) as s:
        for theta in range(0, B, 5):
            seeds = (np.arange(n, dtype=np.uint64) + 1) * 977 + theta
            A = [s.oop_preprocess(n, i, seeds[i:i + 1].view(np.int64).copy())[0] for i in range(n)]
            q = O.oop_query(theta, B, n, seeds)
            out = np.bitwise_xor.reduce(
                np.stack([s.oop_answer(n, i, q[i], A[i]).cpu().numpy() for i in range(n)]), axis=0)
            assert (out == rec[theta]).all()
