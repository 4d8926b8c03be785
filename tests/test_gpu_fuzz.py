"""Seeded fuzz over random geometries (SPEC S:247-style "fuzzed dimension
sweeps"): every path through the C ABI against the oracle, bit-exact."""
import numpy as np
import pytest
import torch

import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _P():
    import paper_2510_03631_b200 as P
    return P


@pytest.mark.parametrize("case", range(12))
def test_fuzz_lwe_paths(cuda_ok, case):
    P = _P()
    rng = np.random.default_rng(1000 + case)
    n_cells = int(rng.integers(1, 3000))
    n_ch = int(rng.integers(1, 9))
    d = int(rng.integers(1, 80))
    m = int(rng.choice([0, rng.integers(1, n_cells + 1)]))
    m_eff = m or n_cells
    rec = synth.uniform_u8_np(case, (n_cells * n_ch, d))
    D = O.pack(rec, n_cells, n_ch, d, m_eff)
    ell = D.shape[0]
    r0 = int(rng.integers(0, ell))
    r1 = int(rng.integers(r0 + 1, ell + 1))
    n = int(rng.choice([1, 3, 4, 17, 64]))
    B = int(rng.choice([1, 2, 5, 31, 64, 100]))
    with P.PirServer(n_cells, n_ch, d, m=m, lwe_n=n, seed_A=case, row_begin=r0, row_end=r1,
                     records=rec) as s:
        qu = synth.uniform_u32_np(case + 50, (m_eff,))
        assert (P.u32(s.answer(qu)) == O.answer(D[r0:r1], qu)).all()
        Q = synth.uniform_u32_np(case + 60, (B, m_eff))
        assert (P.u32(s.answer_batch(Q)) == O.answer_batch(D[r0:r1], Q)).all()
        assert (P.u32(s.hint()) == O.hint(D[r0:r1], O.expand_A(case, m_eff, n))).all()
        p = int(rng.choice([2, 251, 65537, 4294967291]))
        want = ((Q.astype(object) @ D[r0:r1].T.astype(object)) % p).astype(np.uint32)
        assert (P.u32(s.answer_batch_modp(Q, p)) == want).all()


@pytest.mark.parametrize("case", range(8))
def test_fuzz_ens_oop(cuda_ok, case):
    P = _P()
    rng = np.random.default_rng(2000 + case)
    n = int(rng.integers(2, 6))
    r = n * int(rng.integers(1, 900))
    d = int(rng.integers(1, 300))
    rec = synth.uniform_u8_np(case + 7, (r, d))
    nb = (r + 7) // 8
    with P.EnsServer(r, d, records=rec) as s:
        q = synth.uniform_u8_np(case + 8, (nb,))
        if r % 8:
            q[-1] &= (1 << (r % 8)) - 1
        assert (s.answer(q).cpu().numpy() == O.ens_respond(rec, q)).all()
        B = int(rng.choice([3, 40]))
        Q = synth.uniform_u8_np(case + 9, (B, nb))
        if r % 8:
            Q[:, -1] &= (1 << (r % 8)) - 1
        assert (s.answer_batch(Q).cpu().numpy() == O.ens_respond_batch(rec, Q)).all()
        seeds = (np.arange(n, dtype=np.uint64) + 3) * 1299709 + case
        theta = int(rng.integers(0, r))
        qq = O.oop_query(theta, r, n, seeds)
        out = np.zeros(d, np.uint8)
        for i in range(n):
            A = s.oop_preprocess(n, i, seeds[i:i + 1].view(np.int64).copy())[0]
            out ^= s.oop_answer(n, i, qq[i], A).cpu().numpy()
        assert (out == rec[theta]).all()
