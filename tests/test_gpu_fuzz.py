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


@pytest.mark.parametrize("case", range(10))
def test_fuzz_engine_knobs(cuda_ok, case, monkeypatch):
    """The tcgen05 engine under random tuning knobs (lockstep chunk, forced
    K-splits, row panels per tile, K-block size, limb count of the F_p path) on
    shapes long enough in K for lockstep and several column tiles: bit-exact."""
    P = _P()
    rng = np.random.default_rng(3000 + case)
    knobs = {"QPIR_MMA_LOCKSTEP": str(int(rng.choice([0, 1, 2, 16]))),
             "QPIR_MMA_DRIFT": str(int(rng.choice([1, 2]))),
             "QPIR_MMA_SPLIT": str(int(rng.choice([0, 0, 1, 3, 7]))),
             "QPIR_MMA_MT": str(int(rng.choice([1, 2]))),
             "QPIR_MMA_GPB": str(int(rng.choice([4, 8]))),
             "QPIR_MODP2": str(int(rng.choice([0, 1]))),
             "QPIR_MODP3": str(int(rng.choice([0, 1])))}
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    n_cells = int(rng.integers(4000, 12000))
    n_ch = int(rng.integers(1, 5))
    d = int(rng.integers(8, 100))
    n = int(rng.choice([65, 128, 200]))
    B = int(rng.choice([3, 40, 100]))
    rec = synth.uniform_u8_np(case + 70, (n_cells * n_ch, d))
    D = O.pack(rec, n_cells, n_ch, d, n_cells)
    with P.PirServer(n_cells, n_ch, d, lwe_n=n, seed_A=case + 1, records=rec) as s:
        Q = synth.uniform_u32_np(case + 80, (B, n_cells))
        assert (P.u32(s.answer_batch(Q)) == O.answer_batch(D, Q)).all(), knobs
        assert (P.u32(s.hint()) == O.hint(D, O.expand_A(case + 1, n_cells, n))).all(), knobs
        p = int(rng.choice([257, 65521, 65537, 16777213, 2147483647]))
        Qp = Q.copy()
        Qp[0, : min(50, n_cells)] = 65536  # residue 65536 entries (p = 65537 exceptions)
        want = ((Qp.astype(np.uint64) % p).astype(object) @ D.T.astype(object)) % p
        assert (P.u32(s.answer_batch_modp(Qp, p)) == want.astype(np.uint32)).all(), knobs


@pytest.mark.parametrize("case", range(10))
def test_fuzz_scan_knobs(cuda_ok, case, monkeypatch):
    """GEMV and ENS scan under random tuning knobs (rows per thread, groups in
    flight, forced splits, smem chunk, TMA variant, PDL; ENS rows per CTA, rows
    in flight, reduction group, wide / 256-bit kernels, PDL), several answers
    back to back on one stream: bit-exact."""
    P = _P()
    rng = np.random.default_rng(4000 + case)
    knobs = {"QPIR_GEMV_U": str(int(rng.choice([1, 2, 4]))),
             "QPIR_GEMV_UNROLL": str(int(rng.choice([4, 8]))),
             "QPIR_GEMV_SPLIT": str(int(rng.choice([0, 1, 3, 9]))),
             "QPIR_GEMV_CHUNK": str(int(rng.choice([64, 512]))),
             "QPIR_GEMV_L2PF": str(int(rng.choice([0, 1]))),
             "QPIR_GEMV_PDL": str(int(rng.choice([0, 1]))),
             "QPIR_ENS_ROWS": str(int(rng.choice([0, 32, 96]))),
             "QPIR_ENS_UR": str(int(rng.choice([4, 8, 16]))),
             "QPIR_ENS_GROUP": str(int(rng.choice([0, 1, 5]))),
             "QPIR_ENS_WIDE": str(int(rng.choice([0, 1, 2]))),
             "QPIR_ENS_PDL": str(int(rng.choice([0, 1])))}
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    n_cells = int(rng.integers(100, 9000))
    n_ch = int(rng.integers(1, 5))
    d = int(rng.integers(1, 64))
    rec = synth.uniform_u8_np(case + 90, (n_cells * n_ch, d))
    D = O.pack(rec, n_cells, n_ch, d, n_cells)
    with P.PirServer(n_cells, n_ch, d, records=rec) as s:
        qs = [synth.uniform_u32_np(case * 10 + i, (n_cells,)) for i in range(4)]
        outs = [s.answer(torch.from_numpy(q.view(np.int32)).cuda()) for q in qs]
        for q, o in zip(qs, outs):
            assert (P.u32(o) == O.answer(D, q)).all(), knobs
    r = int(rng.integers(33, 5000))
    de = int(rng.choice([16, 48, 3072, int(rng.integers(1, 4000))]))
    rec2 = synth.uniform_u8_np(case + 95, (r, de))
    with P.EnsServer(r, de, records=rec2) as s:
        shs = []
        for i in range(4):
            q = synth.uniform_u8_np(case * 10 + 5 + i, ((r + 7) // 8,))
            if r % 8:
                q[-1] &= (1 << (r % 8)) - 1
            shs.append(q)
        outs = [s.answer(torch.from_numpy(q).cuda()) for q in shs]
        for q, o in zip(shs, outs):
            assert (o.cpu().numpy() == O.ens_respond(rec2, q)).all(), knobs
