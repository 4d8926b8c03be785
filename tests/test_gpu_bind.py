"""NEXT-4: PSD.Puzzle.Bind with HCT puzzles on the GPU (Alg. 1 step 1, P:553-566;
HCT.Puzzle.Gen P:855; record layout P:1686, DESIGN R21) through the C ABI,
bit-exact against the oracle's qo_puzzle_bind_hct + qo_pack."""
import numpy as np
import pytest
import torch

import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _P():
    import paper_2510_03631_b200 as P
    return P


def _u32(t):
    return _P().u32(t)


def _read_D(s, m):
    """The whole shard, exactly: ANS for Q = identity (one query per cell) is D^T."""
    Q = np.eye(m, dtype=np.uint32)
    return _u32(s.answer_batch(Q)).T.astype(np.uint8)


@pytest.mark.parametrize("stride,device", [(600, False), (560, True), (576, False)])
@pytest.mark.parametrize("n_cells,n_ch,m", [(64, 3, 0), (40, 2, 16), (37, 3, 0)])
def test_bind_whole_db_matches_oracle(cuda_ok, n_cells, n_ch, m, stride, device):
    """Every record bound on the GPU: the shard equals the oracle's pack of the
    oracle's bound records, byte for byte.  Spectrum strides 560 / 576 (16-byte
    aligned: register-transposed kernel) and 600 (per-byte kernel); ragged cell
    counts leave partial 16-cell groups."""
    P = _P()
    d = 3072
    n = n_cells * n_ch
    spec = synth.uniform_u8_np(11, (n, stride))
    seed, kappa, n_l = 0xC0FFEE1234, 20, 3
    want_rec = O.puzzle_bind_hct(spec, 0, seed, kappa, n_l, d)
    with P.PirServer(n_cells, n_ch, d, m=m, lwe_n=4) as s:
        s.puzzle_bind_hct(0, torch.from_numpy(spec).cuda() if device else spec, seed, kappa, n_l)
        D = _read_D(s, s.m)
    assert (D == O.pack(want_rec, n_cells, n_ch, d, m or n_cells)).all()


def test_bind_ragged_range_device_spectrum_and_shard(cuda_ok):
    """A ragged theta range with a device spectrum (stride 560) on top of a
    written DB, on a row shard: bound records replaced, the rest untouched."""
    P = _P()
    n_cells, n_ch, d = 48, 2, 3072
    n = n_cells * n_ch
    base = synth.records_np(3, n, d, n_ch)
    t0, cnt = 5, 77
    spec = synth.uniform_u8_np(12, (cnt, 560))  # 16-byte aligned rows: the tiled kernel
    want = base.copy()
    want[t0:t0 + cnt] = O.puzzle_bind_hct(spec, t0, 77, 0xDEADBEEF, 9, d)
    full = O.pack(want, n_cells, n_ch, d, n_cells)
    r0, r1 = 2000, 4096 + 123
    with P.PirServer(n_cells, n_ch, d, lwe_n=4, row_begin=r0, row_end=r1, records=base) as s:
        s.puzzle_bind_hct(t0, torch.from_numpy(spec).cuda(), 77, 0xDEADBEEF, 9)
        D = _read_D(s, n_cells)
    assert (D == full[r0:r1]).all()


def test_bind_then_answer_without_sync(cuda_ok):
    """The bind's pack kernel writes D; the next GEMV (launched right after, no
    sync) must see it (launched without programmatic dependent launch)."""
    P = _P()
    n_cells, n_ch, d = 32, 2, 3072
    n = n_cells * n_ch
    spec = torch.from_numpy(synth.uniform_u8_np(13, (n, 560))).cuda()
    qu = synth.uniform_u32_np(14, (n_cells,))
    want_rec = O.puzzle_bind_hct(spec.cpu().numpy(), 0, 5, 20, 3, d)
    D = O.pack(want_rec, n_cells, n_ch, d, n_cells)
    with P.PirServer(n_cells, n_ch, d, lwe_n=4, stable_inputs=True) as s:
        qd = torch.from_numpy(qu.view(np.int32)).cuda()
        torch.cuda.synchronize()
        s.answer(qd)  # a GEMV in flight before the bind
        s.puzzle_bind_hct(0, spec, 5, 20, 3)
        got = s.answer(qd)
        torch.cuda.synchronize()
        assert (_u32(got) == O.answer(D, qu)).all()


@pytest.mark.parametrize("r,d", [(1000, 3072), (333, 600)])
def test_ens_bind_matches_oracle(cuda_ok, r, d):
    """ENS records bound in place; unit shares return single bound records and a
    random share returns the oracle's XOR of the selected bound records; the
    first scan runs right after the bind with no sync."""
    P = _P()
    spec = synth.uniform_u8_np(r + d, (r, 560))
    want = O.puzzle_bind_hct(spec, 0, 42, 20, 3, d)
    nb = (r + 7) // 8
    share = synth.uniform_u8_np(7, (nb,))
    if r % 8:
        share[-1] &= (1 << (r % 8)) - 1
    with P.EnsServer(r, d, stable_inputs=True) as s:
        sd = torch.from_numpy(share).cuda()
        torch.cuda.synchronize()
        s.puzzle_bind_hct(0, torch.from_numpy(spec).cuda(), 42, 20, 3)
        got = s.answer(sd).cpu().numpy()
        assert (got == O.ens_respond(want, share)).all()
        for t in (0, r // 2, r - 1):
            u = np.zeros(nb, np.uint8)
            u[t >> 3] = 1 << (t & 7)
            assert (s.answer(u).cpu().numpy() == want[t]).all()


def test_bind_errors_name_the_field(cuda_ok):
    P = _P()
    spec = np.zeros((4, 560), np.uint8)
    with P.PirServer(16, 1, 64, lwe_n=4) as s:  # records too small for a puzzle
        with pytest.raises(RuntimeError, match="rec_bytes"):
            s.puzzle_bind_hct(0, spec, 1)
    with P.PirServer(16, 1, 3072, lwe_n=4) as s:
        with pytest.raises(RuntimeError, match="spec_stride"):
            s.puzzle_bind_hct(0, np.zeros((4, 100), np.uint8), 1)
        with pytest.raises(RuntimeError, match="theta range"):
            s.puzzle_bind_hct(14, spec, 1)
        s.puzzle_bind_hct(3, np.zeros((0, 560), np.uint8), 1)  # empty range: a no-op
    with P.PirServer(16, 1, 1000, lwe_n=4) as s:  # room for the puzzle, not for a signature
        s.puzzle_bind_hct(0, spec, 1)
        with pytest.raises(RuntimeError, match="rec_bytes"):
            s.puzzle_bind_hct(0, spec, 1, mldsa_seed=bytes(32))


# ------------------------------------------------------------------ ML-DSA-44 signatures
_XI = bytes((7 * j + 3) & 0xFF for j in range(32))


@pytest.mark.parametrize("device_spec", [True, False])
def test_signed_bind_matches_oracle(cuda_ok, device_spec):
    """Puzzle.Bind with the ML-DSA-44 signature of every puzzle (Alg. 1 step 1):
    the GPU's public key equals the oracle's (and OpenSSL's), and the whole shard
    -- spectrum, puzzle and 2420-byte signature of every record -- equals the
    oracle's pack of the oracle's signed records byte for byte (deterministic
    FIPS 204 signing); ragged cells leave partial 16-cell groups."""
    P = _P()
    n_cells, n_ch, d = 21, 2, 3072
    n = n_cells * n_ch
    spec = synth.uniform_u8_np(21, (n, 560))
    want = O.puzzle_bind_hct_signed(spec, 0, 99, 20, 3, d, _XI)
    with P.PirServer(n_cells, n_ch, d, lwe_n=4) as s:
        pk = s.puzzle_bind_hct(0, torch.from_numpy(spec).cuda() if device_spec else spec, 99, 20, 3,
                               mldsa_seed=_XI)
        D = _read_D(s, n_cells)
    from oracle import mldsa
    assert pk == mldsa.keygen(_XI)[0]
    assert (D == O.pack(want, n_cells, n_ch, d, n_cells)).all()


def test_signed_bind_signatures_verify_with_openssl(cuda_ok):
    """Independent check: signatures read back from the GPU-bound ENS records
    verify under OpenSSL's ML-DSA-44 (cryptography) with the GPU's public key,
    and a corrupted record does not."""
    lib = pytest.importorskip("cryptography.hazmat.primitives.asymmetric.mldsa")
    P = _P()
    r, d = 64, 3072
    spec = synth.uniform_u8_np(22, (r, 560))
    with P.EnsServer(r, d) as s:
        pk = s.puzzle_bind_hct(0, torch.from_numpy(spec).cuda(), 123, 20, 3, mldsa_seed=_XI)
        nb = (r + 7) // 8
        recs = []
        for t in (0, 17, r - 1):
            u = np.zeros(nb, np.uint8)
            u[t >> 3] = 1 << (t & 7)
            recs.append((t, s.answer(u).cpu().numpy()))
    pub = lib.MLDSA44PublicKey.from_public_bytes(pk)
    for t, rec in recs:
        assert (rec[:560] == spec[t]).all()
        pub.verify(rec[597:3017].tobytes(), rec[560:597].tobytes())
    bad = recs[0][1].copy()
    bad[700] ^= 1
    with pytest.raises(Exception):
        pub.verify(bad[597:3017].tobytes(), bad[560:597].tobytes())


def test_signed_bind_ens_matches_oracle(cuda_ok):
    P = _P()
    r, d = 40, 3100
    spec = synth.uniform_u8_np(23, (r, 560))
    want = O.puzzle_bind_hct_signed(spec, 0, 5, 7, 1, d, _XI)
    with P.EnsServer(r, d) as s:
        s.puzzle_bind_hct(0, spec, 5, 7, 1, mldsa_seed=_XI)
        Q = np.zeros((r, (r + 7) // 8), np.uint8)
        for t in range(r):
            Q[t, t >> 3] = 1 << (t & 7)
        got = s.answer_batch(Q).cpu().numpy()
    assert (got == want).all()


def test_signed_bind_crosses_signing_chunks(cuda_ok):
    """More records than one signing launch takes (64K): the persistent signer warps
    draw records from a per-launch device counter, so the records at the chunk edges
    and a random sample must equal the oracle's signed records (and verify under
    OpenSSL's ML-DSA-44 when the package is present)."""
    P = _P()
    r, d = 70000, 3072
    spec = synth.uniform_u8_np(31, (r, 560))
    rng = np.random.default_rng(5)
    picks = sorted(set([0, 1, 65535, 65536, 65537, r - 1] + [int(t) for t in rng.integers(0, r, 18)]))
    with P.EnsServer(r, d) as s:
        pk = s.puzzle_bind_hct(0, torch.from_numpy(spec).cuda(), 9, 20, 3, mldsa_seed=_XI)
        Q = np.zeros((len(picks), (r + 7) // 8), np.uint8)
        for i, t in enumerate(picks):
            Q[i, t >> 3] = 1 << (t & 7)
        got = s.answer_batch(Q).cpu().numpy()
    for i, t in enumerate(picks):
        want = O.puzzle_bind_hct_signed(spec[t:t + 1], t, 9, 20, 3, d, _XI)
        assert (got[i] == want[0]).all(), t
    try:
        from cryptography.hazmat.primitives.asymmetric import mldsa as lib
    except ImportError:
        return
    pub = lib.MLDSA44PublicKey.from_public_bytes(pk)
    for i, t in enumerate(picks):
        pub.verify(got[i, 597:3017].tobytes(), got[i, 560:597].tobytes())


@pytest.mark.parametrize("seed", range(6))
def test_bind_fuzz_geometries(cuda_ok, seed):
    """Random geometries (cells, channels, m, record size, row shard, bound theta
    range, spectrum stride / placement) through both packing kernels: the
    shard equals the oracle's pack of the oracle's bound records, with the
    unbound records left as written."""
    P = _P()
    rng = np.random.default_rng(1000 + seed)
    n_ch = int(rng.integers(1, 4))
    n_cells = int(rng.integers(5, 70))
    m = int(rng.choice([0, 16, 32]))
    d = int(rng.choice([608, 640, 1000, 3072]))
    n = n_cells * n_ch
    t0 = int(rng.integers(0, n // 2))
    cnt = int(rng.integers(1, n - t0 + 1))
    stride = int(rng.choice([560, 576, 600]))
    base = synth.uniform_u8_np(2000 + seed, (n, d))
    spec = synth.uniform_u8_np(3000 + seed, (cnt, stride))
    want = base.copy()
    want[t0:t0 + cnt] = O.puzzle_bind_hct(spec, t0, 55 + seed, 20 + seed, seed, d)
    mm = m or n_cells
    full = O.pack(want, n_cells, n_ch, d, mm)
    ell = full.shape[0]
    r0 = int(rng.integers(0, ell // 2))
    r1 = int(rng.integers(r0 + 1, ell + 1))
    with P.PirServer(n_cells, n_ch, d, m=m, lwe_n=4, row_begin=r0, row_end=r1, records=base) as s:
        sp = torch.from_numpy(spec).cuda() if seed % 2 else spec
        s.puzzle_bind_hct(t0, sp, 55 + seed, 20 + seed, seed)
        D = _read_D(s, s.m)
    assert (D == full[r0:r1]).all()
