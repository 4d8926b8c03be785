"""Pins of the CPU oracle against things other than itself (no GPU needed).

Each test names what fixes the expected value: a published KAT, a library
routine (numpy / torch integer matmul), a closed form, an invariant, or brute
force.  See DESIGN.md "Oracle pins".
"""
import os

import numpy as np
import pytest
import torch

import synth
from oracle import noise
from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
M32 = (1 << 32) - 1


# ------------------------------------------------------------------ Philox
def test_philox_known_answers():
    """Random123 KAT vectors (tests/golden/philox4x32_10_kat.txt)."""
    n = 0
    for line in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        out = O.philox4x32_10(v[0:4], v[4:6])
        assert list(out) == v[6:10], line
        n += 1
    assert n == 3


def test_expand_A_indexing():
    """A[c][j] = Philox(key=seed, ctr=(c, j>>2, 0, 0x41))[j&3] (DESIGN R7)."""
    seed = 0x0123456789ABCDEF
    A = O.expand_A(seed, 37, 12)
    key = [seed & M32, seed >> 32]
    for c in (0, 1, 36):
        for j in range(12):
            assert A[c, j] == O.philox4x32_10([c, j >> 2, 0, 0x41], key)[j & 3]
    # four consecutive j share one Philox block, distinct blocks differ
    assert len(set(A[0].tolist())) == 12


def test_keygen_indexing():
    """s[j] = Philox(key=seed_s, ctr=(j>>2, 0, 0, 0x53))[j&3] (DESIGN R6), each
    element re-derived from the KAT-pinned Philox.  Catches s = 0, a wrong
    domain tag, A's stream reused for s, and a wrong j -> (block, lane) map."""
    seed = 0xFEDCBA9876543210
    n = 19
    s = O.keygen(seed, n)
    key = [seed & M32, seed >> 32]
    assert s.dtype == np.uint32 and s.shape == (n,)
    for j in range(n):
        assert s[j] == O.philox4x32_10([j >> 2, 0, 0, 0x53], key)[j & 3]
    assert (s != 0).all() and len(set(s.tolist())) == n
    # not A's stream: A[c=0..n) is drawn with domain 0x41 and ctr[0] = cell
    A = O.expand_A(seed, 1, n)
    assert (A[0] != s).all()
    # distinct seeds give distinct secrets; the key uses both seed halves
    assert (O.keygen(seed ^ 1, n) != s).any() and (O.keygen(seed ^ (1 << 40), n) != s).any()


# ------------------------------------------------------------------ layout
@pytest.mark.parametrize("n_cells,n_ch,d,m", [(16, 3, 5, 16), (20, 3, 4, 8), (7, 2, 3, 3)])
def test_layout_is_a_bijection(n_cells, n_ch, d, m):
    """S:81-style bijection: (theta, b) -> (row, col) is injective into ell x m."""
    ell = O.ell(n_cells, n_ch, d, m)
    assert ell == -(-n_cells // m) * n_ch * d
    seen = set()
    for theta in range(n_cells * n_ch):
        for b in range(d):
            r, c = O.position(n_ch, d, m, theta, b)
            assert 0 <= r < ell and 0 <= c < m
            seen.add((r, c))
            # one query column per cell: every byte of every channel of a cell
            # sits in column cell % m (multiple-block retrieval)
            assert c == (theta // n_ch) % m
    assert len(seen) == n_cells * n_ch * d
    if n_cells % m == 0:
        assert len(seen) == ell * m  # no unused slots


def test_pack_places_records():
    n_cells, n_ch, d, m = 10, 3, 4, 4
    rec = synth.uniform_u8_np(5, (n_cells * n_ch, d))
    D = O.pack(rec, n_cells, n_ch, d, m)
    for theta in range(n_cells * n_ch):
        rows = O.record_rows(theta, n_ch, d, m)
        col = (theta // n_ch) % m
        assert (D[rows.astype(np.int64), col] == rec[theta]).all()
    # unused slots (cells 10, 11 of the last block) are zero
    assert D[2 * n_ch * d:, 2:].sum() == 0


@pytest.mark.parametrize("n_cells,d", [(7, 5), (64, 48)])
def test_one_channel_pack_is_transpose(n_cells, d):
    """R10 with n_ch = 1 and m = n_cells: D[b][cell] = rec_cell[b], i.e. D = rec^T
    (the full-size Freivalds tests build their right side this way)."""
    rec = synth.uniform_u8_np(6 + d, (n_cells, d))
    assert (O.pack(rec, n_cells, 1, d, n_cells) == rec.T).all()


# ------------------------------------------------------------------ answer
def _np_answer(D, qu):
    # numpy integer matmul (non-BLAS loop in uint32: wraps mod 2^32)
    return D.astype(np.uint32) @ qu.astype(np.uint32)


def _torch_answer(D, qu):
    # torch int64 matmul is exact here (|sum| < m * 255 * 2^32 < 2^63), then mod 2^32
    return (torch.from_numpy(D.astype(np.int64)) @ torch.from_numpy(qu.astype(np.int64))).numpy() & M32


@pytest.mark.parametrize("rows,m", [(1, 1), (3, 17), (130, 1000), (64, 4096)])
def test_answer_matches_library_matmul(rows, m):
    D = synth.uniform_u8_np(11 + m, (rows, m))
    qu = synth.uniform_u32_np(12 + m, (m,))
    a = O.answer(D, qu)
    assert (a == _np_answer(D, qu)).all()
    assert (a.astype(np.int64) == _torch_answer(D, qu)).all()


def test_answer_closed_forms():
    rows, m = 40, 300
    D = synth.uniform_u8_np(21, (rows, m))
    rs = D.astype(np.int64).sum(1)
    # unit query e_c -> column c;   Delta e_c -> Delta * column c
    for c in (0, 7, m - 1):
        e = np.zeros(m, np.uint32)
        e[c] = 1
        assert (O.answer(D, e) == D[:, c]).all()
        e[c] = 1 << 24
        assert (O.answer(D, e).astype(np.int64) == (D[:, c].astype(np.int64) << 24) & M32).all()
    # all-ones -> row sums;   all 0xFFFFFFFF (= -1) -> -row sums mod 2^32
    assert (O.answer(D, np.ones(m, np.uint32)).astype(np.int64) == rs).all()
    assert (O.answer(D, np.full(m, M32, np.uint32)).astype(np.int64) == (-rs) & M32).all()
    # constant D = k -> k * sum(qu)
    qu = synth.uniform_u32_np(22, (m,))
    k = 201
    Dk = np.full((3, m), k, np.uint8)
    assert (O.answer(Dk, qu).astype(np.int64) == (k * int(qu.astype(np.int64).sum())) & M32).all()
    # top-limb-only query x * 2^24 -> 2^24 * (D.x mod 2^8)
    x = synth.uniform_u8_np(23, (m,))
    top = x.astype(np.uint32) << 24
    want = ((D.astype(np.int64) @ x.astype(np.int64)) % 256) << 24
    assert (O.answer(D, top).astype(np.int64) == want).all()


def test_answer_linearity():
    D = synth.uniform_u8_np(31, (50, 513))
    q1 = synth.uniform_u32_np(32, (513,))
    q2 = synth.uniform_u32_np(33, (513,))
    s = (q1.astype(np.int64) + q2) & M32
    lhs = O.answer(D, s.astype(np.uint32)).astype(np.int64)
    rhs = (O.answer(D, q1).astype(np.int64) + O.answer(D, q2)) & M32
    assert (lhs == rhs).all()


def test_answer_batch_columns_and_library():
    D = synth.uniform_u8_np(41, (33, 257))
    Q = synth.uniform_u32_np(42, (5, 257))
    ANS = O.answer_batch(D, Q)
    want = (Q.astype(np.uint32) @ D.astype(np.uint32).T)  # wraps in uint32
    assert (ANS == want).all()
    for b in range(5):
        assert (ANS[b] == O.answer(D, Q[b])).all()


def test_chor_gf2_link():
    """P7: for 0/1 queries and 0/1 D, ans mod 2 is Chor's GF(2) response rho = q.DB
    (Alg. 3), computed here by brute-force XOR of the selected columns."""
    rows, m = 24, 200
    D = (synth.uniform_u8_np(51, (rows, m)) & 1).astype(np.uint8)
    q = (synth.uniform_u32_np(52, (m,)) & 1).astype(np.uint32)
    rho = np.zeros(rows, np.uint8)
    for c in range(m):
        if q[c]:
            rho ^= D[:, c]
    assert ((O.answer(D, q) & 1) == rho).all()


# ------------------------------------------------------------------ hint
def test_hint_matches_library_and_freivalds():
    rows, m, n = 37, 300, 24
    D = synth.uniform_u8_np(61, (rows, m))
    A = O.expand_A(99, m, n)
    H = O.hint(D, A)
    assert (H == D.astype(np.uint32) @ A).all()
    x = synth.uniform_u32_np(62, (n,))
    assert (H @ x == O.answer(D, A @ x)).all()  # H x == D (A x) mod 2^32


# ------------------------------------------------------------------ LWE client
def test_error_distribution():
    """e_c = round(N(0, sigma^2)) (DESIGN R5): moments and tail of 2e5 samples."""
    sigma = 6.4
    e = O.sample_error(7, 0, 200_000, sigma).astype(np.float64)
    assert abs(e.mean()) < 0.06
    assert abs(e.std() - np.sqrt(sigma ** 2 + 1 / 12)) < 0.05  # rounding adds 1/12
    assert np.abs(e).max() < 8 * sigma
    frac = (np.abs(e) <= sigma).mean()  # P(|round(N)| <= sigma) ~ P(|N| <= 6.5) = 0.689
    assert 0.68 < frac < 0.70
    assert (O.sample_error(7, 1, 16, sigma) != O.sample_error(7, 0, 16, sigma)).any()


def _tiny():
    n_cells, n_ch, d = 1024, 16, 8  # BASELINE.json configs[0]
    rec = synth.records_np(1, n_cells * n_ch, d, n_ch)
    D = O.pack(rec, n_cells, n_ch, d, n_cells)
    return n_cells, n_ch, d, rec, D


def test_lwe_identity_exact():
    """P4: ans - H s - Delta D[:, c*] == D e (mod 2^32), exactly, given the sampled e."""
    n_cells, n_ch, d, rec, D = _tiny()
    n = 256
    A = O.expand_A(3, n_cells, n)
    H = O.hint(D, A)
    s = O.keygen(4, n)
    for qidx, cstar in enumerate((0, 513, 1023)):
        qu, e = O.query(A, s, 5, qidx, 6.4, cstar)
        ans = O.answer(D, qu)
        lhs = (ans.astype(np.int64) - (H @ s).astype(np.int64)
               - (D[:, cstar].astype(np.int64) << 24)) & M32
        De = (D.astype(np.int64) @ e.astype(np.int64)) & M32
        assert (lhs == De).all()
        assert np.abs(D.astype(np.int64) @ e.astype(np.int64)).max() < (1 << 23)


def test_bruteforce_decode_every_record_tiny():
    """P1: decode(answer(query(theta))) == record theta for all 16384 records of
    the tiny DB (BASELINE.json configs[0]); one query per cell retrieves all of
    that cell's channels (multiple-block retrieval)."""
    n_cells, n_ch, d, rec, D = _tiny()
    n = 1024
    A = O.expand_A(3, n_cells, n)
    H = O.hint(D, A)
    s = O.keygen(4, n)
    rows_of_cell = np.arange(n_ch * d, dtype=np.uint64)  # m = n_cells: one block
    bad = 0
    for cell in range(n_cells):
        qu, _ = O.query(A, s, 5, cell, 6.4, cell)
        ans = O.answer(D, qu)
        got = O.decode(ans, H, s, rows_of_cell).reshape(n_ch, d)
        bad += int((got != rec[cell * n_ch:(cell + 1) * n_ch]).sum())
    assert bad == 0


def test_negative_control_large_noise():
    """P5: with sigma far beyond the bound, decoding must fail somewhere."""
    n_cells, n_ch, d, rec, D = _tiny()
    n = 64
    A = O.expand_A(3, n_cells, n)
    H = O.hint(D, A)
    s = O.keygen(4, n)
    sigma = 1e5
    assert noise.failure_prob(noise.worst_case_z(sigma, n_cells)) > 0.5
    qu, _ = O.query(A, s, 5, 0, sigma, 17)
    got = O.decode(O.answer(D, qu), H, s, np.arange(n_ch * d, dtype=np.uint64))
    assert (got != rec[17 * n_ch:18 * n_ch].reshape(-1)).sum() > n_ch * d // 2


def test_noise_bound_closed_forms():
    # z = 2^23 / (sigma * 255 * sqrt(m)) -- SURVEY 8(c) worst-case table
    assert noise.worst_case_z(6.4, 1024) == pytest.approx(160.627, rel=1e-4)
    assert noise.worst_case_z(6.4, 8192) == pytest.approx(56.79, rel=1e-3)
    assert noise.worst_case_z(6.4, 65536) == pytest.approx(20.08, rel=1e-3)
    assert noise.worst_case_z(6.4, 262144) == pytest.approx(10.04, rel=1e-3)
    assert noise.failure_prob(noise.worst_case_z(6.4, 262144)) < 1e-22
    mm = noise.max_m_for(6.4, -40.0)
    assert noise.failure_prob(noise.worst_case_z(6.4, mm)) <= 2.0 ** -40
    assert noise.failure_prob(noise.worst_case_z(6.4, mm + 1)) > 2.0 ** -40
