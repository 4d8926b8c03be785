"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (DESIGN "Parity"): bit-exact u32 equality -- every result is a unique value
in Z_{2^32}.  Expected values come only from oracle/ (or closed forms); inputs
come only from synth/ (or the oracle's client for LWE queries).
"""
import numpy as np
import pytest
import torch

import synth
from oracle import oracle as O
from _exact import matmul_mod32  # exact float64-limb products (pinned in test_exact_helper.py)

pytestmark = pytest.mark.gpu
M32 = (1 << 32) - 1


def _srv():
    import paper_2510_03631_b200 as P
    return P


def _u32(t):
    return _srv().u32(t)


def _db(n_cells, n_ch, d, m=0, seed=1):
    rec = synth.records_np(seed, n_cells * n_ch, d, n_ch)
    D = O.pack(rec, n_cells, n_ch, d, m or n_cells)
    return rec, D


# ------------------------------------------------------------------ GEMV (a3)
def test_answer_tiny_host_and_device(cuda_ok):
    P = _srv()
    n_cells, n_ch, d = 1024, 16, 8  # BASELINE.json configs[0]
    rec, D = _db(n_cells, n_ch, d)
    qu = synth.uniform_u32_np(2, (n_cells,))
    want = O.answer(D, qu)
    with P.PirServer(n_cells, n_ch, d, records=rec) as s:  # host records
        out = np.empty(s.ell_local, np.uint32)
        s.answer(qu, out=out)  # host in, host out
        assert (out == want).all()
        got = s.answer(torch.from_numpy(qu.view(np.int32)).cuda())  # device in/out
        assert (_u32(got) == want).all()
        assert s.kernel_launches >= 2
    with P.PirServer(n_cells, n_ch, d, records=torch.from_numpy(rec).cuda()) as s:  # device records
        assert (_u32(s.answer(qu)) == want).all()


RAGGED = [
    # n_cells, n_ch, d, m   (m=0 -> n_cells)
    (1000, 3, 5, 0),      # m not a multiple of 16/128, ell = 15 rows
    (333, 7, 11, 100),    # cells wrap into 4 row blocks (SimplePIR packing)
    (17, 1, 1, 0),        # single tiny row
    (4096, 40, 64, 0),    # 2560 rows, 4096 columns
    (2500, 9, 37, 640),   # several blocks, ragged everything
]


@pytest.mark.parametrize("geo", RAGGED)
@pytest.mark.parametrize("cfg", [dict(), dict(QPIR_GEMV_U="1", QPIR_GEMV_SPLIT="3", QPIR_GEMV_CHUNK="8"),
                                 dict(QPIR_GEMV_U="4", QPIR_GEMV_SPLIT="1", QPIR_GEMV_CHUNK="4"),
                                 dict(QPIR_GEMV_ORDER="1", QPIR_GEMV_SPLIT="5", QPIR_GEMV_UNROLL="8"),
                                 dict(QPIR_MMA_MT="1", QPIR_MMA_SPLIT="3")])
def test_answer_ragged(cuda_ok, geo, cfg, monkeypatch):
    for k, v in cfg.items():
        monkeypatch.setenv(k, v)
    P = _srv()
    n_cells, n_ch, d, m = geo
    rec, D = _db(n_cells, n_ch, d, m, seed=3)
    with P.PirServer(n_cells, n_ch, d, m=m, records=rec) as s:
        assert s.ell == D.shape[0] and s.m == D.shape[1]
        for seed in (4, 5):
            qu = synth.uniform_u32_np(seed, (s.m,))
            assert (_u32(s.answer(qu)) == O.answer(D, qu)).all()
        # closed form: all-0xFFFFFFFF query -> -row sums
        qf = np.full(s.m, M32, np.uint32)
        want = (-D.astype(np.int64).sum(1)) & M32
        assert (_u32(s.answer(qf)).astype(np.int64) == want).all()
        # the tensor-core batch path on the same ragged geometry
        Q = synth.uniform_u32_np(6, (5, s.m))
        assert (_u32(s.answer_batch(Q)) == O.answer_batch(D, Q)).all()


def test_shards_concatenate(cuda_ok):
    """P6: row shards answered separately concatenate to the unsharded answer."""
    P = _srv()
    n_cells, n_ch, d = 2048, 8, 24
    rec, D = _db(n_cells, n_ch, d, seed=6)
    qu = synth.uniform_u32_np(7, (n_cells,))
    want = O.answer(D, qu)
    rec_dev = torch.from_numpy(rec).cuda()
    from paper_2510_03631_b200.dist import shard_rows
    for world in (1, 2, 3, 8):
        parts = []
        for r in range(world):
            r0, r1 = shard_rows(n_cells, n_ch, d, n_cells, world, r)
            with P.PirServer(n_cells, n_ch, d, row_begin=r0, row_end=r1, records=rec_dev) as s:
                assert s.ell_local == r1 - r0
                parts.append(_u32(s.answer(qu)))
        assert (np.concatenate(parts) == want).all()


def test_db_write_streaming(cuda_ok):
    """Streaming the DB in odd-sized chunks gives the same D as one-shot setup."""
    P = _srv()
    n_cells, n_ch, d = 1500, 5, 12
    rec, D = _db(n_cells, n_ch, d, m=512, seed=8)
    qu = synth.uniform_u32_np(9, (512,))
    with P.PirServer(n_cells, n_ch, d, m=512) as s:
        n = n_cells * n_ch
        t = 0
        for k, step in enumerate((1, 7, 333, 1000, 5000)):
            chunk = rec[t:t + step]
            src = torch.from_numpy(chunk).cuda() if k % 2 else chunk
            s.db_write(t, src)
            t += chunk.shape[0]
        s.db_write(t, rec[t:n])
        assert (_u32(s.answer(qu)) == O.answer(D, qu)).all()


def test_mutation_one_db_byte_is_detected(cuda_ok):
    """SURVEY 5 mutation test: the parity checks have teeth.  Flip one byte of
    one record through qpir_db_write: the GEMV, the batch and the hint must then
    differ from the unmutated oracle in exactly that byte's row, by exactly
    delta * (query or A entry of its column) mod 2^32 (linearity of D -> D.x),
    and agree with the oracle on the mutated DB."""
    P = _srv()
    n_cells, n_ch, d, n = 1024, 16, 8, 64
    rec, D = _db(n_cells, n_ch, d, seed=90)
    theta, b = 5 * n_ch + 11, 6
    row, col = O.position(n_ch, d, n_cells, theta, b)
    qu = synth.uniform_u32_np(91, (n_cells,))
    Q = synth.uniform_u32_np(92, (5, n_cells))
    A = O.expand_A(93, n_cells, n)
    with P.PirServer(n_cells, n_ch, d, lwe_n=n, seed_A=93, records=rec) as s:
        assert (_u32(s.answer(qu)) == O.answer(D, qu)).all()
        assert (_u32(s.hint()) == O.hint(D, A)).all()
        bad = rec[theta].copy()
        delta = 0x5A
        bad[b] ^= delta
        s.db_write(theta, bad[None, :])
        D2 = D.copy()
        D2[row, col] = bad[b]
        diff = (int(bad[b]) - int(rec[theta][b])) & M32
        got, want = _u32(s.answer(qu)), O.answer(D, qu)
        assert (got != want).sum() == 1 and got[row] == (int(want[row]) + diff * int(qu[col])) & M32
        assert (got == O.answer(D2, qu)).all()
        gotB, wantB = _u32(s.answer_batch(Q)), O.answer_batch(D, Q)
        assert ((gotB != wantB).sum(0) > 0).sum() == 1 and (gotB[:, row] != wantB[:, row]).all()
        assert (gotB == O.answer_batch(D2, Q)).all()
        gotH, wantH = _u32(s.hint()), O.hint(D, A)
        assert ((gotH != wantH).sum(1) > 0).sum() == 1
        assert (gotH[row] == ((wantH[row].astype(np.int64) + diff * A[col].astype(np.int64)) & M32)).all()
        assert (gotH == O.hint(D2, A)).all()


@pytest.mark.parametrize("n_cells", [65536, 131072])
def test_wraparound_kat_gemv_and_tc(cuda_ok, n_cells, monkeypatch):
    """P9: all-0xFF D times all-0xFFFFFFFF queries with ONE K-split, so a single
    accumulator sums the whole row: every byte-limb sum is 255*255*m
    (4.26e9 > 2^31 at m = 65536; 8.52e9 > 2^32 at m = 131072), so the GEMV's
    dp4a accumulators and the tensor-core s32 TMEM accumulators must wrap mod
    2^32 (idesc saturate bit 0), never saturate.  QPIR_GEMV_SPLIT=1 /
    QPIR_MMA_SPLIT=1 force one unit per row tile (the auto split would cut K
    into pieces whose sums stay below 2^31).  Expected value in closed form:
    sum_c 255 * (2^32 - 1) = -255 * m mod 2^32."""
    monkeypatch.setenv("QPIR_GEMV_SPLIT", "1")
    monkeypatch.setenv("QPIR_MMA_SPLIT", "1")
    P = _srv()
    n_ch, d = 1, 128
    rec = np.full((n_cells * n_ch, d), 255, np.uint8)
    want = (-255 * n_cells) & M32
    with P.PirServer(n_cells, n_ch, d, records=rec) as s:
        qf = np.full(n_cells, M32, np.uint32)
        assert (_u32(s.answer(qf)) == want).all()
        Q = np.full((4, n_cells), M32, np.uint32)
        ans = _u32(s.answer_batch(Q))
        assert (ans == want).all()
        # mixed extreme limbs: 0xFF00FF00 has limbs (0, 255, 0, 255)
        Q2 = np.full((3, n_cells), 0xFF00FF00, np.uint32)
        assert (_u32(s.answer_batch(Q2)) == (255 * 0xFF00FF00 * n_cells) & M32).all()
        assert (_u32(s.answer(Q2[0])) == (255 * 0xFF00FF00 * n_cells) & M32).all()


# ------------------------------------------------------------------ batch (a6)
@pytest.mark.parametrize("B", [1, 3, 8, 64, 65, 200])
def test_answer_batch_small(cuda_ok, B):
    P = _srv()
    n_cells, n_ch, d, m = 1200, 6, 30, 0
    rec, D = _db(n_cells, n_ch, d, m, seed=10)
    Q = synth.uniform_u32_np(11 + B, (B, n_cells))
    want = O.answer_batch(D, Q)
    with P.PirServer(n_cells, n_ch, d, records=rec) as s:
        got = _u32(s.answer_batch(Q))
        assert got.shape == want.shape
        assert (got == want).all()
        # P6: column j of the batch == single answer of query j (host in/out too)
        out = np.empty((B, s.ell_local), np.uint32)
        s.answer_batch(Q, out=out)
        assert (out == want).all()
        j = B // 2
        assert (_u32(s.answer(Q[j])) == got[j]).all()


def test_answer_batch_ragged_shard(cuda_ok):
    P = _srv()
    n_cells, n_ch, d, m = 999, 5, 33, 333
    rec, D = _db(n_cells, n_ch, d, m, seed=12)
    Q = synth.uniform_u32_np(13, (37, m))
    r0, r1 = 31, 401
    with P.PirServer(n_cells, n_ch, d, m=m, row_begin=r0, row_end=r1, records=rec) as s:
        assert (_u32(s.answer_batch(Q)) == O.answer_batch(D[r0:r1], Q)).all()


# ------------------------------------------------------------------ hint (a7)
@pytest.mark.parametrize("n", [4, 9, 64, 1024])
def test_hint_small(cuda_ok, n):
    P = _srv()
    n_cells, n_ch, d = 700, 4, 20
    rec, D = _db(n_cells, n_ch, d, seed=14)
    seed_A = 0xDEADBEEF12345678
    A = O.expand_A(seed_A, n_cells, n)
    want = O.hint(D, A)
    with P.PirServer(n_cells, n_ch, d, lwe_n=n, seed_A=seed_A, records=rec) as s:
        got = _u32(s.hint())
        assert got.shape == want.shape
        assert (got == want).all()
        host = np.empty((s.ell_local, n), np.uint32)
        s.hint(out=host)
        assert (host == want).all()


# ------------------------------------------------------------------ LWE end to end
def test_lwe_end_to_end_tiny_bruteforce(cuda_ok):
    """P1 through the GPU path: hint and answers from the CUDA kernels, queries
    and decode from the oracle client; every one of the 16384 records of the
    tiny DB (BASELINE.json configs[0]) must decode exactly."""
    P = _srv()
    n_cells, n_ch, d, n = 1024, 16, 8, 1024
    rec, D = _db(n_cells, n_ch, d, seed=15)
    seed_A = 77
    A = O.expand_A(seed_A, n_cells, n)
    s_key = O.keygen(78, n)
    Q = np.stack([O.query(A, s_key, 79, c, 6.4, c)[0] for c in range(n_cells)])
    with P.PirServer(n_cells, n_ch, d, lwe_n=n, seed_A=seed_A, records=rec) as s:
        H = _u32(s.hint())
        assert (H == O.hint(D, A)).all()
        ANS = _u32(s.answer_batch(Q))  # all 1024 queries in one batch
        for c in (0, 511, 1023):
            assert (_u32(s.answer(Q[c])) == ANS[c]).all()
    rows = np.arange(n_ch * d, dtype=np.uint64)
    bad = 0
    for c in range(n_cells):
        got = O.decode(ANS[c], H, s_key, rows).reshape(n_ch, d)
        bad += int((got != rec[c * n_ch:(c + 1) * n_ch]).sum())
    assert bad == 0


# ------------------------------------------------------------------ full sizes
def _setup_synth_db(P, n_cells, n_ch, d, seed, chunk_cells=2048, **kw):
    s = P.PirServer(n_cells, n_ch, d, **kw)
    for c0 in range(0, n_cells, chunk_cells):
        nc = min(chunk_cells, n_cells - c0)
        r = synth.records(seed, c0 * n_ch, nc * n_ch, d, n_ch, device="cuda")
        s.db_write(c0 * n_ch, r)
    torch.cuda.synchronize()
    return s


def _sampled_rows(seed, rows, n_cells, n_ch, d):
    """Rows of D (m = n_cells) regenerated from synth, for sampled exact checks."""
    cells = torch.arange(n_cells, dtype=torch.int64)
    out = np.empty((len(rows), n_cells), np.uint8)
    for i, r in enumerate(rows):
        ch, b = divmod(int(r), d)
        out[i] = synth.byte_column(seed, cells * n_ch + ch, b, d, n_ch).numpy()
    return out


def test_c2_regional_full(cuda_ok):
    """BASELINE.json configs[1]: 8192 cells x 40 ch x 3072 B = 1.007 GB, exact
    full answer vs the oracle."""
    P = _srv()
    n_cells, n_ch, d = 8192, 40, 3072
    seed = 21
    s = _setup_synth_db(P, n_cells, n_ch, d, seed)
    rec = synth.records(seed, 0, n_cells * n_ch, d, n_ch, device="cuda").cpu().numpy()
    D = O.pack(rec, n_cells, n_ch, d, n_cells)
    del rec
    qu = synth.uniform_u32_np(22, (n_cells,))
    assert (_u32(s.answer(qu)) == O.answer(D, qu)).all()
    s.close()


@pytest.mark.slow
def test_c3_nationwide_sampled(cuda_ok):
    """configs[2] on one GPU: 262144 cells x 40 x 3072 = 32.2 GB; 48 sampled rows exact."""
    P = _srv()
    n_cells, n_ch, d = 262144, 40, 3072
    seed = 23
    s = _setup_synth_db(P, n_cells, n_ch, d, seed)
    qu = synth.uniform_u32_np(24, (n_cells,))
    got = _u32(s.answer(qu))
    rng = np.random.default_rng(0)
    rows = np.concatenate([[0, 1, s.ell - 1], rng.choice(s.ell, 45, replace=False)])
    Dr = _sampled_rows(seed, rows, n_cells, n_ch, d)
    assert (got[rows] == O.answer(Dr, qu)).all()
    s.close()


def _channel_slab(seed, ch, n_cells, n_ch, d):
    """Rows [ch*d, (ch+1)*d) of D for m = n_cells (one row block, DESIGN R10:
    D[ch*d + b][cell] = rec_{cell*n_ch + ch}[b]), i.e. the transpose of the
    channel's records (synth, generated on the GPU only for speed).  That this
    equals the oracle's pack of a one-channel DB is pinned in
    tests/test_oracle.py::test_one_channel_pack_is_transpose; the oracle's
    element-by-element pack is ~9 s per 201 MB channel, too slow for 40."""
    theta = torch.arange(n_cells, device="cuda", dtype=torch.int64) * n_ch + ch
    rec = synth.records_at(seed, theta, d, n_ch, 512).cpu().numpy()
    return np.ascontiguousarray(rec.T)


@pytest.mark.slow
@pytest.mark.parametrize("B", [64, 256])
def test_c4_batch_sampled(cuda_ok, B):
    """configs[3]: 65536 cells x 40 x 3072 = 8.05 GB, B concurrent queries;
    24 sampled rows exact for all B queries, + 2 columns == single answers,
    + Freivalds (40 rounds over Z_{2^32}, P8 of SURVEY 8(c)) on the FULL ANS:
    ANS^T X == D (Q^T X), channel by channel, both sides exact float64-limb
    products (tests/_exact.py) of the oracle-packed D and the inputs.  For a
    wrong product E != 0 (mod 2^32) a uniform column of X gives E x == 0 with probability <= 1/2, so 40 columns miss with <= 2^-40."""
    P = _srv()
    n_cells, n_ch, d = 65536, 40, 3072
    seed = 25
    s = _setup_synth_db(P, n_cells, n_ch, d, seed)
    Q = synth.uniform_u32_np(26, (B, n_cells))
    ANS = _u32(s.answer_batch(Q))
    rng = np.random.default_rng(1)
    rows = np.concatenate([[0, s.ell - 1], rng.choice(s.ell, 22, replace=False)])
    Dr = _sampled_rows(seed, rows, n_cells, n_ch, d)
    assert (ANS[:, rows] == O.answer_batch(Dr, Q)).all()
    for j in (0, B - 1):
        assert (_u32(s.answer(Q[j])) == ANS[j]).all()
    s.close()
    X = synth.uniform_u32_np(27, (B, 40))             # 40 Freivalds rounds
    left = matmul_mod32(np.ascontiguousarray(ANS.T), X)          # ANS^T X (ell, 40)
    V = np.ascontiguousarray(matmul_mod32(np.ascontiguousarray(Q.T), X).T)  # (Q^T X)^T
    for ch in range(n_ch):
        right = matmul_mod32(_channel_slab(seed, ch, n_cells, n_ch, d), np.ascontiguousarray(V.T))
        assert (left[ch * d:(ch + 1) * d] == right).all(), f"Freivalds fails in channel {ch}"


@pytest.mark.slow
def test_c5_hint_shard_sampled(cuda_ok):
    """configs[4], one rank's shard at G = 8: rows [0, 15360) of the 32 GB DB,
    n = 1024; 64 sampled rows of H exact against the oracle's D.A, and
    Freivalds (40 rounds over Z_{2^32}) on the FULL shard: H X == D (A X)."""
    P = _srv()
    n_cells, n_ch, d, n = 262144, 40, 3072, 1024
    seed, seed_A = 27, 0x5EED
    from paper_2510_03631_b200.dist import shard_rows
    r0, r1 = shard_rows(n_cells, n_ch, d, n_cells, 8, 0)
    assert r0 == 0 and (r1 - r0) % d == 0
    s = _setup_synth_db(P, n_cells, n_ch, d, seed, lwe_n=n, seed_A=seed_A, row_begin=r0, row_end=r1)
    H = _u32(s.hint())
    s.close()
    rng = np.random.default_rng(2)
    rows = np.concatenate([[0, r1 - r0 - 1], rng.choice(r1 - r0, 62, replace=False)])
    Dr = _sampled_rows(seed, rows + r0, n_cells, n_ch, d)
    A = O.expand_A(seed_A, n_cells, n)
    assert (H[rows] == O.hint(Dr, A)).all()
    X = synth.uniform_u32_np(28, (n, 40))
    left = matmul_mod32(H, X)                          # H X (rows, 40)
    AX = matmul_mod32(A, X)                            # A X (m, 40)
    del A
    for ch in range((r1 - r0) // d):
        right = matmul_mod32(_channel_slab(seed, ch, n_cells, n_ch, d), AX)
        assert (left[ch * d:(ch + 1) * d] == right).all(), f"Freivalds fails in channel {ch}"


@pytest.mark.parametrize("stable", [False, True])
@pytest.mark.parametrize("cfg", [dict(), dict(QPIR_GEMV_SPLIT="7"), dict(QPIR_GEMV_PDL="0")])
def test_back_to_back_answers_pdl(cuda_ok, cfg, stable, monkeypatch):
    """Back-to-back GEMVs on one stream overlap under programmatic dependent
    launch; split-K scratch and outputs must not race (every answer exact).
    stable: QPIR_FLAG_STABLE_INPUTS (the queries were written before the loop),
    the whole scan runs before griddepcontrol.wait -- the bench's setting."""
    for k, v in cfg.items():
        monkeypatch.setenv(k, v)
    P = _srv()
    n_cells, n_ch, d = 4096, 8, 64
    rec, D = _db(n_cells, n_ch, d, seed=40)
    Qs = [synth.uniform_u32_np(41 + i, (n_cells,)) for i in range(24)]
    with P.PirServer(n_cells, n_ch, d, records=torch.from_numpy(rec).cuda(),
                     stable_inputs=stable) as s:
        qd = [torch.from_numpy(q.view(np.int32)).cuda() for q in Qs]
        torch.cuda.synchronize()
        same = torch.empty(s.ell_local, dtype=torch.int32, device="cuda")
        outs = []
        for i, q in enumerate(qd):
            if i % 3 == 2:
                s.answer(q, out=same)  # reuse one output buffer (WAW across launches)
            else:
                outs.append((i, s.answer(q)))
        torch.cuda.synchronize()
        for i, o in outs:
            assert (_u32(o) == O.answer(D, Qs[i])).all(), i
        assert (_u32(same) == O.answer(D, Qs[23])).all()


@pytest.mark.parametrize("cfg", [dict(), dict(QPIR_GEMV_SPLIT="1"), dict(QPIR_GEMV_L2PF="1")])
def test_pdl_inputs_written_by_previous_kernel(cuda_ok, cfg, monkeypatch):
    """Programmatic dependent launch hazard (PDL: the next kernel may start
    before the previous one ends, and only its writes are visible after
    griddepcontrol.wait).  No syncs anywhere between the producers and the
    answers: (1) a torch kernel writes qu on the stream right before each of
    1000 answers; (2) each answer's query is the previous GEMV's output
    (GEMV -> GEMV on one stream, the case where the producer triggers its
    dependents early); (3) a device-side db_write (pack kernel writes D) is
    followed at once by an answer.  Every result must be exact."""
    for k, v in cfg.items():
        monkeypatch.setenv(k, v)
    P = _srv()
    n_cells, n_ch, d = 2048, 1, 2048  # ell = m = 2048: an answer can be the next query
    rec, D = _db(n_cells, n_ch, d, seed=95)
    base = synth.uniform_u32_np(96, (n_cells,))
    keys = torch.arange(1000, dtype=torch.int32, device="cuda") * 0x9E3779B1
    with P.PirServer(n_cells, n_ch, d, records=torch.from_numpy(rec).cuda()) as s:
        assert s.ell_local == n_cells
        qb = torch.from_numpy(base.view(np.int32)).cuda()
        qd = torch.empty_like(qb)
        outs = torch.empty((1000, s.ell_local), dtype=torch.int32, device="cuda")
        for i in range(1000):
            torch.bitwise_xor(qb, keys[i], out=qd)  # kernel writes qu, then the answer
            s.answer(qd, out=outs[i])
        # chain: query i+1 = answer i
        chain = torch.empty((8, s.ell_local), dtype=torch.int32, device="cuda")
        s.answer(qb, out=chain[0])
        for i in range(1, 8):
            s.answer(chain[i - 1], out=chain[i])
        # device db_write immediately followed by an answer (no sync)
        rec2 = rec.copy()
        rec2[::7] ^= 0x3C
        s.db_write(0, torch.from_numpy(rec2).cuda())
        after = s.answer(qb)
        torch.cuda.synchronize()
        o = _u32(outs)
        kk = keys.cpu().numpy().view(np.uint32)
        want = O.answer_batch(D, base[None, :] ^ kk[:, None])
        bad = np.nonzero((o != want).any(1))[0]
        assert bad.size == 0, f"answers {bad[:10]} wrong"
        c = _u32(chain)
        q = base
        for i in range(8):
            q = O.answer(D, q)
            assert (c[i] == q).all(), i
        assert (_u32(after) == O.answer(O.pack(rec2, n_cells, n_ch, d, n_cells), base)).all()


def test_concurrent_streams_have_private_scratch(cuda_ok, monkeypatch):
    """Calls on different streams of one context use per-stream arenas (host-query
    staging, split-K partials, tickets, limb planes): interleaved answers and
    batches on two streams must all be exact."""
    monkeypatch.setenv("QPIR_GEMV_SPLIT", "6")
    P = _srv()
    n_cells, n_ch, d = 3000, 6, 40
    rec, D = _db(n_cells, n_ch, d, seed=50)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    with P.PirServer(n_cells, n_ch, d, records=rec) as s:
        jobs = []
        for i in range(16):
            st = streams[i % 2]
            if i % 4 == 3:
                Q = synth.uniform_u32_np(60 + i, (5, n_cells))
                pin = torch.from_numpy(Q.view(np.int32)).pin_memory()
                out = torch.empty((5, s.ell_local), dtype=torch.int32, device="cuda")
                s.answer_batch(pin, out=out, stream=st)
                jobs.append((out, O.answer_batch(D, Q), pin))
            else:
                q = synth.uniform_u32_np(60 + i, (n_cells,))
                pin = torch.from_numpy(q.view(np.int32)).pin_memory()
                out = torch.empty(s.ell_local, dtype=torch.int32, device="cuda")
                s.answer(pin, out=out, stream=st)  # async H2D into the stream's arena
                jobs.append((out, O.answer(D, q), pin))
        torch.cuda.synchronize()
        for out, want, _ in jobs:
            assert (_u32(out) == want).all()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("n_cells", [16384, 16768])
def test_lockstep_gemms_on_concurrent_streams(cuda_ok, monkeypatch, n_cells):
    """The tcgen05 engine's K-lockstep (CTAs of a wave wait for the slowest
    arrived CTA) with two hints and a batch running at once on three streams, so
    that some CTAs of each grid are not resident while others spin: no deadlock,
    every result exact; chunk sizes 1 and 16 K-blocks; 16768 cells = 131 K-blocks,
    so the last K-split is shorter and credits its missing chunks."""
    P = _srv()
    n_ch, d, n = 2, 24, 256  # 16384 cells: G = 1024 groups, 128 K-blocks; N = 1024
    rec, D = _db(n_cells, n_ch, d, seed=91)
    A = O.expand_A(5, n_cells, n)
    Hw = O.hint(D, A)
    Q = synth.uniform_u32_np(92, (128, n_cells))
    want = O.answer_batch(D, Q)
    for ls in ("1", "16"):
        monkeypatch.setenv("QPIR_MMA_LOCKSTEP", ls)
        with P.PirServer(n_cells, n_ch, d, lwe_n=n, seed_A=5, records=rec) as s:
            sts = [torch.cuda.Stream() for _ in range(3)]
            Qd = torch.from_numpy(Q.view(np.int32)).cuda()
            outs = []
            for rep in range(3):
                h1 = s.hint(stream=sts[0])
                h2 = s.hint(stream=sts[1])
                b = s.answer_batch(Qd, stream=sts[2])
                outs.append((h1, h2, b))
            torch.cuda.synchronize()
            for h1, h2, b in outs:
                assert (_u32(h1) == Hw).all() and (_u32(h2) == Hw).all()
                assert (_u32(b) == want).all()


def test_host_input_ring_grows_and_reuses(cuda_ok):
    """Host (pinned and pageable) queries go through the arena's copy stream and
    two-slot staging ring: batches of growing B (forcing slot reallocation while
    earlier kernels may still read the other slot) and answers interleaved on
    one stream without syncs -- all exact."""
    P = _srv()
    n_cells, n_ch, d = 2000, 5, 24
    rec, D = _db(n_cells, n_ch, d, seed=81)
    st = torch.cuda.Stream()
    with P.PirServer(n_cells, n_ch, d, records=rec) as s:
        jobs = []
        for i, B in enumerate([1, 3, 2, 9, 4, 17, 17, 5]):
            Q = synth.uniform_u32_np(900 + i, (B, n_cells))
            src = torch.from_numpy(Q.view(np.int32))
            src = src.pin_memory() if i % 2 == 0 else src  # pinned / pageable
            out = torch.empty((B, s.ell_local), dtype=torch.int32, device="cuda")
            s.answer_batch(src, out=out, stream=st)
            jobs.append((out, O.answer_batch(D, Q), src))
            q = synth.uniform_u32_np(950 + i, (n_cells,))
            qs = torch.from_numpy(q.view(np.int32))
            qs = qs.pin_memory() if i % 3 else qs
            o1 = torch.empty(s.ell_local, dtype=torch.int32, device="cuda")
            s.answer(qs, out=o1, stream=st)
            jobs.append((o1, O.answer(D, q), qs))
        st.synchronize()
        for out, want, _ in jobs:
            assert (_u32(out) == want).all()


def test_cuda_graph_capture_and_replay(cuda_ok):
    """The C-ABI calls are capturable into a CUDA graph once a first eager call
    has sized the stream's scratch: answers (split-K GEMV with PDL edges) and a
    tcgen05 batch captured, replayed twice with the query buffers rewritten in
    place between replays -- every output exact."""
    P = _srv()
    n_cells, n_ch, d = 3000, 6, 40
    rec, D = _db(n_cells, n_ch, d, seed=71)
    st = torch.cuda.Stream()
    with P.PirServer(n_cells, n_ch, d, records=rec) as s:
        qd = [torch.empty(n_cells, dtype=torch.int32, device="cuda") for _ in range(6)]
        Qd = torch.empty((5, n_cells), dtype=torch.int32, device="cuda")
        outs = [torch.empty(s.ell_local, dtype=torch.int32, device="cuda") for _ in range(6)]
        outB = torch.empty((5, s.ell_local), dtype=torch.int32, device="cuda")
        with torch.cuda.stream(st):  # eager first: sizes the stream's arena
            s.answer(qd[0], out=outs[0], stream=st)
            s.answer_batch(Qd, out=outB, stream=st)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st, capture_error_mode="relaxed"):
            for i in range(6):
                s.answer(qd[i], out=outs[i], stream=st)
            s.answer_batch(Qd, out=outB, stream=st)
        for rep in range(2):
            qs = [synth.uniform_u32_np(700 + 10 * rep + i, (n_cells,)) for i in range(6)]
            Q = synth.uniform_u32_np(800 + rep, (5, n_cells))
            for i in range(6):
                qd[i].copy_(torch.from_numpy(qs[i].view(np.int32)))
            Qd.copy_(torch.from_numpy(Q.view(np.int32)))
            torch.cuda.synchronize()
            with torch.cuda.stream(st):
                g.replay()
            st.synchronize()
            for i in range(6):
                assert (_u32(outs[i]) == O.answer(D, qs[i])).all(), (rep, i)
            assert (_u32(outB) == O.answer_batch(D, Q)).all(), rep


def test_errors_name_the_field(cuda_ok):
    """Lengths, alignment and foreign pointers are rejected with the field named
    and nothing written (QPIR_E_DIMENSION / QPIR_E_PARAM)."""
    P = _srv()
    from paper_2510_03631_b200 import _lib as L
    n_cells, n_ch, d = 512, 2, 16
    rec, D = _db(n_cells, n_ch, d, seed=70)
    with P.PirServer(n_cells, n_ch, d, records=rec) as s:
        with pytest.raises(P.QpirError) as ei:
            s.answer(np.zeros(n_cells - 1, np.uint32))
        assert ei.value.code == L.QPIR_E_DIMENSION and "m:" in str(ei.value)
        raw = torch.zeros(4 * n_cells + 4, dtype=torch.uint8, device="cuda")
        out = torch.empty(s.ell_local, dtype=torch.int32, device="cuda")
        rc = L._L.qpir_answer(s._ctx, raw.data_ptr() + 1, n_cells, out.data_ptr(), s.ell_local,
                              None)
        with pytest.raises(P.QpirError) as ei:
            L._check(rc, s._ctx)
        assert ei.value.code == L.QPIR_E_PARAM and "aligned" in str(ei.value)
        with pytest.raises(P.QpirError) as ei:
            s.answer_batch(np.zeros((0, n_cells), np.uint32))
        assert ei.value.code == L.QPIR_E_PARAM and "B:" in str(ei.value)
        # the context is still usable after errors
        q = synth.uniform_u32_np(71, (n_cells,))
        assert (_u32(s.answer(q)) == O.answer(D, q)).all()


@pytest.mark.slow
def test_next_rows_full_size_sampled(cuda_ok):
    """configs[1]-sized record set (327680 paper-shaped 3 KB records = 1.007 GB):
    FTR (3-limb tcgen05, mod 65537) and the bit-plane tensor-core ENS batch, every
    query exact on 24 sampled record-byte columns (the oracle on those columns)."""
    P = _srv()
    n_cells, n_ch, d = 8192, 40, 3072
    r = n_cells * n_ch
    seed = 81
    rec_dev = synth.records(seed, 0, r, d, n_ch, device="cuda")
    rng = np.random.default_rng(3)
    cols = np.sort(np.concatenate([[0, 13, 596, d - 1], rng.choice(d, 20, replace=False)]))
    rec_cols = rec_dev[:, torch.from_numpy(cols).cuda()].cpu().numpy()
    with P.FtrServer(r, d, records=rec_dev) as f:
        Q = synth.uniform_u32_np(82, (16, r)) % 65537
        got = P.u32(f.answer_batch(Q))[:, cols]
        assert (got == O.ftr_respond_batch(rec_cols, Q)).all()
    with P.EnsServer(r, d, records=rec_dev) as e:
        nb = (r + 7) // 8
        Qs = synth.uniform_u8_np(83, (48, nb))
        got = e.answer_batch(Qs).cpu().numpy()[:, cols]
        assert (got == O.ens_respond_batch(rec_cols, Qs)).all()


@pytest.mark.parametrize("split", ["0", "3"])
def test_limb_chunking_batch_and_hint(cuda_ok, split, monkeypatch):
    """A 1 MB limb budget forces Q' (queries) and A' (hint columns) to be built and
    multiplied in chunks; results are unchanged (strided hint chunks with K-splits
    add into a pre-zeroed H)."""
    monkeypatch.setenv("QPIR_LIMB_BUDGET_MB", "1")
    monkeypatch.setenv("QPIR_MMA_SPLIT", split)
    P = _srv()
    n_cells, n_ch, d, n = 4096, 3, 40, 300
    rec, D = _db(n_cells, n_ch, d, seed=90)
    with P.PirServer(n_cells, n_ch, d, lwe_n=n, seed_A=91, records=rec) as s:
        Q = synth.uniform_u32_np(92, (150, n_cells))   # 600 limb cols x 4096 > 1 MB
        assert (_u32(s.answer_batch(Q)) == O.answer_batch(D, Q)).all()
        want = ((Q.astype(object) @ D.T.astype(object)) % 65537).astype(np.uint32)
        assert (_u32(s.answer_batch_modp(Q, 65537)) == want).all()
        assert (_u32(s.hint()) == O.hint(D, O.expand_A(91, n_cells, n))).all()
