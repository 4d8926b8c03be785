"""GPU parity for QPADL-ENS (Chor XOR PIR, NEXT-1) through the C ABI against
the oracle (bit-exact bytes)."""
import numpy as np
import pytest
import torch

import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _P():
    import paper_2510_03631_b200 as P
    return P


def _share(seed, r):
    q = synth.uniform_u8_np(seed, ((r + 7) // 8,))
    if r % 8:
        q[-1] &= (1 << (r % 8)) - 1
    return q


@pytest.mark.parametrize("r,d", [(1000, 24), (77, 5), (4099, 100), (513, 3072), (20000, 16),
                                 (3001, 2500), (100, 16384)])
@pytest.mark.parametrize("rows,group,wide", [("0", "0", "1"), ("8", "0", "1"), ("8", "3", "1"),
                                             ("8", "1", "1"), ("96", "0", "1"), ("0", "0", "0"),
                                             ("64", "5", "0"), ("0", "0", "2"), ("32", "2", "2")])
def test_ens_answer_matches_oracle(cuda_ok, r, d, rows, group, wide, monkeypatch):
    monkeypatch.setenv("QPIR_ENS_ROWS", rows)
    monkeypatch.setenv("QPIR_ENS_GROUP", group)
    monkeypatch.setenv("QPIR_ENS_WIDE", wide)
    P = _P()
    rec = synth.uniform_u8_np(r + d, (r, d))
    with P.EnsServer(r, d, records=rec) as s:
        nb = (r + 7) // 8
        assert (s.answer(np.zeros(nb, np.uint8)).cpu().numpy() == 0).all()
        for j in (0, r // 2, r - 1):
            e = np.zeros(nb, np.uint8)
            e[j >> 3] = 1 << (j & 7)
            assert (s.answer(e).cpu().numpy() == rec[j]).all()
        for seed in (1, 2):
            q = _share(seed, r)
            want = O.ens_respond(rec, q)
            out = np.empty(d, np.uint8)
            s.answer(q, out=out)  # host in / host out
            assert (out == want).all()
            got = s.answer(torch.from_numpy(q).cuda())  # device in / device out
            assert (got.cpu().numpy() == want).all()


@pytest.mark.parametrize("B", [1, 7, 64, 128, 130, 256, 300])
@pytest.mark.parametrize("tc", ["0", "1", "ss"])
def test_ens_batch_matches_oracle(cuda_ok, B, tc, monkeypatch):
    """tc = 1: GF(2) product on tcgen05 with the bit-rows in TMEM (A operand
    written by tcgen05.st, ens_mma.cuh TS form; units of 128 shares x 32 record
    bytes, B > 128: several share tiles); tc = ss: the shared-memory form (B <=
    128: one share tile x 64 record bytes per unit, B > 128: two share tiles x
    32 bytes); tc = 0: CUDA-core predicated-XOR kernel."""
    monkeypatch.setenv("QPIR_ENS_TC", "0" if tc == "0" else "1")
    monkeypatch.setenv("QPIR_ENS_TS", "0" if tc == "ss" else "1")
    P = _P()
    r, d = 3001, 200
    rec = synth.uniform_u8_np(5, (r, d))
    Q = np.stack([_share(100 + b, r) for b in range(B)])
    want = O.ens_respond_batch(rec, Q)
    with P.EnsServer(r, d, records=torch.from_numpy(rec).cuda()) as s:
        got = s.answer_batch(Q).cpu().numpy()
        assert s.last_path == ("cuda_cores" if tc == "0" else "tensor")
        assert (got == want).all()
        assert (s.answer(Q[B // 2]).cpu().numpy() == want[B // 2]).all()
        assert s.last_path == "scan"


@pytest.mark.parametrize("ts", ["1", "0"])
def test_ens_tc_extreme_bits(cuda_ok, ts, monkeypatch):
    """Tensor-core path on all-0xFF records and all-ones shares: every bit-row
    count is r (accumulated as r * 2^i for bit i, up to r * 128), so the
    response is all-ones iff r is odd -- each weight 2^0..2^7 must land on its
    own bit; then unit shares return single records exactly."""
    monkeypatch.setenv("QPIR_ENS_TC", "1")
    monkeypatch.setenv("QPIR_ENS_TS", ts)
    P = _P()
    for r in (4097, 4096):
        d = 77
        rec = np.full((r, d), 0xFF, np.uint8)
        nb = (r + 7) // 8
        ones = np.full((40, nb), 0xFF, np.uint8)
        if r % 8:
            ones[:, -1] = (1 << (r % 8)) - 1
        with P.EnsServer(r, d, records=rec) as s:
            got = s.answer_batch(ones).cpu().numpy()
            assert (got == (0xFF if r % 2 else 0)).all()
        rec = synth.uniform_u8_np(r, (r, d))
        units = np.zeros((40, nb), np.uint8)
        idx = np.linspace(0, r - 1, 40).astype(int)
        units[np.arange(40), idx >> 3] = (1 << (idx & 7)).astype(np.uint8)
        with P.EnsServer(r, d, records=rec) as s:
            assert (s.answer_batch(units).cpu().numpy() == rec[idx]).all()


def test_ens_bruteforce_reconstruct(cuda_ok):
    """Lemma 1: XOR of the l GPU responses == record theta, every theta."""
    P = _P()
    r, d, l = 384, 40, 3
    rec = synth.uniform_u8_np(6, (r, d))
    with P.EnsServer(r, d, records=rec) as s:
        shares = np.concatenate([O.ens_query(t, r, l, 500 + t) for t in range(r)])  # (r*l, nb)
        resp = s.answer_batch(shares).cpu().numpy().reshape(r, l, d)
    for t in range(r):
        assert (O.ens_reconstruct(resp[t]) == rec[t]).all()


@pytest.mark.parametrize("ts", ["1", "0"])
@pytest.mark.parametrize("split", ["0", "3"])
def test_ens_tc_ragged_and_split(cuda_ok, split, ts, monkeypatch):
    """Ragged r / d (d not a multiple of 16, r not of 128) and forced K-splits
    (parities combined with atomicXor) on the tensor-core path."""
    monkeypatch.setenv("QPIR_ENS_TC", "1")
    monkeypatch.setenv("QPIR_ENS_TS", ts)
    monkeypatch.setenv("QPIR_MMA_SPLIT", split)
    P = _P()
    for r, d, B in [(70001, 5, 33), (1000, 37, 40), (4097, 3072, 17)]:
        rec = synth.uniform_u8_np(r * 3 + d, (r, d))
        Q = np.stack([_share(700 + b, r) for b in range(B)])
        with P.EnsServer(r, d, records=rec) as s:
            assert (s.answer_batch(Q).cpu().numpy() == O.ens_respond_batch(rec, Q)).all()
            # DB update invalidates the bit-planes
            rec2 = rec.copy()
            rec2[5] ^= 0xFF
            s.db_write(5, rec2[5:6])
            assert (s.answer_batch(Q).cpu().numpy() == O.ens_respond_batch(rec2, Q)).all()


@pytest.mark.parametrize("tc", ["0", "1"])
def test_ens_mutation_one_byte_is_detected(cuda_ok, tc, monkeypatch):
    """SURVEY 5 mutation test for ENS: flip bits of one byte of record t via
    db_write; a response whose share selects t changes in exactly that byte (by
    exactly the flipped bits), one that does not select t is unchanged."""
    monkeypatch.setenv("QPIR_ENS_TC", tc)
    P = _P()
    r, d, t, b, flip = 4099, 100, 1234, 57, 0x21
    rec = synth.uniform_u8_np(61, (r, d))
    Q = np.stack([_share(62 + i, r) for i in range(40)])
    sel = (Q[:, t >> 3] >> (t & 7)) & 1
    assert sel.any() and not sel.all()
    with P.EnsServer(r, d, records=rec) as s:
        before = s.answer_batch(Q).cpu().numpy()
        assert (before == O.ens_respond_batch(rec, Q)).all()
        bad = rec[t].copy()
        bad[b] ^= flip
        s.db_write(t, bad[None, :])
        after = s.answer_batch(Q).cpu().numpy()
    delta = before ^ after
    assert (delta[sel == 0] == 0).all()
    assert (delta[sel == 1][:, b] == flip).all()
    delta[:, b] = 0
    assert (delta == 0).all()


def test_ens_db_write_and_c2_scale(cuda_ok):
    """configs[1]-sized ENS DB (327680 paper-shaped 3 KB records = 1.007 GB)."""
    P = _P()
    n_cells, n_ch, d = 8192, 40, 3072
    r = n_cells * n_ch
    with P.EnsServer(r, d) as s:
        chunk = 65536
        for t0 in range(0, r, chunk):
            s.db_write(t0, synth.records(31, t0, min(chunk, r - t0), d, n_ch, device="cuda"))
        rec = synth.records(31, 0, r, d, n_ch, device="cuda").cpu().numpy()
        q = _share(32, r)
        assert (s.answer(q).cpu().numpy() == O.ens_respond(rec, q)).all()
        Q = np.stack([_share(40 + b, r) for b in range(3)])
        assert (s.answer_batch(Q).cpu().numpy() == O.ens_respond_batch(rec, Q)).all()


@pytest.mark.parametrize("r,d", [(20000, 3072), (50000, 64), (4099, 100)])
@pytest.mark.parametrize("pdl,stable", [("1", False), ("0", False), ("1", True)])
def test_ens_oop_back_to_back_no_sync(cuda_ok, r, d, pdl, stable, monkeypatch):
    """Single-share answers and OOP online answers queued back to back on one
    stream (programmatic dependent launch lets each scan start while the previous
    one drains; the in-kernel finaliser re-zeroes the accumulator): every
    response still equals the oracle's."""
    monkeypatch.setenv("QPIR_ENS_PDL", pdl)
    P = _P()
    rec = synth.uniform_u8_np(r + d + 7, (r, d))
    n = 4
    k = r // n
    rec = rec[: k * n]
    r = k * n
    shares = [_share(100 + i, r) for i in range(6)]
    qs = [_share(200 + i, k) for i in range(6)]
    As = [synth.uniform_u8_np(300 + i, (d,)) for i in range(6)]
    with P.EnsServer(r, d, records=rec, stable_inputs=stable) as s:
        st = torch.cuda.Stream()
        dev = [torch.from_numpy(x).cuda() for x in shares]
        dq = [torch.from_numpy(x).cuda() for x in qs]
        dA = [torch.from_numpy(x).cuda() for x in As]
        torch.cuda.synchronize()
        outs = []
        for i in range(6):
            outs.append(s.answer(dev[i], stream=st))
            outs.append(s.oop_answer(n, i % n, dq[i], dA[i], stream=st))
        st.synchronize()
        for i in range(6):
            assert (outs[2 * i].cpu().numpy() == O.ens_respond(rec, shares[i])).all(), i
            want = O.oop_respond(rec, n, i % n, qs[i], As[i])
            assert (outs[2 * i + 1].cpu().numpy() == want).all(), i


def test_ens_oop_cuda_graph(cuda_ok):
    """Single-share ENS and OOP online answers captured into a CUDA graph (PDL
    edges, in-kernel finalisation) and replayed with new shares: exact."""
    P = _P()
    r, d, n = 8000, 3072, 4
    k = r // n
    rec = synth.uniform_u8_np(31, (r, d))
    st = torch.cuda.Stream()
    with P.EnsServer(r, d, records=rec) as s:
        sh = torch.empty((r + 7) // 8, dtype=torch.uint8, device="cuda")
        q = torch.empty((k + 7) // 8, dtype=torch.uint8, device="cuda")
        A = torch.empty(d, dtype=torch.uint8, device="cuda")
        o1 = torch.empty(d, dtype=torch.uint8, device="cuda")
        o2 = torch.empty(d, dtype=torch.uint8, device="cuda")
        with torch.cuda.stream(st):
            s.answer(sh, out=o1, stream=st)
            s.oop_answer(n, 1, q, A, out=o2, stream=st)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st, capture_error_mode="relaxed"):
            s.answer(sh, out=o1, stream=st)
            s.oop_answer(n, 1, q, A, out=o2, stream=st)
        for rep in range(2):
            share, qq = _share(40 + rep, r), _share(50 + rep, k)
            AA = synth.uniform_u8_np(60 + rep, (d,))
            sh.copy_(torch.from_numpy(share))
            q.copy_(torch.from_numpy(qq))
            A.copy_(torch.from_numpy(AA))
            torch.cuda.synchronize()
            with torch.cuda.stream(st):
                g.replay()
            st.synchronize()
            assert (o1.cpu().numpy() == O.ens_respond(rec, share)).all(), rep
            assert (o2.cpu().numpy() == O.oop_respond(rec, n, 1, qq, AA)).all(), rep
