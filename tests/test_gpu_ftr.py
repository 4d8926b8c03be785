"""GPU parity for QPADL-FTR (Goldberg PIR over F_p, NEXT-2): the tcgen05 limb
GEMM with the mod-p epilogue (qpir_answer_batch_modp) against the oracle."""
import numpy as np
import pytest
import torch

import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu
P = 65537


def _P():
    import paper_2510_03631_b200 as Pk
    return Pk


@pytest.mark.parametrize("r,s,B", [(700, 33, 1), (1000, 24, 5), (3001, 200, 64), (70000, 16, 9),
                                   (5000, 300, 128), (2000, 40, 129), (9000, 20, 300)])
@pytest.mark.parametrize("fuse,split", [("1", "0"), ("0", "0"), ("1", "5")])
def test_ftr_batch_matches_oracle(cuda_ok, r, s, B, fuse, split, monkeypatch):
    """FTR batch vs the oracle; fuse = 1: the 2-limb split runs in the GEMM's
    converter warps (any CTA converts any K-block, flags per K-block), with auto
    or forced K-splits; B > 128 spans several N tiles of the limb operand."""
    monkeypatch.setenv("QPIR_FTR_FUSE", fuse)
    monkeypatch.setenv("QPIR_MMA_SPLIT", split)
    Pk = _P()
    rec = synth.uniform_u8_np(r + s, (r, s))
    Q = synth.uniform_u32_np(B + 3, (B, r)) % P
    want = O.ftr_respond_batch(rec, Q)
    with Pk.FtrServer(r, s, records=rec) as srv:
        got = Pk.u32(srv.answer_batch(Q))
        assert got.shape == want.shape
        assert (got == want).all()
        assert (Pk.u32(srv.answer(torch.from_numpy(Q[0].view(np.int32)).cuda())) == want[0]).all()


def test_ftr_any_u32_and_other_primes(cuda_ok):
    """Exact for any u32 query entries and any modulus: compare with int64 numpy."""
    Pk = _P()
    r, s = 70001, 8  # > 66051 cells: forces several exact K-splits
    rec = np.full((r, s), 255, np.uint8)
    rec[::7] = synth.uniform_u8_np(9, rec[::7].shape)
    Q = synth.uniform_u32_np(10, (3, r))
    for p in (2, 65537, 2147483647, 4294967291):
        want = ((Q.astype(object) @ rec.astype(object)) % p).astype(np.uint32)
        with Pk.FtrServer(r, s, p=p, records=rec) as srv:
            assert (Pk.u32(srv.answer_batch(Q)) == want).all(), p


def test_ftr_end_to_end_reconstruct(cuda_ok):
    """Lemma 1: Lagrange interpolation of t + 1 GPU responses recovers record theta."""
    Pk = _P()
    r, s, l, t = 512, 40, 4, 2
    rec = synth.uniform_u8_np(11, (r, s))
    thetas = [0, 17, 255, 511]
    Q = np.concatenate([O.ftr_query(th, r, l, t, seed=50 + th) for th in thetas])  # (len*l, r)
    with Pk.FtrServer(r, s, records=rec) as srv:
        resp = Pk.u32(srv.answer_batch(Q)).reshape(len(thetas), l, s)
    for i, th in enumerate(thetas):
        got = O.ftr_reconstruct(resp[i][1:t + 2], [2, 3, 4])  # servers 2..4
        assert (got == rec[th]).all()


@pytest.mark.parametrize("fuse", ["1", "0"])
def test_ftr_two_limb_exceptions(cuda_ok, fuse, monkeypatch):
    """p <= 65537 runs on 2 byte limbs; for p = 65537 the residue 65536 is the one
    value 2 limbs cannot hold and goes through the exception list (cap entries per
    query) or, past the cap, the rescan path.  Exact in every case, with the
    limb split fused into the GEMM (converter warps, fuse = 1) or as its own
    kernel (fuse = 0)."""
    monkeypatch.setenv("QPIR_FTR_FUSE", fuse)
    Pk = _P()
    r, s = 70001, 8  # 2 K-splits; cap = 64 + 4 * ceil-ish(r / p) = 72
    rec = synth.uniform_u8_np(21, (r, s))
    cap = 64 + 4 * ((r + 65536) // 65537)
    Q = synth.uniform_u32_np(22, (5, r))
    rng = np.random.default_rng(23)
    for b, n_exc in enumerate([cap, cap + 1, int(0.3 * r)]):
        cols = rng.choice(r, n_exc, replace=False)
        k = rng.integers(0, 65535, n_exc, dtype=np.uint64)  # raw u32 with residue 65536
        Q[b, cols] = (65536 + k * 65537).astype(np.uint32)
    Q[3, :] = 65536  # every entry
    for p in (65537, 65521, 257, 65536):
        want = ((Q % p).astype(np.int64) @ rec.astype(np.int64)) % p
        with Pk.FtrServer(r, s, p=p, records=rec) as srv:
            got = Pk.u32(srv.answer_batch(Q))
        assert (got == want.astype(np.uint32)).all(), p


def test_ftr_and_batches_back_to_back(cuda_ok):
    """FTR (2-limb, exception lists, growing and shrinking batch sizes) and LWE
    batches queued back to back on one stream with no syncs and a hint in
    between: every result exact."""
    Pk = _P()
    r, s = 70001, 12
    rec = synth.uniform_u8_np(41, (r, s))
    st = torch.cuda.Stream()
    with Pk.FtrServer(r, s, records=rec) as srv:
        jobs = []
        for i, B in enumerate([5, 64, 3, 128, 7, 64]):
            Q = synth.uniform_u32_np(600 + i, (B, r))
            Q[0, i * 10:i * 10 + 40] = 65536 + 65537 * i  # residue 65536 entries
            Qd = torch.from_numpy(Q.view(np.int32)).cuda()
            if i % 2:
                out = srv.answer_batch(Qd, stream=st)
                want = ((Q % P).astype(np.int64) @ rec.astype(np.int64)) % P
            else:
                out = srv.server.answer_batch(Qd, stream=st)  # plain LWE batch, mod 2^32
                want = (Q.astype(np.uint64) @ rec.astype(np.uint64)) & 0xFFFFFFFF
            jobs.append((out, want.astype(np.uint32), Qd))
            if i == 2:
                jobs.append((srv.server.hint(stream=st), None, None))
        st.synchronize()
        for out, want, _ in jobs:
            if want is not None:
                assert (Pk.u32(out) == want).all()


@pytest.mark.timeout(300, method="thread")  # a hang must end the process, not the box
def test_ftr_captured_in_cuda_graph(cuda_ok):
    """An FTR batch captured into a CUDA graph (after an eager call sized the
    stream's scratch) replays exactly with the queries rewritten in place: the
    library takes the split-kernel form under capture, because the fused form's
    converter counter and K-block epochs advance on the host per launch (a
    replayed fused capture would wait on stale flags)."""
    Pk = _P()
    r, s, B = 20000, 40, 64
    rec = synth.uniform_u8_np(77, (r, s))
    st = torch.cuda.Stream()
    with Pk.FtrServer(r, s, records=rec) as srv:
        Qd = torch.empty((B, r), dtype=torch.int32, device="cuda")
        out = torch.empty((B, srv.server.ell_local), dtype=torch.int32, device="cuda")
        with torch.cuda.stream(st):
            srv.answer_batch(Qd.zero_(), out=out, stream=st)  # eager: fused form, sizes the arena
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st, capture_error_mode="relaxed"):
            srv.answer_batch(Qd, out=out, stream=st)
        for rep in range(3):
            Q = synth.uniform_u32_np(900 + rep, (B, r))
            Q[rep, :50] = 65536  # residue 65536: the exception list
            Qd.copy_(torch.from_numpy(Q.view(np.int32)))
            torch.cuda.synchronize()
            with torch.cuda.stream(st):
                g.replay()
            st.synchronize()
            want = ((Q % P).astype(np.int64) @ rec.astype(np.int64)) % P
            assert (Pk.u32(out) == want.astype(np.uint32)).all(), rep
        # eager calls after the capture still take the fused form and stay exact
        Q = synth.uniform_u32_np(999, (B, r))
        res = srv.answer_batch(torch.from_numpy(Q.view(np.int32)).cuda(), stream=st)
        st.synchronize()
        got = Pk.u32(res)
        assert (got == (((Q % P).astype(np.int64) @ rec.astype(np.int64)) % P).astype(np.uint32)).all()


@pytest.mark.parametrize("l,t", [(5, 1), (7, 2), (9, 2)])
def test_ftr_byzantine_responses_decoded(cuda_ok, l, t):
    """nu-Byzantine robustness (Lemma 1 proof P:1227):
    nu = floor((l - t - 1) / 2) of the l GPU responses are corrupted (a faulty
    or malicious server adds garbage); Berlekamp-Welch decoding (oracle client)
    of the GPU responses still returns record theta exactly and names exactly the
    corrupted servers.  The paper's Guruswami-Sudan list decoder would tolerate
    nu < l - floor(sqrt(l t)) (e.g. l = 9, t = 2: 5 vs 3 here; DESIGN R21)."""
    Pk = _P()
    r, s = 3001, 96
    nu = (l - t - 1) // 2
    rec = synth.uniform_u8_np(31 + l, (r, s))
    thetas = [0, 1500, r - 1]
    Q = np.concatenate([O.ftr_query(th, r, l, t, seed=70 + th) for th in thetas])
    with Pk.FtrServer(r, s, records=rec) as srv:
        resp = Pk.u32(srv.answer_batch(Q)).reshape(len(thetas), l, s)
    assert (resp.reshape(-1, s) == O.ftr_respond_batch(rec, Q)).all()
    rng = np.random.default_rng(l * 10 + t)
    al = np.arange(1, l + 1)
    for i, th in enumerate(thetas):
        bad_srv = rng.choice(l, nu, replace=False)
        corrupted = resp[i].copy()
        for j in bad_srv:
            corrupted[j] = (corrupted[j] + rng.integers(1, P, s)) % P
        got, flagged = O.ftr_decode(corrupted, al, t)
        assert (got == rec[th]).all()
        assert set(np.nonzero(flagged)[0]) == set(bad_srv)
        # plain Lagrange on the same corrupted set is wrong (the decoder is needed)
        if nu:
            assert (O.ftr_reconstruct(corrupted, al) != rec[th]).any()
