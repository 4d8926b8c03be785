"""Device glue of the multi-GPU layer with a one-rank NCCL group (the pool gives
one GPU per call; multi-rank combining logic is covered by test_dist_gloo.py)."""
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture
def nccl1(cuda_ok):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_distributed_pir_ens_ftr_one_rank(nccl1):
    from paper_2510_03631_b200.dist import DistributedEns, DistributedFtr, DistributedPIR
    n_cells, n_ch, d = 1024, 8, 24
    rec = synth.uniform_u8_np(3, (n_cells * n_ch, d))
    D = O.pack(rec, n_cells, n_ch, d, n_cells)
    pir = DistributedPIR(n_cells, n_ch, d, records=torch.from_numpy(rec).cuda())
    qu = synth.uniform_u32_np(4, (n_cells,))
    got = pir.answer(torch.from_numpy(qu.view(np.int32)).cuda())
    assert (got.cpu().numpy().view(np.uint32) == O.answer(D, qu)).all()
    Q = synth.uniform_u32_np(5, (3, n_cells))
    got = pir.answer_batch(torch.from_numpy(Q.view(np.int32)).cuda())
    assert (got.cpu().numpy().view(np.uint32) == O.answer_batch(D, Q)).all()
    qs = [torch.from_numpy(synth.uniform_u32_np(20 + i, (n_cells,)).view(np.int32)).cuda()
          for i in range(7)]
    many = pir.answer_many(qs)
    torch.cuda.synchronize()
    for i, a in enumerate(many):
        assert (a.cpu().numpy().view(np.uint32) == O.answer(D, qs[i].cpu().numpy().view(np.uint32))).all()

    r = rec.shape[0]
    ens = DistributedEns(r, d, records=torch.from_numpy(rec).cuda())
    share = synth.uniform_u8_np(6, ((r + 7) // 8,))
    assert (ens.answer(torch.from_numpy(share).cuda()).cpu().numpy() == O.ens_respond(rec, share)).all()

    ftr = DistributedFtr(r, d, records=torch.from_numpy(rec).cuda())
    Qf = synth.uniform_u32_np(7, (2, r)) % 65537
    got = ftr.answer_batch(torch.from_numpy(Qf.view(np.int32)).cuda())
    assert (got.cpu().numpy() == O.ftr_respond_batch(rec, Qf)).all()


@pytest.mark.parametrize("n,length", [(1, 3072), (2, 3072), (5, 17), (8, 100000)])
def test_combine_kernels_match_definitions(cuda_ok, n, length):
    """qpir_xor_fold / qpir_sum_mod_p (the cross-rank fold after the all-gather)
    against their definitions written out in numpy: XOR over parts, and the
    exact integer sum reduced mod p; host pointers are refused (no fallback)."""
    from paper_2510_03631_b200 import _lib
    parts8 = synth.uniform_u8_np(60 + n, (n, length))
    out8 = torch.empty(length, dtype=torch.uint8, device="cuda")
    _lib.qpir_xor_fold(torch.from_numpy(parts8).cuda(), n, length, out8)
    assert (out8.cpu().numpy() == np.bitwise_xor.reduce(parts8, axis=0)).all()
    for p in (65537, 2, 4294967291):
        parts32 = synth.uniform_u32_np(70 + n, (n, length)) % p
        out32 = torch.empty(length, dtype=torch.int32, device="cuda")
        _lib.qpir_sum_mod_p(torch.from_numpy(parts32.view(np.int32)).cuda(), n, length, p, out32)
        want = (parts32.astype(object).sum(0) % p).astype(np.uint32)
        assert (out32.cpu().numpy().view(np.uint32) == want).all(), p
    with pytest.raises(_lib.QpirError):
        _lib.qpir_xor_fold(parts8, n, length, out8)  # host parts
