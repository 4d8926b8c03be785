"""Multi-rank host logic on CPU (gloo, world_size 2): whole-channel row
shards and the answer gather reassemble the unsharded answer exactly.  The
per-rank slice answers come from the oracle here (no GPU); on the GPU box the
same gather runs over NCCL on the kernels' slices (bench.py, N > 1)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_03631_b200.dist import gather_answer, shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, geo, B, q):
    import synth
    from oracle import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_cells, n_ch, d, m = geo
        rec = synth.records_np(3, n_cells * n_ch, d, n_ch)
        D = O.pack(rec, n_cells, n_ch, d, m)
        bounds = [shard_rows(n_cells, n_ch, d, m, world, r) for r in range(world)]
        sizes = [b - a for a, b in bounds]
        r0, r1 = bounds[rank]
        Q = synth.uniform_u32_np(4, (B, m))
        local = O.answer_batch(D[r0:r1], Q)              # [B, ell_local]
        t = torch.from_numpy(local.view(np.int32))
        if B == 1:
            t = t[0]
        full = gather_answer(t, sizes).numpy().view(np.uint32)
        want = O.answer_batch(D, Q)
        ok = bool((full == (want[0] if B == 1 else want)).all())
        q.put((rank, ok, sizes))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("geo,B", [((64, 4, 6, 64), 1), ((50, 3, 5, 16), 1), ((40, 5, 4, 40), 3)])
def test_gather_reassembles_answer(geo, B):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, geo, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res


def test_shard_rows_whole_channels():
    # 122880 rows = 40 channels x 3072 B: whole channels per rank for G = 1..8
    for world in (1, 2, 4, 8):
        b = [shard_rows(262144, 40, 3072, 262144, world, r) for r in range(world)]
        assert b[0][0] == 0 and b[-1][1] == 40 * 3072
        assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
        assert all((e - s) % 3072 == 0 and (e - s) == 122880 // world for s, e in b)
    # uneven: 3 channel units over 2 ranks -> 2 + 1
    assert [shard_rows(10, 3, 5, 10, 2, r) for r in range(2)] == [(0, 10), (10, 15)]
    with pytest.raises(ValueError):
        shard_rows(10, 1, 5, 10, 2, 0)


def _worker_next(rank, world, port, q):
    import synth
    from oracle import oracle as O
    # communication only (the device fold kernels are covered by test_gpu_dist.py);
    # the fold itself is written out here, from the definitions (XOR / sum mod p)
    from paper_2510_03631_b200.dist import gather_parts, shard_records
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, d, p = 203, 17, 65537
        rec = synth.uniform_u8_np(9, (r, d))
        # ENS: shards on byte boundaries of the share, partials XOR-combined
        t0, t1 = shard_records(r, world, rank, align=8)
        share = synth.uniform_u8_np(10, ((r + 7) // 8,))
        share[-1] &= (1 << (r % 8)) - 1
        local = share[t0 // 8:(t1 + 7) // 8]
        part = torch.from_numpy(O.ens_respond(rec[t0:t1], local))
        parts = gather_parts(part).numpy()
        folded = np.bitwise_xor.reduce(parts, axis=0)
        ok_ens = bool((folded == O.ens_respond(rec, share)).all())
        # FTR: contiguous shards, partial sums mod p combined exactly
        f0, f1 = shard_records(r, world, rank)
        Q = synth.uniform_u32_np(11, (3, r)) % p
        partf = torch.from_numpy(O.ftr_respond_batch(rec[f0:f1], Q[:, f0:f1]).view(np.int32))
        pf = gather_parts(partf).numpy().view(np.uint32).astype(np.int64)
        ok_ftr = bool(((pf.sum(0) % p) == O.ftr_respond_batch(rec, Q)).all())
        q.put((rank, ok_ens, ok_ftr))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_next_rows_shard_and_combine(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_next, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(e and f for _, e, f in res), res
