"""Multi-GPU layer (step a5): row-shard D over ranks, gather answers.

One process per GPU (torchrun), torch.distributed for the plumbing.  Rows of D
are independent, so each rank answers its own whole-channel shard with its
own kernels and the only exchange is the final gather of answer slices over
NCCL (NVLink / NVSwitch).  The query is replicated (each rank copies it from
host, or it is broadcast once).  No collective sits inside the data path.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(n_cells: int, n_ch: int, d: int, m: int, world: int, rank: int):
    """Whole-channel row shard [row_begin, row_end) of rank (DESIGN "Multi-GPU").

    Rows come in units of d (one (row-block, channel) pair = one record byte
    range); units are split as evenly as possible, earlier ranks get the extra.
    """
    n_blk = -(-n_cells // m)
    units = n_blk * n_ch
    if world > units:
        raise ValueError(f"world {world} > {units} channel units")
    base, extra = divmod(units, world)
    u0 = rank * base + min(rank, extra)
    u1 = u0 + base + (1 if rank < extra else 0)
    return u0 * d, u1 * d


def gather_answer(ans_local: torch.Tensor, shard_sizes, group=None) -> torch.Tensor:
    """Concatenate every rank's answer slice (along the last dim) on every rank.

    ans_local: [..., ell_local] int32 (u32 bits).  Shards may differ in size by
    one unit; slices are padded to the largest and trimmed after all_gather.
    """
    world = dist.get_world_size(group)
    mx = max(shard_sizes)
    lead = ans_local.shape[:-1]
    if ans_local.shape[-1] != mx:
        pad = torch.zeros(*lead, mx, dtype=ans_local.dtype, device=ans_local.device)
        pad[..., : ans_local.shape[-1]] = ans_local
        ans_local = pad
    ans_local = ans_local.contiguous()
    if dist.get_backend(group) == "nccl":
        buf = torch.empty((world, *lead, mx), dtype=ans_local.dtype, device=ans_local.device)
        dist.all_gather_into_tensor(buf, ans_local.unsqueeze(0), group=group)
        slices = [buf[r] for r in range(world)]
    else:  # gloo (CPU tests, single-GPU functional runs): list all_gather on host
        host = ans_local.cpu()
        slices = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(slices, host, group=group)
        slices = [t.to(ans_local.device) for t in slices]
    parts = [slices[r][..., : shard_sizes[r]] for r in range(world)]
    return torch.cat(parts, dim=-1)


class DistributedPIR:
    """Row-sharded PIR server: each rank holds one shard on its own GPU."""

    def __init__(self, n_cells: int, n_ch: int, rec_bytes: int, *, m: int = 0,
                 lwe_n: int = 1024, seed_A: int = 0, device: int | None = None,
                 records=None, group=None, stable_inputs: bool = False):
        from . import PirServer

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        m_eff = m or n_cells
        self.bounds = [shard_rows(n_cells, n_ch, rec_bytes, m_eff, self.world, r)
                       for r in range(self.world)]
        self.sizes = [b - a for a, b in self.bounds]
        r0, r1 = self.bounds[self.rank]
        dev = torch.cuda.current_device() if device is None else device
        self.server = PirServer(n_cells, n_ch, rec_bytes, m=m, lwe_n=lwe_n, seed_A=seed_A,
                                row_begin=r0, row_end=r1, device=dev, records=records,
                                stable_inputs=stable_inputs)

    def answer(self, qu, gather: bool = True):
        a = self.server.answer(qu)
        return gather_answer(a, self.sizes, self.group) if gather else a

    def answer_many(self, queries, stream=None):
        """Answer a sequence of single queries, overlapping the NCCL gather of
        query i with the GEMV of query i + 1 (two answer-slice buffers, a side
        stream for the collective).  Returns the list of full answers."""
        dev = torch.device("cuda", self.server.device)
        main = stream or torch.cuda.current_stream(dev)
        comm = torch.cuda.Stream(dev)
        bufs = [torch.empty(self.server.ell_local, dtype=torch.int32, device=dev)
                for _ in range(2)]
        done = [None, None]
        outs = []
        for i, q in enumerate(queries):
            b = i % 2
            if done[b] is not None:
                main.wait_event(done[b])  # the slice's previous gather has read it
            self.server.answer(q, out=bufs[b], stream=main)
            ready = torch.cuda.Event()
            ready.record(main)
            comm.wait_event(ready)
            with torch.cuda.stream(comm):
                outs.append(gather_answer(bufs[b], self.sizes, self.group))
                done[b] = torch.cuda.Event()
                done[b].record(comm)
        main.wait_stream(comm)
        return outs

    def answer_batch(self, Q, gather: bool = True):
        a = self.server.answer_batch(Q)
        return gather_answer(a, self.sizes, self.group) if gather else a

    def hint(self, gather: bool = False):
        h = self.server.hint()
        if not gather:
            return h
        return gather_answer(h.t().contiguous(), self.sizes, self.group).t()


# ---------------------------------------------------------------- NEXT rows
def shard_records(r: int, world: int, rank: int, align: int = 1):
    """Contiguous record shard [t0, t1) of rank (whole multiples of `align`)."""
    units = -(-r // align)
    base, extra = divmod(units, world)
    u0 = rank * base + min(rank, extra)
    u1 = u0 + base + (1 if rank < extra else 0)
    return min(r, u0 * align), min(r, u1 * align)


def gather_parts(part: torch.Tensor, group=None) -> torch.Tensor:
    """[world, *part.shape] stack of every rank's partial response (rank-major),
    on part's device -- communication only (NCCL all-gather over NVLink; gloo
    list all-gather through host memory in CPU tests)."""
    world = dist.get_world_size(group)
    part = part.contiguous()
    if dist.get_backend(group) == "nccl":
        buf = torch.empty((world, *part.shape), dtype=part.dtype, device=part.device)
        dist.all_gather_into_tensor(buf, part.unsqueeze(0), group=group)
        return buf
    host = part.cpu()
    parts = [torch.empty_like(host) for _ in range(world)]
    dist.all_gather(parts, host, group=group)
    return torch.stack(parts).to(part.device)


def xor_combine(part: torch.Tensor, group=None) -> torch.Tensor:
    """XOR of every rank's uint8 partial response (NCCL has no XOR reduction):
    all-gather the d-byte partials, then fold them with the library's device
    kernel (qpir_xor_fold)."""
    from . import _lib
    parts = gather_parts(part, group)
    out = torch.empty_like(part)
    _lib.qpir_xor_fold(parts, parts.shape[0], part.numel(), out)
    return out


def sum_mod_p(part_u32: torch.Tensor, p: int, group=None) -> torch.Tensor:
    """Sum of every rank's partial F_p response (values < p) mod p, exactly:
    all-gather the u32 partials, then fold them with the library's device
    kernel (qpir_sum_mod_p, 64-bit sums)."""
    from . import _lib
    parts = gather_parts(part_u32, group)
    out = torch.empty_like(part_u32)
    _lib.qpir_sum_mod_p(parts, parts.shape[0], part_u32.numel(), p, out)
    return out


class DistributedEns:
    """QPADL-ENS with the records sharded over ranks: each GPU XORs the selected
    records of its shard; the d-byte partials are XOR-combined."""

    def __init__(self, n_records: int, rec_bytes: int, *, device: int | None = None,
                 records=None, group=None, stable_inputs: bool = False):
        from . import EnsServer

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.r, self.d = n_records, rec_bytes
        self.t0, self.t1 = shard_records(n_records, self.world, self.rank, align=8)
        dev = torch.cuda.current_device() if device is None else device
        local = None if records is None else records[self.t0:self.t1]
        self.server = EnsServer(self.t1 - self.t0, rec_bytes, device=dev, records=local,
                                stable_inputs=stable_inputs)

    def local_share(self, share_bits: torch.Tensor) -> torch.Tensor:
        """Slice of a full r-bit share for this shard (shards start on byte boundaries)."""
        nb = (self.t1 - self.t0 + 7) // 8
        return share_bits[..., self.t0 // 8: self.t0 // 8 + nb].contiguous()

    def answer(self, share_bits):
        return xor_combine(self.server.answer(self.local_share(share_bits)), self.group)


class DistributedFtr:
    """QPADL-FTR with the records sharded over ranks: partial rho . DB mod p per
    shard, summed across ranks mod p."""

    def __init__(self, n_records: int, rec_bytes: int, *, p: int = 65537,
                 device: int | None = None, records=None, group=None):
        from . import FtrServer

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.p = p
        self.t0, self.t1 = shard_records(n_records, self.world, self.rank)
        dev = torch.cuda.current_device() if device is None else device
        local = None if records is None else records[self.t0:self.t1]
        self.server = FtrServer(self.t1 - self.t0, rec_bytes, p=p, device=dev, records=local)

    def answer_batch(self, Q):
        part = self.server.answer_batch(Q[:, self.t0:self.t1].contiguous())
        return sum_mod_p(part, self.p, self.group)
