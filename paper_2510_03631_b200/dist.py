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
                 records=None, group=None):
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
                                row_begin=r0, row_end=r1, device=dev, records=records)

    def answer(self, qu, gather: bool = True):
        a = self.server.answer(qu)
        return gather_answer(a, self.sizes, self.group) if gather else a

    def answer_batch(self, Q, gather: bool = True):
        a = self.server.answer_batch(Q)
        return gather_answer(a, self.sizes, self.group) if gather else a

    def hint(self, gather: bool = False):
        h = self.server.hint()
        if not gather:
            return h
        return gather_answer(h.t().contiguous(), self.sizes, self.group).t()
