"""Seeded synthetic inputs for the LWE-PIR answer path.

This module is the ONLY code shared by the oracle side (tests) and the CUDA side
(bench.py, tests): it generates input bytes and holds none of the method's
arithmetic (no layout, no products, no LWE).  It is counter-based: every byte is
a pure function of (seed, record index theta, byte index), evaluated with torch
integer ops, so the same call gives the same bytes on CPU and on any CUDA device
and any subset (a sampled row of D, a chunk of records) can be regenerated alone.

Record recipe ("each DB entry fixed at 3KB"; P:1686 HCT
puzzle 37 B; P:1688 ML-DSA signature 2420 B; P:515 entries carry EIRP and
spectrum data):
  d == 3072 ("paper-shaped"):
    [0,4)  cell_x  u32 LE     [4,8) cell_y u32 LE   [8,10) channel u16 LE
    [10,12) time-validity window u16 (= 0, one window, DESIGN R9)
    [12,14) EIRP i16 LE, 0.01 dBm fixed point, uniform in [-1000, 3600)
    [14]   availability flag (0/1)
    [15,560) pseudo-random spectrum payload          (560 B spectrum data)
    [560,592) HCT nonce n_s (random) [592,596) kappa = 20 u32 LE [596] n_l = 3
    [597,3017) pseudo-random "ML-DSA signature"       (2420 B)
    [3017,3072) zero padding
  any other d: every byte pseudo-random (C1 uses d = 8).
Queries for throughput runs are uniform u32 (the answer's cost does not depend
on values; correctness runs use real LWE queries from the oracle).
"""
from __future__ import annotations

import numpy as np
import torch

_M32 = 0xFFFFFFFF
PAPER_RECORD_BYTES = 3072


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for 0 <= x < 2^32 held in int64, without int64 overflow."""
    lo, hi = c & 0xFFFF, c >> 16
    return (x * lo + ((x * hi) & 0xFFFF) * 65536) & _M32


def hash32(x: torch.Tensor) -> torch.Tensor:
    """lowbias32 integer hash (C. Wellons), on int64 tensors holding u32 values."""
    x = x & _M32
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def _seed_words(seed: int):
    return seed & _M32, (seed >> 32) & _M32


def record_words(seed: int, theta: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """u32 word w of record theta (int64 tensors, broadcastable) -> int64 in [0, 2^32)."""
    s0, s1 = _seed_words(seed)
    k = hash32((theta & _M32) ^ s0)
    k = hash32(k ^ ((theta >> 32) & _M32) ^ 0x5BD1E995)
    return hash32(hash32((k + w) & _M32) ^ s1)


def _to_i32(v: torch.Tensor) -> torch.Tensor:
    """u32 value in int64 -> same bit pattern as int32 (no out-of-range cast)."""
    return (v - ((v >> 31) << 32)).to(torch.int32)


def _le_bytes(v: torch.Tensor, nbytes: int) -> torch.Tensor:
    """[N] int64 -> [N, nbytes] uint8 little-endian."""
    sh = torch.arange(nbytes, device=v.device, dtype=torch.int64) * 8
    return ((v.unsqueeze(-1) >> sh) & 0xFF).to(torch.uint8)


def records_at(seed: int, theta: torch.Tensor, d: int, n_ch: int, n_cols: int,
               upto: int | None = None) -> torch.Tensor:
    """Records for an int64 tensor of indices theta -> [len(theta), upto or d] uint8."""
    nb = d if upto is None else min(d, upto)
    nw = (nb + 3) // 4
    w = torch.arange(nw, device=theta.device, dtype=torch.int64)
    words = record_words(seed, theta.unsqueeze(1), w.unsqueeze(0))  # [N, nw]
    rec = _to_i32(words).view(torch.uint8).reshape(theta.numel(), nw * 4)[:, :nb].clone()
    if d == PAPER_RECORD_BYTES:
        _apply_structure(seed, rec, theta, n_ch, n_cols, nb)
    return rec


def _apply_structure(seed: int, rec: torch.Tensor, theta: torch.Tensor, n_ch: int,
                     n_cols: int, nb: int) -> None:
    cell = theta // n_ch
    ch = theta % n_ch
    fields = []
    fields.append((0, _le_bytes(cell % n_cols, 4)))
    fields.append((4, _le_bytes(cell // n_cols, 4)))
    fields.append((8, _le_bytes(ch, 2)))
    fields.append((10, _le_bytes(torch.zeros_like(theta), 2)))
    h = hash32(record_words(seed, theta, torch.full_like(theta, 0x7FFF0000)))
    eirp = (h % 4600) - 1000
    fields.append((12, _le_bytes(eirp & 0xFFFF, 2)))
    fields.append((14, _le_bytes((h >> 20) & 1, 1)))
    fields.append((592, _le_bytes(torch.full_like(theta, 20), 4)))
    fields.append((596, _le_bytes(torch.full_like(theta, 3), 1)))
    for off, val in fields:
        if off >= nb:
            continue
        k = min(val.shape[1], nb - off)
        rec[:, off:off + k] = val[:, :k]
    if nb > 3017:
        rec[:, 3017:nb] = 0


def records(seed: int, theta_begin: int, n_records: int, d: int, n_ch: int,
            n_cols: int = 512, device="cpu") -> torch.Tensor:
    """Records theta_begin .. theta_begin + n_records - 1 -> [n_records, d] uint8."""
    theta = torch.arange(theta_begin, theta_begin + n_records, device=device, dtype=torch.int64)
    return records_at(seed, theta, d, n_ch, n_cols)


def records_np(seed: int, n_records: int, d: int, n_ch: int, n_cols: int = 512) -> np.ndarray:
    return records(seed, 0, n_records, d, n_ch, n_cols, "cpu").numpy()


def byte_column(seed: int, theta: torch.Tensor, b: int, d: int, n_ch: int,
                n_cols: int = 512) -> torch.Tensor:
    """Byte b of each record in theta -> uint8 [len(theta)] (for sampled rows of D)."""
    if d == PAPER_RECORD_BYTES and (b < 600 or b >= 3017):
        return records_at(seed, theta, d, n_ch, n_cols, upto=b + 1)[:, b]
    v = record_words(seed, theta, torch.full_like(theta, b // 4))
    return ((v >> (8 * (b % 4))) & 0xFF).to(torch.uint8)


def uniform_u32(seed: int, shape, device="cpu") -> torch.Tensor:
    """Uniform u32 values (bit pattern held in int32) for throughput queries."""
    n = int(np.prod(shape))
    idx = torch.arange(n, device=device, dtype=torch.int64)
    s0, s1 = _seed_words(seed)
    v = hash32(hash32(idx ^ s0) ^ s1 ^ 0x2545F491)
    return _to_i32(v).reshape(shape)


def uniform_u32_np(seed: int, shape) -> np.ndarray:
    return uniform_u32(seed, shape).numpy().view(np.uint32)


def uniform_u8_np(seed: int, shape) -> np.ndarray:
    return (uniform_u32(seed, shape).numpy().view(np.uint32) & 0xFF).astype(np.uint8)
