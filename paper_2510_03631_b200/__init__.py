"""B200-native LWE-PIR answer engine for QPADL spectrum databases (arXiv 2510.03631).

Public API (thin wrappers over the C ABI in include/qpir.h):
    PirServer(...)            one rank-local context holding a row shard of D
        .answer(qu)           ans = D.qu mod 2^32         (GEMV, HBM-bound)
        .answer_batch(Q)      ANS = D.Q mod 2^32          (tcgen05 int8-limb GEMM)
        .hint()               H = D.A mod 2^32            (tcgen05 int8-limb GEMM)
    EnsServer(...)            QPADL-ENS (Chor XOR PIR, NEXT-1): records theta-major
        .answer(share)        XOR of the selected records (HBM scan, sparse rows skipped)
        .answer_batch(Q)      multi-request form (Alg. 3)
    FtrServer(...)            QPADL-FTR (Goldberg PIR over F_p, NEXT-2): rho . DB mod p
        .answer_batch(Q)      on the tcgen05 limb engine with a mod-p epilogue (Alg. 4)
    dist.DistributedPIR       row-sharded over ranks, NCCL gather of answer slices
u32 values are carried in torch.int32 tensors (same bits); use u32() to view them.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import QpirError, qpir_params  # noqa: F401

__all__ = ["PirServer", "EnsServer", "FtrServer", "QpirError", "u32", "qpir_params"]


def _st(device: int, stream):
    """Default stream of a call: torch's current stream on the context's device
    (calls then order with torch work, including inside torch.cuda.stream(...))."""
    return torch.cuda.current_stream(device) if stream is None else stream


def u32(t) -> np.ndarray:
    """torch int32 (u32 bit pattern) tensor -> numpy uint32 array (copies to host)."""
    if isinstance(t, np.ndarray):
        return t.view(np.uint32)
    return t.detach().cpu().numpy().view(np.uint32)


def _mldsa_bufs(mldsa_seed):
    """Host buffers for the ML-DSA key seed (32 bytes) and the public key out."""
    if mldsa_seed is None:
        return None, None
    seed = np.frombuffer(bytes(mldsa_seed), np.uint8).copy()
    assert seed.size == 32, "mldsa_seed: 32 bytes"
    return seed, np.zeros(1312, np.uint8)


class PirServer:
    """A context over rows [row_begin, row_end) of the DB matrix on one GPU."""

    def __init__(self, n_cells: int, n_ch: int, rec_bytes: int, *, m: int = 0,
                 lwe_n: int = 1024, seed_A: int = 0, row_begin: int = 0, row_end: int = 0,
                 device: int = 0, records=None, stream=None, stable_inputs: bool = False):
        # stable_inputs: QPIR_FLAG_STABLE_INPUTS (include/qpir.h) -- device query
        # buffers are never written by the kernel right before an answer call
        p = qpir_params(n_cells=n_cells, n_ch=n_ch, rec_bytes=rec_bytes, m=m, lwe_n=lwe_n,
                        log_q=32, log_p=8, reserved0=0, seed_A=seed_A, row_begin=row_begin,
                        row_end=row_end, device=device,
                        flags=_lib.QPIR_FLAG_STABLE_INPUTS if stable_inputs else 0)
        self.device = device
        self.lwe_n = lwe_n
        self._ctx = _lib.qpir_setup(p, records, _st(device, stream))
        self.ell, self.m, self.ell_local, self.row_begin = _lib.qpir_geometry(self._ctx)
        self.n_cells, self.n_ch, self.rec_bytes = n_cells, n_ch, rec_bytes

    # ------------------------------------------------------------------ DB
    def db_write(self, theta_begin: int, records, stream=None) -> None:
        n = int(records.shape[0]) if records.ndim == 2 else records.numel() // self.rec_bytes
        _lib.qpir_db_write(self._ctx, theta_begin, records, n, _st(self.device, stream))

    def puzzle_bind_hct(self, theta_begin: int, spectrum, seed_psd: int, kappa: int = 20,
                        n_l: int = 3, mldsa_seed: bytes | None = None, stream=None):
        """NEXT-4 PSD.Puzzle.Bind (Alg. 1 step 1): records theta_begin .. + len(spectrum)
        built on the GPU (spectrum row || HCT puzzle || ML-DSA-44 signature of the
        puzzle under the key from `mldsa_seed`, or a zero slot without a seed) and
        written into the shard (include/qpir.h qpir_puzzle_bind_hct).  Returns the
        1312-byte public key when signing."""
        assert spectrum.ndim == 2 and str(spectrum.dtype) in ("uint8", "torch.uint8")
        seed, pk = _mldsa_bufs(mldsa_seed)
        _lib.qpir_puzzle_bind_hct(self._ctx, theta_begin, spectrum, int(spectrum.shape[0]),
                                  int(spectrum.shape[1]), seed_psd, kappa, n_l, seed, pk,
                                  _st(self.device, stream))
        return None if pk is None else pk.tobytes()

    # ------------------------------------------------------------------ answers
    def _dev(self):
        return torch.device("cuda", self.device)

    def answer(self, qu, out=None, stream=None):
        if out is None:
            out = torch.empty(self.ell_local, dtype=torch.int32, device=self._dev())
        _lib.qpir_answer(self._ctx, qu, out, _st(self.device, stream))
        return out

    def answer_batch(self, Q, out=None, stream=None):
        B = int(Q.shape[0])
        if out is None:
            out = torch.empty((B, self.ell_local), dtype=torch.int32, device=self._dev())
        _lib.qpir_answer_batch(self._ctx, Q, B, out, _st(self.device, stream))
        return out

    def answer_batch_modp(self, Q, p: int, out=None, stream=None):
        B = int(Q.shape[0])
        if out is None:
            out = torch.empty((B, self.ell_local), dtype=torch.int32, device=self._dev())
        _lib.qpir_answer_batch_modp(self._ctx, Q, B, p, out, _st(self.device, stream))
        return out

    def hint(self, out=None, stream=None):
        if out is None:
            out = torch.empty((self.ell_local, self.lwe_n), dtype=torch.int32, device=self._dev())
        _lib.qpir_hint(self._ctx, out, _st(self.device, stream))
        return out

    @property
    def kernel_launches(self) -> int:
        return _lib.qpir_kernel_launches(self._ctx)

    def close(self) -> None:
        if getattr(self, "_ctx", None):
            _lib.qpir_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class EnsServer:
    """QPADL-ENS server (Chor XOR PIR): r records of d bytes on one GPU."""

    def __init__(self, n_records: int, rec_bytes: int, *, device: int = 0, records=None,
                 stream=None, stable_inputs: bool = False):
        p = _lib.qpir_ens_params(n_records=n_records, rec_bytes=rec_bytes, device=device,
                                 flags=_lib.QPIR_FLAG_STABLE_INPUTS if stable_inputs else 0)
        self.device = device
        self.r, self.d = n_records, rec_bytes
        self.share_bytes = (n_records + 7) // 8
        self._ctx = _lib.qpir_ens_setup(p, records, _st(device, stream))

    def db_write(self, theta_begin: int, records, stream=None) -> None:
        n = int(records.shape[0]) if records.ndim == 2 else records.numel() // self.d
        _lib.qpir_ens_db_write(self._ctx, theta_begin, records, n, _st(self.device, stream))

    def puzzle_bind_hct(self, theta_begin: int, spectrum, seed_psd: int, kappa: int = 20,
                        n_l: int = 3, mldsa_seed: bytes | None = None, stream=None):
        """NEXT-4 PSD.Puzzle.Bind on the ENS records (qpir_ens_puzzle_bind_hct)."""
        assert spectrum.ndim == 2 and str(spectrum.dtype) in ("uint8", "torch.uint8")
        seed, pk = _mldsa_bufs(mldsa_seed)
        _lib.qpir_ens_puzzle_bind_hct(self._ctx, theta_begin, spectrum, int(spectrum.shape[0]),
                                      int(spectrum.shape[1]), seed_psd, kappa, n_l, seed, pk,
                                      _st(self.device, stream))
        return None if pk is None else pk.tobytes()

    def answer(self, share, out=None, stream=None):
        if out is None:
            out = torch.empty(self.d, dtype=torch.uint8, device=torch.device("cuda", self.device))
        _lib.qpir_ens_answer(self._ctx, share, out, _st(self.device, stream))
        return out

    def answer_batch(self, shares, out=None, stream=None):
        B = int(shares.shape[0])
        if out is None:
            out = torch.empty((B, self.d), dtype=torch.uint8,
                              device=torch.device("cuda", self.device))
        _lib.qpir_ens_answer_batch(self._ctx, shares, B, out, _st(self.device, stream))
        return out

    # ---- NEXT-3: OOP / CIP-PIR offline-online on the same records
    def oop_preprocess(self, n_chunks: int, server: int, seeds, out=None, stream=None):
        """Offline: A = PRG(S).(non-flip chunks) for each seed (n_seeds x d bytes)."""
        n = int(seeds.shape[0])
        if out is None:
            out = torch.empty((n, self.d), dtype=torch.uint8, device=torch.device("cuda", self.device))
        _lib.qpir_oop_preprocess(self._ctx, n_chunks, server, seeds, out, _st(self.device, stream))
        return out

    def oop_answer(self, n_chunks: int, server: int, q, A, out=None, stream=None):
        """Online: R_i = A_i XOR q_i . chunk_i (touches 1/n of the DB)."""
        if out is None:
            out = torch.empty(self.d, dtype=torch.uint8, device=torch.device("cuda", self.device))
        _lib.qpir_oop_answer(self._ctx, n_chunks, server, q, A, out, _st(self.device, stream))
        return out

    @property
    def last_path(self) -> str:
        """Kernel path of the last call: "scan", "cuda_cores", "tensor" (or "none")."""
        return ("none", "scan", "cuda_cores", "tensor")[_lib.qpir_ens_last_path(self._ctx)]

    @property
    def kernel_launches(self) -> int:
        return _lib.qpir_ens_kernel_launches(self._ctx)

    def close(self) -> None:
        if getattr(self, "_ctx", None):
            _lib.qpir_ens_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class FtrServer:
    """QPADL-FTR server (Goldberg Shamir-share PIR over F_p): r records of s byte-words.

    The records are the columns of a PirServer with n_ch = 1 (row b = byte b of
    every record), so the response rho . DB mod p is the field-mode batch GEMM."""

    P_DEFAULT = 65537

    def __init__(self, n_records: int, rec_bytes: int, *, p: int = P_DEFAULT, device: int = 0,
                 records=None, stream=None):
        self.p = p
        self.r, self.s = n_records, rec_bytes
        self.server = PirServer(n_records, 1, rec_bytes, lwe_n=4, device=device,
                                records=records, stream=stream)

    def db_write(self, theta_begin: int, records, stream=None) -> None:
        self.server.db_write(theta_begin, records, stream)

    def answer_batch(self, Q, out=None, stream=None):
        return self.server.answer_batch_modp(Q, self.p, out, stream)

    def answer(self, rho, stream=None):
        return self.answer_batch(rho.reshape(1, -1), stream=stream)[0]

    @property
    def kernel_launches(self) -> int:
        return self.server.kernel_launches

    def close(self) -> None:
        self.server.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
