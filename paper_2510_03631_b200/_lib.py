"""Thin ctypes binding of libqpir.so (include/qpir.h) -- argument marshalling only.

Every function here keeps the C name and forwards pointers and lengths; all
computation happens in the CUDA kernels behind the C ABI.  There is no CPU
fallback: if libqpir.so is missing this module raises at import.
Buffers may be torch tensors (CUDA or CPU), numpy arrays, or raw integer
addresses.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# QPIR_LIB: load another build of the same ABI (A/B measurements against an
# earlier build of this library; there is no other implementation behind it)
LIB_PATH = os.environ.get("QPIR_LIB") or os.path.join(_HERE, "libqpir.so")

QPIR_OK = 0
QPIR_E_PARAM = 1
QPIR_E_DIMENSION = 2
QPIR_E_STATE = 3
QPIR_E_OOM = 4
QPIR_E_CUDA = 5

EXPORTS = (
    "qpir_setup", "qpir_db_write", "qpir_geometry", "qpir_answer", "qpir_answer_batch",
    "qpir_hint", "qpir_kernel_launches", "qpir_last_error", "qpir_destroy",
    "qpir_answer_batch_modp", "qpir_ens_setup", "qpir_ens_db_write", "qpir_ens_answer", "qpir_ens_answer_batch",
    "qpir_ens_kernel_launches", "qpir_ens_last_error", "qpir_ens_destroy",
    "qpir_oop_preprocess", "qpir_oop_answer", "qpir_ens_last_path",
    "qpir_xor_fold", "qpir_sum_mod_p", "qpir_combine_last_error",
    "qpir_puzzle_bind_hct", "qpir_ens_puzzle_bind_hct",
)

# qpir_ens_last_path values (include/qpir.h)
QPIR_ENS_PATH_NONE, QPIR_ENS_PATH_SCAN, QPIR_ENS_PATH_CUDA_CORES, QPIR_ENS_PATH_TENSOR = 0, 1, 2, 3


class qpir_params(ctypes.Structure):
    _fields_ = [
        ("n_cells", ctypes.c_uint64),
        ("n_ch", ctypes.c_uint64),
        ("rec_bytes", ctypes.c_uint64),
        ("m", ctypes.c_uint64),
        ("lwe_n", ctypes.c_uint32),
        ("log_q", ctypes.c_uint32),
        ("log_p", ctypes.c_uint32),
        ("reserved0", ctypes.c_uint32),
        ("seed_A", ctypes.c_uint64),
        ("row_begin", ctypes.c_uint64),
        ("row_end", ctypes.c_uint64),
        ("device", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


class qpir_ens_params(ctypes.Structure):
    _fields_ = [
        ("n_records", ctypes.c_uint64),
        ("rec_bytes", ctypes.c_uint64),
        ("device", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


QPIR_FLAG_STABLE_INPUTS = 1  # include/qpir.h


class QpirError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"qpir error {code}: {msg}")
        self.code = code


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_2510_03631_b200/build.py` "
        "(there is no CPU fallback)"
    )

class _OlderBuild:
    """QPIR_LIB pointing at an earlier build (A/B timing): symbols it lacks
    become stubs that raise when called, so the rest still binds."""

    def __init__(self, lib):
        self._lib = lib

    def __getattr__(self, name):
        try:
            return getattr(self._lib, name)
        except AttributeError:
            def stub(*_a):
                raise QpirError(QPIR_E_STATE, f"{name}: not exported by {LIB_PATH}")
            setattr(self, name, stub)
            return stub


_L = ctypes.CDLL(LIB_PATH)
if os.environ.get("QPIR_LIB"):
    _L = _OlderBuild(_L)
_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_L.qpir_setup.argtypes = [ctypes.POINTER(qpir_params), _vp, _u64, _vp, ctypes.POINTER(_vp)]
_L.qpir_db_write.argtypes = [_vp, _u64, _u64, _vp, _u64, _vp]
_L.qpir_puzzle_bind_hct.argtypes = [_vp, _u64, _u64, _vp, _u64, _u64, _u64, ctypes.c_uint32,
                                    ctypes.c_uint8, _vp, _vp, _vp]
_L.qpir_ens_puzzle_bind_hct.argtypes = _L.qpir_puzzle_bind_hct.argtypes
_L.qpir_geometry.argtypes = [_vp, ctypes.POINTER(_u64), ctypes.POINTER(_u64),
                             ctypes.POINTER(_u64), ctypes.POINTER(_u64)]
_L.qpir_answer.argtypes = [_vp, _vp, _u64, _vp, _u64, _vp]
_L.qpir_answer_batch.argtypes = [_vp, _vp, _u64, _u64, _vp, _u64, _vp]
_L.qpir_hint.argtypes = [_vp, _vp, _u64, _vp]
_L.qpir_answer_batch_modp.argtypes = [_vp, _vp, _u64, _u64, ctypes.c_uint32, _vp, _u64, _vp]
_L.qpir_kernel_launches.argtypes = [_vp]
_L.qpir_kernel_launches.restype = _u64
_L.qpir_last_error.argtypes = [_vp]
_L.qpir_last_error.restype = ctypes.c_char_p
_L.qpir_destroy.argtypes = [_vp]
_L.qpir_ens_setup.argtypes = [ctypes.POINTER(qpir_ens_params), _vp, _u64, _vp, ctypes.POINTER(_vp)]
_L.qpir_ens_db_write.argtypes = [_vp, _u64, _u64, _vp, _u64, _vp]
_L.qpir_ens_answer.argtypes = [_vp, _vp, _u64, _vp, _u64, _vp]
_L.qpir_ens_answer_batch.argtypes = [_vp, _vp, _u64, _u64, _vp, _u64, _vp]
_L.qpir_ens_kernel_launches.argtypes = [_vp]
_L.qpir_ens_kernel_launches.restype = _u64
_L.qpir_ens_last_path.argtypes = [_vp]
_L.qpir_ens_last_path.restype = ctypes.c_int
_L.qpir_ens_last_error.argtypes = [_vp]
_L.qpir_ens_last_error.restype = ctypes.c_char_p
_L.qpir_ens_destroy.argtypes = [_vp]
_L.qpir_oop_preprocess.argtypes = [_vp, ctypes.c_uint32, ctypes.c_uint32, _vp, _u64, _vp, _u64, _vp]
_L.qpir_oop_answer.argtypes = [_vp, ctypes.c_uint32, ctypes.c_uint32, _vp, _u64, _vp, _u64, _vp,
                               _u64, _vp]
_L.qpir_xor_fold.argtypes = [_vp, _u64, _u64, _vp, _vp]
_L.qpir_sum_mod_p.argtypes = [_vp, _u64, _u64, ctypes.c_uint32, _vp, _vp]
_L.qpir_combine_last_error.argtypes = []
_L.qpir_combine_last_error.restype = ctypes.c_char_p
for _name in EXPORTS:
    getattr(_L, _name)


def _addr(x) -> int | None:
    """Raw address of a buffer (torch tensor, numpy array or int) without copying."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):  # torch.Tensor
        assert x.is_contiguous(), "qpir buffers must be contiguous"
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"], "qpir buffers must be C-contiguous"
        return x.ctypes.data
    raise TypeError(f"unsupported buffer type {type(x)}")


def _numel(x) -> int:
    if hasattr(x, "numel"):
        return int(x.numel())
    return int(np.asarray(x).size)


def _stream(stream) -> int | None:
    """cudaStream_t handle.  None -> torch's current stream on the current
    device (so calls order with torch work inside `with torch.cuda.stream(s)`);
    an int is passed through (0 = the legacy default stream)."""
    if stream is None:
        import torch
        if not torch.cuda.is_available():
            return None
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream  # torch.cuda.Stream


def _check(rc: int, ctx=None):
    if rc != QPIR_OK:
        msg = _L.qpir_last_error(ctx).decode()
        raise QpirError(rc, msg)


def _check_ens(rc: int, ctx=None):
    if rc != QPIR_OK:
        raise QpirError(rc, _L.qpir_ens_last_error(ctx).decode())


# ------------------------------------------------------------ C names
def qpir_setup(params: qpir_params, records=None, stream=None) -> int:
    """Returns the context handle (int).  records: full theta-ordered u8 array or None."""
    out = _vp()
    rec_len = _numel(records) if records is not None else 0
    rc = _L.qpir_setup(ctypes.byref(params), _addr(records), rec_len, _stream(stream),
                       ctypes.byref(out))
    _check(rc, None)
    return out.value


def qpir_db_write(ctx: int, theta_begin: int, records, n_records: int, stream=None):
    _check(_L.qpir_db_write(ctx, theta_begin, n_records, _addr(records), _numel(records),
                            _stream(stream)), ctx)


def qpir_puzzle_bind_hct(ctx: int, theta_begin: int, spectrum, n_records: int, spec_stride: int,
                         seed_psd: int, kappa: int, n_l: int, mldsa_seed=None, mldsa_pk=None,
                         stream=None):
    _check(_L.qpir_puzzle_bind_hct(ctx, theta_begin, n_records, _addr(spectrum), spec_stride,
                                   _numel(spectrum), seed_psd, kappa, n_l,
                                   None if mldsa_seed is None else _addr(mldsa_seed),
                                   None if mldsa_pk is None else _addr(mldsa_pk),
                                   _stream(stream)), ctx)


def qpir_ens_puzzle_bind_hct(ctx: int, theta_begin: int, spectrum, n_records: int,
                             spec_stride: int, seed_psd: int, kappa: int, n_l: int,
                             mldsa_seed=None, mldsa_pk=None, stream=None):
    _check_ens(_L.qpir_ens_puzzle_bind_hct(ctx, theta_begin, n_records, _addr(spectrum),
                                           spec_stride, _numel(spectrum), seed_psd, kappa, n_l,
                                           None if mldsa_seed is None else _addr(mldsa_seed),
                                           None if mldsa_pk is None else _addr(mldsa_pk),
                                           _stream(stream)), ctx)


def qpir_geometry(ctx: int):
    v = [_u64() for _ in range(4)]
    _check(_L.qpir_geometry(ctx, *[ctypes.byref(x) for x in v]), ctx)
    return tuple(int(x.value) for x in v)  # ell, m, ell_local, row_begin


def qpir_answer(ctx: int, qu, ans_local, stream=None):
    _check(_L.qpir_answer(ctx, _addr(qu), _numel(qu), _addr(ans_local), _numel(ans_local),
                          _stream(stream)), ctx)


def qpir_answer_batch(ctx: int, Q, B: int, ans_local, stream=None):
    _check(_L.qpir_answer_batch(ctx, _addr(Q), B, _numel(Q), _addr(ans_local),
                                _numel(ans_local), _stream(stream)), ctx)


def qpir_answer_batch_modp(ctx: int, Q, B: int, p: int, ans_local, stream=None):
    _check(_L.qpir_answer_batch_modp(ctx, _addr(Q), B, _numel(Q), p, _addr(ans_local),
                                     _numel(ans_local), _stream(stream)), ctx)


def qpir_hint(ctx: int, H_local, stream=None):
    _check(_L.qpir_hint(ctx, _addr(H_local), _numel(H_local), _stream(stream)), ctx)


def qpir_kernel_launches(ctx: int) -> int:
    return int(_L.qpir_kernel_launches(ctx))


def qpir_last_error(ctx: int | None = None) -> str:
    return _L.qpir_last_error(ctx).decode()


def qpir_destroy(ctx: int) -> None:
    _L.qpir_destroy(ctx)


# ------------------------------------------------------------ ENS (Chor XOR PIR)
def qpir_ens_setup(params: qpir_ens_params, records=None, stream=None) -> int:
    out = _vp()
    rec_len = _numel(records) if records is not None else 0
    rc = _L.qpir_ens_setup(ctypes.byref(params), _addr(records), rec_len, _stream(stream),
                           ctypes.byref(out))
    _check_ens(rc, None)
    return out.value


def qpir_ens_db_write(ctx: int, theta_begin: int, records, n_records: int, stream=None):
    _check_ens(_L.qpir_ens_db_write(ctx, theta_begin, n_records, _addr(records),
                                    _numel(records), _stream(stream)), ctx)


def qpir_ens_answer(ctx: int, share, out, stream=None):
    _check_ens(_L.qpir_ens_answer(ctx, _addr(share), _numel(share), _addr(out), _numel(out),
                                  _stream(stream)), ctx)


def qpir_ens_answer_batch(ctx: int, shares, B: int, out, stream=None):
    _check_ens(_L.qpir_ens_answer_batch(ctx, _addr(shares), B, _numel(shares), _addr(out),
                                        _numel(out), _stream(stream)), ctx)


def qpir_ens_kernel_launches(ctx: int) -> int:
    return int(_L.qpir_ens_kernel_launches(ctx))


def qpir_ens_last_path(ctx: int) -> int:
    return int(_L.qpir_ens_last_path(ctx))


def qpir_ens_last_error(ctx: int | None = None) -> str:
    return _L.qpir_ens_last_error(ctx).decode()


def qpir_ens_destroy(ctx: int) -> None:
    _L.qpir_ens_destroy(ctx)


# ------------------------------------------------------------ OOP (CIP-PIR offline-online)
def qpir_oop_preprocess(ctx: int, n_chunks: int, server: int, seeds, A_out, stream=None):
    _check_ens(_L.qpir_oop_preprocess(ctx, n_chunks, server, _addr(seeds), _numel(seeds),
                                      _addr(A_out), _numel(A_out), _stream(stream)), ctx)


def qpir_oop_answer(ctx: int, n_chunks: int, server: int, q, A, out, stream=None):
    _check_ens(_L.qpir_oop_answer(ctx, n_chunks, server, _addr(q), _numel(q), _addr(A), _numel(A),
                                  _addr(out), _numel(out), _stream(stream)), ctx)


# ------------------------------------------------------------ cross-rank combine
def _check_combine(rc: int):
    if rc != QPIR_OK:
        raise QpirError(rc, _L.qpir_combine_last_error().decode())


def qpir_xor_fold(parts, n_parts: int, length: int, out, stream=None):
    _check_combine(_L.qpir_xor_fold(_addr(parts), n_parts, length, _addr(out), _stream(stream)))


def qpir_sum_mod_p(parts, n_parts: int, length: int, p: int, out, stream=None):
    _check_combine(_L.qpir_sum_mod_p(_addr(parts), n_parts, length, p, _addr(out),
                                     _stream(stream)))
