"""ctypes front-end for the plain C oracle (oracle/qpir_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module.  The product
path (paper_2510_03631_b200/) never imports, links or executes anything under
oracle/; the two share no code.  All arithmetic lives in qpir_oracle.c; this
file only marshals numpy arrays.

Citations (PAPER.md lines, DESIGN.md readings) are on each C function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qpir_oracle.c")
_LIB = os.path.join(_HERE, "libqpir_oracle.so")

_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, OpenMP over independent rows)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.qo_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
        L.qo_expand_A.argtypes = [_u64, _u64, _u32, _u32p]
        L.qo_ell.argtypes = [_u64, _u64, _u64, _u64]
        L.qo_ell.restype = _u64
        L.qo_position.argtypes = [_u64, _u64, _u64, _u64, _u64, _u64p, _u64p]
        L.qo_pack.argtypes = [_u8p, _u64, _u64, _u64, _u64, _u8p]
        L.qo_answer.argtypes = [_u8p, _u64, _u64, _u32p, _u32p]
        L.qo_answer_batch.argtypes = [_u8p, _u64, _u64, _u32p, _u64, _u32p]
        L.qo_hint.argtypes = [_u8p, _u64, _u64, _u32p, _u32, _u32p]
        L.qo_keygen.argtypes = [_u64, _u32, _u32p]
        L.qo_sample_error.argtypes = [_u64, _u32, _u64, ctypes.c_double, _i32p]
        L.qo_query.argtypes = [_u32p, _u64, _u32, _u32p, _u64, _u32, ctypes.c_double, _u64,
                               _u32p, _i32p, _i32p]
        L.qo_decode.argtypes = [_u32p, _u32p, _u32, _u32p, _u64p, _u64, _u8p]
        L.qo_ens_query.argtypes = [_u64, _u64, _u32, _u64, _u8p]
        L.qo_ens_respond.argtypes = [_u8p, _u64, _u64, _u8p, _u8p]
        L.qo_ens_respond_batch.argtypes = [_u8p, _u64, _u64, _u8p, _u64, _u8p]
        L.qo_ens_reconstruct.argtypes = [_u8p, _u32, _u64, _u8p]
        L.qo_ftr_query.argtypes = [_u64, _u64, _u32, _u32, _u32, _u64, _u32p]
        L.qo_ftr_respond.argtypes = [_u8p, _u64, _u64, _u32p, _u32, _u32p]
        L.qo_ftr_respond_batch.argtypes = [_u8p, _u64, _u64, _u32p, _u64, _u32, _u32p]
        L.qo_ftr_reconstruct.argtypes = [_u32p, _u32p, _u32, _u64, _u32, _u32p]
        L.qo_ftr_reconstruct.restype = ctypes.c_int
        L.qo_ftr_decode_bw.argtypes = [_u32p, _u32p, _u32, _u64, _u32, _u32, _u32p, _u32p]
        L.qo_ftr_decode_bw.restype = ctypes.c_int
        L.qo_oop_preprocess.argtypes = [_u8p, _u64, _u64, _u32, _u32, _u64, _u8p]
        L.qo_oop_query.argtypes = [_u64, _u64, _u32, _u64p, _u8p]
        L.qo_oop_respond.argtypes = [_u8p, _u64, _u64, _u32, _u32, _u8p, _u8p, _u8p]
        L.qo_num_threads.restype = ctypes.c_int
        L.qo_set_num_threads.argtypes = [ctypes.c_int]
        L.qo_hct_puzzle_gen.argtypes = [_u64, _u64, _u32, ctypes.c_uint8, _u8p]
        L.qo_puzzle_bind_hct.argtypes = [_u8p, _u64, _u64, _u64, _u64, _u32, ctypes.c_uint8, _u64, _u8p]
        _lib = L
    return _lib


def _p(a: np.ndarray, t):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(t)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------- Philox / A
def philox4x32_10(ctr, key) -> np.ndarray:
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().qo_philox4x32_10(_p(c, _u32p), _p(k, _u32p), _p(out, _u32p))
    return out


def expand_A(seed_A: int, m: int, n: int) -> np.ndarray:
    A = np.empty((m, n), np.uint32)
    lib().qo_expand_A(seed_A, m, n, _p(A, _u32p))
    return A


# ---------------------------------------------------------------- layout
def ell(n_cells: int, n_ch: int, d: int, m: int) -> int:
    return int(lib().qo_ell(n_cells, n_ch, d, m))


def position(n_ch: int, d: int, m: int, theta: int, b: int):
    r = ctypes.c_uint64()
    c = ctypes.c_uint64()
    lib().qo_position(n_ch, d, m, theta, b, ctypes.byref(r), ctypes.byref(c))
    return int(r.value), int(c.value)


def pack(records: np.ndarray, n_cells: int, n_ch: int, d: int, m: int) -> np.ndarray:
    rec = _c(records, np.uint8).reshape(-1)
    assert rec.size == n_cells * n_ch * d
    D = np.empty((ell(n_cells, n_ch, d, m), m), np.uint8)
    lib().qo_pack(_p(rec, _u8p), n_cells, n_ch, d, m, _p(D, _u8p))
    return D


# ---------------------------------------------------------------- server side
def answer(D: np.ndarray, qu: np.ndarray) -> np.ndarray:
    D = _c(D, np.uint8)
    qu = _c(qu, np.uint32)
    rows, m = D.shape
    assert qu.shape == (m,)
    ans = np.empty(rows, np.uint32)
    lib().qo_answer(_p(D, _u8p), rows, m, _p(qu, _u32p), _p(ans, _u32p))
    return ans


def answer_batch(D: np.ndarray, Q: np.ndarray) -> np.ndarray:
    D = _c(D, np.uint8)
    Q = _c(Q, np.uint32)
    rows, m = D.shape
    B = Q.shape[0]
    assert Q.shape == (B, m)
    ANS = np.empty((B, rows), np.uint32)
    lib().qo_answer_batch(_p(D, _u8p), rows, m, _p(Q, _u32p), B, _p(ANS, _u32p))
    return ANS


def hint(D: np.ndarray, A: np.ndarray) -> np.ndarray:
    D = _c(D, np.uint8)
    A = _c(A, np.uint32)
    rows, m = D.shape
    assert A.shape[0] == m
    n = A.shape[1]
    H = np.empty((rows, n), np.uint32)
    lib().qo_hint(_p(D, _u8p), rows, m, _p(A, _u32p), n, _p(H, _u32p))
    return H


# ---------------------------------------------------------------- client side
def keygen(seed_s: int, n: int) -> np.ndarray:
    s = np.empty(n, np.uint32)
    lib().qo_keygen(seed_s, n, _p(s, _u32p))
    return s


def sample_error(seed_e: int, qidx: int, m: int, sigma: float) -> np.ndarray:
    e = np.empty(m, np.int32)
    lib().qo_sample_error(seed_e, qidx, m, sigma, _p(e, _i32p))
    return e


def query(A: np.ndarray, s: np.ndarray, seed_e: int, qidx: int, sigma: float, col_star: int):
    """Returns (qu, e)."""
    A = _c(A, np.uint32)
    s = _c(s, np.uint32)
    m, n = A.shape
    qu = np.empty(m, np.uint32)
    e = np.empty(m, np.int32)
    lib().qo_query(_p(A, _u32p), m, n, _p(s, _u32p), seed_e, qidx, sigma, col_star,
                   _p(qu, _u32p), _p(e, _i32p), None)
    return qu, e


def decode(ans: np.ndarray, H: np.ndarray, s: np.ndarray, rows) -> np.ndarray:
    ans = _c(ans, np.uint32)
    H = _c(H, np.uint32)
    s = _c(s, np.uint32)
    rows = _c(rows, np.uint64)
    n = H.shape[1]
    assert s.shape == (n,) and H.shape[0] == ans.shape[0]
    out = np.empty(rows.size, np.uint8)
    lib().qo_decode(_p(ans, _u32p), _p(H, _u32p), n, _p(s, _u32p), _p(rows, _u64p),
                    rows.size, _p(out, _u8p))
    return out


def record_rows(theta: int, n_ch: int, d: int, m: int) -> np.ndarray:
    """Rows of D holding record theta's d bytes (all in one column)."""
    return np.array([position(n_ch, d, m, theta, b)[0] for b in range(d)], np.uint64)


# ---------------------------------------------------------------- ENS (Chor, NEXT-1)
def ens_query(theta: int, r: int, l: int, seed: int) -> np.ndarray:
    """l shares of r bits (l x ceil(r/8) bytes, bit t at byte t>>3, bit t&7)."""
    sh = np.empty((l, (r + 7) // 8), np.uint8)
    lib().qo_ens_query(theta, r, l, seed, _p(sh, _u8p))
    return sh


def ens_respond(records: np.ndarray, share: np.ndarray) -> np.ndarray:
    rec = _c(records, np.uint8)
    r, d = rec.shape
    sh = _c(share, np.uint8)
    assert sh.shape == ((r + 7) // 8,)
    out = np.empty(d, np.uint8)
    lib().qo_ens_respond(_p(rec, _u8p), r, d, _p(sh, _u8p), _p(out, _u8p))
    return out


def ens_respond_batch(records: np.ndarray, Q: np.ndarray) -> np.ndarray:
    rec = _c(records, np.uint8)
    r, d = rec.shape
    Q = _c(Q, np.uint8)
    B = Q.shape[0]
    assert Q.shape == (B, (r + 7) // 8)
    out = np.empty((B, d), np.uint8)
    lib().qo_ens_respond_batch(_p(rec, _u8p), r, d, _p(Q, _u8p), B, _p(out, _u8p))
    return out


def ens_reconstruct(resp: np.ndarray) -> np.ndarray:
    resp = _c(resp, np.uint8)
    l, d = resp.shape
    out = np.empty(d, np.uint8)
    lib().qo_ens_reconstruct(_p(resp, _u8p), l, d, _p(out, _u8p))
    return out


# ---------------------------------------------------------------- FTR (Goldberg, NEXT-2)
FTR_P = 65537


def ftr_query(theta: int, r: int, l: int, t: int, seed: int, p: int = FTR_P) -> np.ndarray:
    """l shares (l x r u32); server i evaluates at alpha_i = i + 1."""
    sh = np.empty((l, r), np.uint32)
    lib().qo_ftr_query(theta, r, l, t, p, seed, _p(sh, _u32p))
    return sh


def ftr_respond(records: np.ndarray, rho: np.ndarray, p: int = FTR_P) -> np.ndarray:
    rec = _c(records, np.uint8)
    r, s_ = rec.shape
    rho = _c(rho, np.uint32)
    assert rho.shape == (r,)
    out = np.empty(s_, np.uint32)
    lib().qo_ftr_respond(_p(rec, _u8p), r, s_, _p(rho, _u32p), p, _p(out, _u32p))
    return out


def ftr_respond_batch(records: np.ndarray, Q: np.ndarray, p: int = FTR_P) -> np.ndarray:
    rec = _c(records, np.uint8)
    r, s_ = rec.shape
    Q = _c(Q, np.uint32)
    B = Q.shape[0]
    assert Q.shape == (B, r)
    out = np.empty((B, s_), np.uint32)
    lib().qo_ftr_respond_batch(_p(rec, _u8p), r, s_, _p(Q, _u32p), B, p, _p(out, _u32p))
    return out


def ftr_reconstruct(resp: np.ndarray, alpha, p: int = FTR_P) -> np.ndarray:
    resp = _c(resp, np.uint32)
    k, s_ = resp.shape
    al = _c(alpha, np.uint32)
    assert al.shape == (k,)
    out = np.empty(s_, np.uint32)
    rc = lib().qo_ftr_reconstruct(_p(resp, _u32p), _p(al, _u32p), k, s_, p, _p(out, _u32p))
    if rc != 0:
        raise ValueError("evaluation points must be distinct")
    return out


class FtrDecodeError(ValueError):
    """Robust reconstruction failed: too few responses or more than
    floor((k - t - 1) / 2) of them wrong."""


def ftr_decode(resp: np.ndarray, alpha, t: int, p: int = FTR_P):
    """Berlekamp-Welch unique decoding (qo_ftr_decode_bw): returns (block, bad)
    where bad[i] = 1 marks server i's response as inconsistent with the decoded
    polynomial.  Raises FtrDecodeError beyond the unique-decoding radius."""
    resp = _c(resp, np.uint32)
    k, s_ = resp.shape
    al = _c(alpha, np.uint32)
    assert al.shape == (k,)
    out = np.empty(s_, np.uint32)
    bad = np.empty(k, np.uint32)
    rc = lib().qo_ftr_decode_bw(_p(resp, _u32p), _p(al, _u32p), k, s_, t, p, _p(out, _u32p),
                                _p(bad, _u32p))
    if rc == -1:
        raise ValueError("evaluation points must be distinct")
    if rc == 1:
        raise FtrDecodeError(f"k = {k} responses <= t = {t}: incomplete")
    if rc == 2:
        raise FtrDecodeError(f"more than {(k - t - 1) // 2} corrupted responses")
    return out, bad.astype(bool)


# ---------------------------------------------------------------- OOP (CIP-PIR, NEXT-3)
def oop_preprocess(records: np.ndarray, n: int, i: int, seed: int) -> np.ndarray:
    rec = _c(records, np.uint8)
    B, d = rec.shape
    assert B % n == 0
    A = np.empty(d, np.uint8)
    lib().qo_oop_preprocess(_p(rec, _u8p), B, d, n, i, seed, _p(A, _u8p))
    return A


def oop_query(theta: int, B: int, n: int, seeds) -> np.ndarray:
    sd = _c(seeds, np.uint64)
    assert sd.shape == (n,) and B % n == 0
    q = np.empty((n, (B // n + 7) // 8), np.uint8)
    lib().qo_oop_query(theta, B, n, _p(sd, _u64p), _p(q, _u8p))
    return q


def oop_respond(records: np.ndarray, n: int, i: int, q_i: np.ndarray, A_i: np.ndarray) -> np.ndarray:
    rec = _c(records, np.uint8)
    B, d = rec.shape
    q = _c(q_i, np.uint8)
    A = _c(A_i, np.uint8)
    out = np.empty(d, np.uint8)
    lib().qo_oop_respond(_p(rec, _u8p), B, d, n, i, _p(q, _u8p), _p(A, _u8p), _p(out, _u8p))
    return out


def num_threads() -> int:
    return int(lib().qo_num_threads())


def set_num_threads(t: int) -> None:
    lib().qo_set_num_threads(t)


# ------------------------------------------------------------------ NEXT-4
HCT_PUZZLE_BYTES = 37     # 32-byte nonce + 4-byte kappa + 1-byte level
SPECTRUM_BYTES = 560


def hct_puzzle_gen(seed_psd: int, theta: int, kappa: int, n_l: int) -> np.ndarray:
    """HCT.Puzzle.Gen of record theta -> 37 bytes (qo_hct_puzzle_gen)."""
    out = np.zeros(HCT_PUZZLE_BYTES, np.uint8)
    lib().qo_hct_puzzle_gen(seed_psd, theta, kappa, n_l, _p(out, _u8p))
    return out


def puzzle_bind_hct(spectrum: np.ndarray, theta0: int, seed_psd: int, kappa: int, n_l: int,
                    d: int) -> np.ndarray:
    """PSD.Puzzle.Bind (Alg. 1 step 1) over records theta0 .. theta0 + n - 1;
    spectrum: n x >= 560 bytes.  Returns n x d records (signature slot zero)."""
    sp = _c(spectrum, np.uint8)
    assert sp.ndim == 2 and sp.shape[1] >= SPECTRUM_BYTES and d >= SPECTRUM_BYTES + HCT_PUZZLE_BYTES
    n = sp.shape[0]
    out = np.empty((n, d), np.uint8)
    lib().qo_puzzle_bind_hct(_p(sp, _u8p), sp.shape[1], theta0, n, seed_psd, kappa, n_l, d,
                             _p(out, _u8p))
    return out


def puzzle_bind_hct_signed(spectrum: np.ndarray, theta0: int, seed_psd: int, kappa: int, n_l: int,
                           d: int, mldsa_seed: bytes) -> np.ndarray:
    """PSD.Puzzle.Bind with the ML-DSA signature of Alg. 1 step 1:
    record = spectrum || pi_theta || sigma, sigma = ML-DSA-44.Sign(sk_PSD, pi_theta)
    (deterministic variant, empty context; oracle/mldsa.py), bytes [597, 3017)."""
    from oracle import mldsa
    assert d >= 3017
    rec = puzzle_bind_hct(spectrum, theta0, seed_psd, kappa, n_l, d)
    for i in range(rec.shape[0]):
        sig = mldsa.sign(mldsa_seed, rec[i, 560:597].tobytes())
        rec[i, 597:3017] = np.frombuffer(sig, np.uint8)
    return rec
