"""Pins of the ML-DSA-44 oracle (oracle/mldsa.py, FIPS 204) against an
independent implementation (OpenSSL's ML-DSA via the `cryptography` package)
and against plain definitions -- NEXT-4 signature step."""
import random

import pytest

from oracle import mldsa as M

lib = pytest.importorskip("cryptography.hazmat.primitives.asymmetric.mldsa")


def _seed(i):
    return bytes((i * 37 + j * 11) & 0xFF for j in range(32))


def test_sizes_match_fips204_and_the_paper():
    # FIPS 204 Table 2 (ML-DSA-44): pk 1312, sk 2560, sig 2420; "2420 bytes"
    pk, sk = M.keygen(_seed(1))
    assert (len(pk), len(sk)) == (1312, 2560)
    assert len(M.sign(_seed(1), b"x")) == 2420


@pytest.mark.parametrize("i", range(4))
def test_keygen_matches_library(i):
    """KeyGen_internal from a seed gives the library's public key byte for byte
    (pins ExpandA, ExpandS, NTT / NTT^-1, Power2Round, pkEncode)."""
    xi = _seed(i)
    pk, _ = M.keygen(xi)
    assert pk == lib.MLDSA44PrivateKey.from_seed_bytes(xi).public_key().public_bytes_raw()


@pytest.mark.parametrize("i,msg,ctx", [(0, b"", b""), (1, b"puzzle" * 7, b""),
                                       (2, bytes(37), b"PSD"), (3, bytes(range(200)), b"")])
def test_library_verifies_oracle_signatures(i, msg, ctx):
    """Every deterministic oracle signature is accepted by the library's verifier
    (pins ExpandMask, SampleInBall, the hint, the rejection conditions, sigEncode)."""
    xi = _seed(i)
    sig = M.sign(xi, msg, ctx)
    pub = lib.MLDSA44PrivateKey.from_seed_bytes(xi).public_key()
    pub.verify(sig, msg, ctx if ctx else None)  # raises InvalidSignature on failure


def test_oracle_verifies_library_signatures_and_rejects_tampering():
    xi = _seed(5)
    pk, _ = M.keygen(xi)
    key = lib.MLDSA44PrivateKey.from_seed_bytes(xi)
    for msg in (b"a", b"record 17", bytes(37)):
        sig = key.sign(msg)  # hedged (randomised) signature of the library
        assert M.verify(pk, msg, sig)
        assert not M.verify(pk, msg + b"!", sig)
        bad = bytearray(sig)
        bad[100] ^= 1
        assert not M.verify(pk, msg, bytes(bad))
        assert not M.verify(pk, msg, sig, b"ctx")


def test_signing_is_deterministic():
    assert M.sign(_seed(7), b"m") == M.sign(_seed(7), b"m")
    assert M.sign(_seed(7), b"m") != M.sign(_seed(7), b"n")


def test_ntt_is_negacyclic_convolution():
    """NTT^-1(NTT(a) o NTT(b)) = a * b mod (X^256 + 1, q): schoolbook product."""
    rng = random.Random(3)
    a = [rng.randrange(M.Q) for _ in range(256)]
    b = [rng.randrange(M.Q) for _ in range(256)]
    want = [0] * 256
    for i in range(256):
        for j in range(256):
            k, s = (i + j) % 256, (1 if i + j < 256 else -1)
            want[k] = (want[k] + s * a[i] * b[j]) % M.Q
    got = M.ntt_inv([x * y % M.Q for x, y in zip(M.ntt(a), M.ntt(b))])
    assert got == want
    assert M.ntt_inv(M.ntt(a)) == a


def test_decompose_and_hints_closed_forms():
    """Decompose: r = r1 * 2 gamma2 + r0 (mod q), r1 in [0, 43]; UseHint(MakeHint(z, r), r)
    = HighBits(r + z) whenever |z| <= gamma2 (FIPS 204 Lemma 1-style property)."""
    rng = random.Random(4)
    for _ in range(2000):
        r = rng.randrange(M.Q)
        r1, r0 = M.decompose(r)
        assert 0 <= r1 <= 43 and (r1 * 2 * M.GAMMA2 + r0 - r) % M.Q == 0
        z = rng.randrange(-M.GAMMA2, M.GAMMA2 + 1)
        h = M.make_hint(z % M.Q, r)
        assert M.use_hint(h, r) == M.high_bits((r + z) % M.Q)
