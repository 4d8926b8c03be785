"""ML-DSA-44 (FIPS 204, "Module-Lattice-Based Digital Signature Standard",
August 2024) in plain Python -- the oracle of the NEXT-4 signature step
(Alg. 1 step 1 of the paper, "sigma <- ML-DSA.Sign(sk_PSD, pi_theta)";
the 2420-byte signature of PAPER.md:1688 is ML-DSA-44).

TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py's cpu_baseline).  Written
step by step from FIPS 204 in its order and notation; hashlib's SHAKE128 /
SHAKE256 are the library primitives (H = SHAKE256, G = SHAKE128).  Pinned
against an independent implementation (OpenSSL's ML-DSA through the
`cryptography` package): key generation from a seed must give the library's
public key byte for byte, the library must verify every signature made here,
and this verifier must accept the library's (randomised) signatures and
reject tampered ones (tests/test_oracle_mldsa.py).

Signing is the deterministic variant of FIPS 204 (rnd = {0}^32, Alg. 2 line 5
"or rnd <- {0}^32 for the deterministic variant"), so the GPU signer can be
compared byte for byte.
"""
from __future__ import annotations

import functools
import hashlib

# FIPS 204 Table 1, ML-DSA-44
Q = 8380417
D = 13
TAU = 39
LAMBDA = 128
GAMMA1 = 1 << 17
GAMMA2 = (Q - 1) // 88
K, L = 4, 4
ETA = 2
BETA = TAU * ETA
OMEGA = 80
ZETA = 1753
PK_BYTES, SK_BYTES, SIG_BYTES = 1312, 2560, 2420


def H(data: bytes, n: int) -> bytes:
    return hashlib.shake_256(data).digest(n)


def G(data: bytes, n: int) -> bytes:
    return hashlib.shake_128(data).digest(n)


class _Stream:
    """Incremental squeeze: byte i of the XOF output, extending as needed."""

    def __init__(self, xof, data: bytes, chunk: int):
        self.xof, self.data, self.buf, self.pos, self.chunk = xof, data, b"", 0, chunk

    def read(self, n: int) -> bytes:
        while self.pos + n > len(self.buf):
            self.buf = self.xof(self.data, len(self.buf) + self.chunk)
        out = self.buf[self.pos:self.pos + n]
        self.pos += n
        return out


# ------------------------------------------------------------ conversions (Sec. 7.1)
def _bitlen(a: int) -> int:
    return a.bit_length()


def simple_bit_pack(w, b: int) -> bytes:
    """Alg. 16 SimpleBitPack: coefficients in [0, b], bitlen(b) bits each, LSB first."""
    c = _bitlen(b)
    acc, nb = 0, 0
    for i, x in enumerate(w):
        acc |= x << (i * c)
    nb = 256 * c // 8
    return acc.to_bytes(nb, "little")


def bit_pack(w, a: int, b: int) -> bytes:
    """Alg. 17 BitPack: coefficients in [-a, b], stored as b - w_i in bitlen(a + b) bits."""
    c = _bitlen(a + b)
    acc = 0
    for i, x in enumerate(w):
        acc |= (b - x) << (i * c)
    return acc.to_bytes(256 * c // 8, "little")


def simple_bit_unpack(v: bytes, b: int):
    c = _bitlen(b)
    acc = int.from_bytes(v, "little")
    return [(acc >> (i * c)) & ((1 << c) - 1) for i in range(256)]


def bit_unpack(v: bytes, a: int, b: int):
    """Alg. 19 BitUnpack: w_i = b - (the c-bit field i)."""
    c = _bitlen(a + b)
    acc = int.from_bytes(v, "little")
    return [b - ((acc >> (i * c)) & ((1 << c) - 1)) for i in range(256)]


def hint_bit_pack(h) -> bytes:
    """Alg. 20 HintBitPack."""
    y = [0] * (OMEGA + K)
    index = 0
    for i in range(K):
        for j in range(256):
            if h[i][j] != 0:
                y[index] = j
                index += 1
        y[OMEGA + i] = index
    return bytes(y)


def hint_bit_unpack(y: bytes):
    """Alg. 21 HintBitUnpack (None = malformed)."""
    h = [[0] * 256 for _ in range(K)]
    index = 0
    for i in range(K):
        if y[OMEGA + i] < index or y[OMEGA + i] > OMEGA:
            return None
        first = index
        while index < y[OMEGA + i]:
            if index > first and y[index - 1] >= y[index]:
                return None
            h[i][y[index]] = 1
            index += 1
    for i in range(index, OMEGA):
        if y[i] != 0:
            return None
    return h


def pk_encode(rho: bytes, t1) -> bytes:  # Alg. 22
    return rho + b"".join(simple_bit_pack(t1[i], (1 << (_bitlen(Q - 1) - D)) - 1) for i in range(K))


def pk_decode(pk: bytes):  # Alg. 23
    rho = pk[:32]
    t1 = [simple_bit_unpack(pk[32 + 320 * i:32 + 320 * (i + 1)], (1 << 10) - 1) for i in range(K)]
    return rho, t1


def sk_encode(rho, Kk, tr, s1, s2, t0) -> bytes:  # Alg. 24
    out = rho + Kk + tr
    out += b"".join(bit_pack(s1[i], ETA, ETA) for i in range(L))
    out += b"".join(bit_pack(s2[i], ETA, ETA) for i in range(K))
    out += b"".join(bit_pack(t0[i], (1 << (D - 1)) - 1, 1 << (D - 1)) for i in range(K))
    return out


def sig_encode(c_tilde: bytes, z, h) -> bytes:  # Alg. 26
    return c_tilde + b"".join(bit_pack(z[i], GAMMA1 - 1, GAMMA1) for i in range(L)) + hint_bit_pack(h)


def sig_decode(sig: bytes):  # Alg. 27
    c_tilde = sig[:LAMBDA // 4]
    off = LAMBDA // 4
    z = []
    for i in range(L):
        z.append(bit_unpack(sig[off:off + 576], GAMMA1 - 1, GAMMA1))
        off += 576
    return c_tilde, z, hint_bit_unpack(sig[off:])


def w1_encode(w1) -> bytes:  # Alg. 28
    return b"".join(simple_bit_pack(w1[i], (Q - 1) // (2 * GAMMA2) - 1) for i in range(K))


# ------------------------------------------------------------ sampling (Sec. 7.3)
def sample_in_ball(rho: bytes):
    """Alg. 29 SampleInBall."""
    c = [0] * 256
    st = _Stream(H, rho, 136)
    s = st.read(8)
    hbits = int.from_bytes(s, "little")
    for i in range(256 - TAU, 256):
        j = st.read(1)[0]
        while j > i:
            j = st.read(1)[0]
        c[i] = c[j]
        c[j] = -1 if (hbits >> (i + TAU - 256)) & 1 else 1
    return c


def rej_ntt_poly(rho: bytes):
    """Alg. 30 RejNTTPoly with CoeffFromThreeBytes (Alg. 14)."""
    a = []
    st = _Stream(G, rho, 168 * 5)
    while len(a) < 256:
        s = st.read(3)
        z = ((s[2] & 127) << 16) | (s[1] << 8) | s[0]
        if z < Q:
            a.append(z)
    return a


def _coeff_from_half_byte(b: int):
    """Alg. 15 for eta = 2."""
    if b < 15:
        return 2 - (b % 5)
    return None


def rej_bounded_poly(rho: bytes):
    """Alg. 31 RejBoundedPoly."""
    a = []
    st = _Stream(H, rho, 136 * 2)
    while len(a) < 256:
        z = st.read(1)[0]
        z0 = _coeff_from_half_byte(z % 16)
        z1 = _coeff_from_half_byte(z // 16)
        if z0 is not None:
            a.append(z0)
        if z1 is not None and len(a) < 256:
            a.append(z1)
    return a


def expand_a(rho: bytes):
    """Alg. 32 ExpandA: A[r][s] = RejNTTPoly(rho || s || r)."""
    return [[rej_ntt_poly(rho + bytes([s, r])) for s in range(L)] for r in range(K)]


def expand_s(rho: bytes):
    """Alg. 33 ExpandS."""
    s1 = [rej_bounded_poly(rho + r.to_bytes(2, "little")) for r in range(L)]
    s2 = [rej_bounded_poly(rho + (r + L).to_bytes(2, "little")) for r in range(K)]
    return s1, s2


def expand_mask(rho: bytes, mu: int):
    """Alg. 34 ExpandMask: y[r] = BitUnpack(H(rho || (mu + r), 32c), gamma1 - 1, gamma1)."""
    c = 1 + _bitlen(GAMMA1 - 1)
    return [bit_unpack(H(rho + (mu + r).to_bytes(2, "little"), 32 * c), GAMMA1 - 1, GAMMA1)
            for r in range(L)]


# ------------------------------------------------------------ arithmetic (Sec. 7.4, 7.5)
def mod_pm(r: int, alpha: int) -> int:
    """r mod+- alpha: the representative in (-alpha/2, alpha/2]."""
    r0 = r % alpha
    if r0 > alpha // 2:
        r0 -= alpha
    return r0


def power2round(r: int):  # Alg. 35
    rp = r % Q
    r0 = mod_pm(rp, 1 << D)
    return (rp - r0) >> D, r0


def decompose(r: int):  # Alg. 36
    rp = r % Q
    r0 = mod_pm(rp, 2 * GAMMA2)
    if rp - r0 == Q - 1:
        return 0, r0 - 1
    return (rp - r0) // (2 * GAMMA2), r0


def high_bits(r: int) -> int:  # Alg. 37
    return decompose(r)[0]


def low_bits(r: int) -> int:  # Alg. 38
    return decompose(r)[1]


def make_hint(z: int, r: int) -> int:  # Alg. 39
    return int(high_bits(r) != high_bits(r + z))


def use_hint(h: int, r: int) -> int:  # Alg. 40
    m = (Q - 1) // (2 * GAMMA2)
    r1, r0 = decompose(r)
    if h == 1 and r0 > 0:
        return (r1 + 1) % m
    if h == 1 and r0 <= 0:
        return (r1 - 1) % m
    return r1


def _brv8(m: int) -> int:
    return int(f"{m:08b}"[::-1], 2)


ZETAS = [pow(ZETA, _brv8(m), Q) for m in range(256)]


def ntt(w):
    """Alg. 41 NTT."""
    a = [x % Q for x in w]
    m = 0
    ln = 128
    while ln >= 1:
        start = 0
        while start < 256:
            m += 1
            z = ZETAS[m]
            for j in range(start, start + ln):
                t = z * a[j + ln] % Q
                a[j + ln] = (a[j] - t) % Q
                a[j] = (a[j] + t) % Q
            start += 2 * ln
        ln //= 2
    return a


def ntt_inv(w):
    """Alg. 42 NTT^-1."""
    a = list(w)
    m = 256
    ln = 1
    while ln < 256:
        start = 0
        while start < 256:
            m -= 1
            z = -ZETAS[m]
            for j in range(start, start + ln):
                t = a[j]
                a[j] = (t + a[j + ln]) % Q
                a[j + ln] = (t - a[j + ln]) % Q
                a[j + ln] = z * a[j + ln] % Q
            start += 2 * ln
        ln *= 2
    f = 8347681  # 256^-1 mod q
    return [f * x % Q for x in a]


def _pw(a, b):
    return [x * y % Q for x, y in zip(a, b)]


def _add(a, b):
    return [(x + y) % Q for x, y in zip(a, b)]


def _sub(a, b):
    return [(x - y) % Q for x, y in zip(a, b)]


def _mat_vec(A_hat, v_hat):
    out = []
    for r in range(K):
        acc = [0] * 256
        for s in range(L):
            acc = _add(acc, _pw(A_hat[r][s], v_hat[s]))
        out.append(acc)
    return out


def _inf_norm(vec) -> int:
    return max(abs(mod_pm(x, Q)) for p in vec for x in p)


# ------------------------------------------------------------ internal algorithms (Sec. 6)
def keygen_internal(xi: bytes):
    """Alg. 6 ML-DSA.KeyGen_internal -> (pk, sk)."""
    seed = H(xi + bytes([K, L]), 128)
    rho, rho_p, Kk = seed[:32], seed[32:96], seed[96:128]
    A_hat = expand_a(rho)
    s1, s2 = expand_s(rho_p)
    t = _mat_vec(A_hat, [ntt(p) for p in s1])
    t = [_add(ntt_inv(t[i]), s2[i]) for i in range(K)]
    t1 = [[power2round(x)[0] for x in p] for p in t]
    t0 = [[power2round(x)[1] for x in p] for p in t]
    pk = pk_encode(rho, t1)
    tr = H(pk, 64)
    sk = sk_encode(rho, Kk, tr, s1, s2, t0)
    return pk, sk


@functools.lru_cache(maxsize=8)
def _sk_parts(xi: bytes):
    """The signing key's parts straight from the key generation (equal to
    skDecode(skEncode(...)), Alg. 25): rho, K, tr, s1, s2, t0."""
    seed = H(xi + bytes([K, L]), 128)
    rho, rho_p, Kk = seed[:32], seed[32:96], seed[96:128]
    A_hat = expand_a(rho)
    s1, s2 = expand_s(rho_p)
    t = _mat_vec(A_hat, [ntt(p) for p in s1])
    t = [_add(ntt_inv(t[i]), s2[i]) for i in range(K)]
    t0 = [[power2round(x)[1] for x in p] for p in t]
    t1 = [[power2round(x)[0] for x in p] for p in t]
    tr = H(pk_encode(rho, t1), 64)
    return rho, Kk, tr, s1, s2, t0, A_hat


def sign_internal(xi: bytes, m_prime: bytes, rnd: bytes = bytes(32)) -> bytes:
    """Alg. 7 ML-DSA.Sign_internal (key given by its seed xi)."""
    rho, Kk, tr, s1, s2, t0, A_hat = _sk_parts(xi)
    s1_hat = [ntt(p) for p in s1]
    s2_hat = [ntt(p) for p in s2]
    t0_hat = [ntt(p) for p in t0]
    mu = H(tr + m_prime, 64)
    rho_pp = H(Kk + rnd + mu, 64)
    kappa = 0
    while True:
        y = expand_mask(rho_pp, kappa)
        w = [ntt_inv(p) for p in _mat_vec(A_hat, [ntt(p) for p in y])]
        w1 = [[high_bits(x) for x in p] for p in w]
        c_tilde = H(mu + w1_encode(w1), LAMBDA // 4)
        c = sample_in_ball(c_tilde)
        c_hat = ntt(c)
        cs1 = [ntt_inv(_pw(c_hat, s1_hat[i])) for i in range(L)]
        cs2 = [ntt_inv(_pw(c_hat, s2_hat[i])) for i in range(K)]
        z = [_add(y[i], cs1[i]) for i in range(L)]
        r0 = [[low_bits(x) for x in _sub(w[i], cs2[i])] for i in range(K)]
        kappa += L
        if _inf_norm(z) >= GAMMA1 - BETA or max(abs(x) for p in r0 for x in p) >= GAMMA2 - BETA:
            continue
        ct0 = [ntt_inv(_pw(c_hat, t0_hat[i])) for i in range(K)]
        h = [[make_hint((-ct0[i][j]) % Q, (w[i][j] - cs2[i][j] + ct0[i][j]) % Q) for j in range(256)]
             for i in range(K)]
        if _inf_norm(ct0) >= GAMMA2 or sum(map(sum, h)) > OMEGA:
            continue
        zc = [[mod_pm(x, Q) for x in p] for p in z]
        return sig_encode(c_tilde, zc, h)


def verify_internal(pk: bytes, m_prime: bytes, sig: bytes) -> bool:
    """Alg. 8 ML-DSA.Verify_internal."""
    if len(pk) != PK_BYTES or len(sig) != SIG_BYTES:
        return False
    rho, t1 = pk_decode(pk)
    c_tilde, z, h = sig_decode(sig)
    if h is None:
        return False
    A_hat = expand_a(rho)
    tr = H(pk, 64)
    mu = H(tr + m_prime, 64)
    c = sample_in_ball(c_tilde)
    c_hat = ntt(c)
    az = _mat_vec(A_hat, [ntt([x % Q for x in p]) for p in z])
    t1_hat = [ntt([(x << D) % Q for x in p]) for p in t1]
    w_approx = [ntt_inv(_sub(az[i], _pw(c_hat, t1_hat[i]))) for i in range(K)]
    w1 = [[use_hint(h[i][j], w_approx[i][j]) for j in range(256)] for i in range(K)]
    c_tilde2 = H(mu + w1_encode(w1), LAMBDA // 4)
    znorm = max(abs(x) for p in z for x in p)
    return znorm < GAMMA1 - BETA and c_tilde == c_tilde2


def _m_prime(msg: bytes, ctx: bytes = b"") -> bytes:
    """Alg. 2 line 10 / Alg. 3 line 5: M' = 0 || |ctx| || ctx || M (pure ML-DSA)."""
    assert len(ctx) <= 255
    return bytes([0, len(ctx)]) + ctx + msg


def keygen(xi: bytes):
    """ML-DSA.KeyGen with the seed given (Alg. 1 without the RNG)."""
    return keygen_internal(xi)


def sign(xi: bytes, msg: bytes, ctx: bytes = b"") -> bytes:
    """ML-DSA.Sign, deterministic variant (rnd = {0}^32)."""
    return sign_internal(xi, _m_prime(msg, ctx))


def verify(pk: bytes, msg: bytes, sig: bytes, ctx: bytes = b"") -> bool:
    return verify_internal(pk, _m_prime(msg, ctx), sig)
