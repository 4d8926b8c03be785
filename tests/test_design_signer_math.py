"""CPU checks of the ML-DSA signer's lane index arithmetic and constants
(csrc/mldsa.cuh), emulated lane by lane in Python and compared with the plain
definitions: Keccak-f[1600] (FIPS 202 Sec. 3.2, checked against hashlib's
SHAKE256), the NTT / NTT^-1 of FIPS 204 Alg. 41 / 42, and the Montgomery
constants.  The GPU signatures themselves are pinned byte for byte against the
oracle (tests/test_gpu_bind.py); these tests pin the layouts that the CUDA code
uses, so a wrong lane table shows up on a CPU-only machine."""
import hashlib
import random
import re
from pathlib import Path

SRC = (Path(__file__).resolve().parents[1] / "paper_2510_03631_b200" / "csrc" / "mldsa.cuh").read_text()
M64 = (1 << 64) - 1
RC = [int(x, 16) for x in re.findall(r"0x([0-9a-f]{16})ull", SRC[SRC.index("kRC[24]"):SRC.index("kRC[24]") + 1400])]
RHO = [0, 1, 62, 28, 27, 36, 44, 6, 55, 20, 3, 10, 43, 25, 39, 41, 45, 15, 21, 8, 18, 2, 61, 56, 14]
Q = 8380417


def _const(name):
    return int(re.search(name + r"\s*=\s*(\d+)u?;", SRC).group(1))


def rol(v, r):
    return ((v << r) | (v >> (64 - r))) & M64 if r else v


def keccak_f(A):
    """FIPS 202 Sec. 3.2: theta, rho, pi, chi, iota on A[x + 5y]."""
    A = list(A)
    for rd in range(24):
        C = [A[x] ^ A[x + 5] ^ A[x + 10] ^ A[x + 15] ^ A[x + 20] for x in range(5)]
        D = [C[(x - 1) % 5] ^ rol(C[(x + 1) % 5], 1) for x in range(5)]
        A = [A[i] ^ D[i % 5] for i in range(25)]
        B = [0] * 25
        for x in range(5):
            for y in range(5):
                B[y + 5 * ((2 * x + 3 * y) % 5)] = rol(A[x + 5 * y], RHO[x + 5 * y])
        A = [B[i] ^ ((~B[(i % 5 + 1) % 5 + 5 * (i // 5)] & M64) & B[(i % 5 + 2) % 5 + 5 * (i // 5)])
             for i in range(25)]
        A[0] ^= RC[rd]
    return A


def _cmod(a, b):  # C's % (sign of the dividend)
    r = abs(a) % b
    return -r if a < 0 else r


def _funnel(lo, hi, s):  # __funnelshift_l(lo, hi, s): upper 32 bits of (hi:lo) << s
    return ((((hi << 32) | lo) << s) >> 32) & 0xFFFFFFFF


def _rol_lane(v, sw, rr):  # rol_lane(): half swap, two funnel shifts
    lo, hi = v & 0xFFFFFFFF, v >> 32
    x0, x1 = (hi, lo) if sw else (lo, hi)
    return (_funnel(x0, x1, rr) << 32) | _funnel(x1, x0, rr)


def warp25(A):
    """keccak_warp_n<1> with the KLane tables: lane i < 25 holds A[i]."""
    K = []
    for lane in range(32):
        l = lane if lane < 25 else 0
        x, y = l % 5, l // 5
        pisrc = lambda X, Y: (3 * (_cmod(Y - 3 * X, 5) + 10)) % 5 + 5 * X  # noqa: E731
        r = RHO[l]
        K.append(dict(c1=x + 5 * ((y + 1) % 5), c2=x + 5 * ((y + 2) % 5), c4=x + 5 * ((y + 4) % 5),
                      xm1=(x + 4) % 5 + 5 * y, xp1=(x + 1) % 5 + 5 * y, p0=pisrc(x, y),
                      p1=pisrc((x + 1) % 5, y), p2=pisrc((x + 2) % 5, y), sw=int(r >= 32), rr=r & 31,
                      rc=M64 if lane == 0 else 0))
    a = list(A) + [0] * 7
    for rd in range(24):
        sh = lambda v, f: [v[K[l][f]] for l in range(32)]  # noqa: E731
        t4 = sh(a, "c4")
        s1 = [a[l] ^ v for l, v in enumerate(sh(a, "c1"))]
        c = [s1[l] ^ v ^ t4[l] for l, v in enumerate(sh(s1, "c2"))]
        cm, cp = sh(c, "xm1"), sh(c, "xp1")
        a = [_rol_lane(a[l] ^ cm[l] ^ rol(cp[l], 1), K[l]["sw"], K[l]["rr"]) for l in range(32)]
        b0, b1, b2 = sh(a, "p0"), sh(a, "p1"), sh(a, "p2")
        a = [b0[l] ^ ((~b1[l] & M64) & b2[l]) ^ (RC[rd] & K[l]["rc"]) for l in range(32)]
    return a[:25]


def col4(states):
    """keccak_col4 with the KCol tables: lane 5s + x holds column x of state s;
    pi / chi through the shared buffer (row stride KC_ROW words)."""
    row = _const("KC_ROW")
    a = [[states[min(l // 5, 3)][l % 5 + 5 * y] for y in range(5)] for l in range(32)]
    pis = [0] * 512
    for rd in range(24):
        C = [a[l][0] ^ a[l][1] ^ a[l][2] ^ a[l][3] ^ a[l][4] for l in range(32)]
        new = []
        for l in range(32):
            s, x = min(l // 5, 3), l % 5
            cm, cp = C[5 * s + (x + 4) % 5], C[5 * s + (x + 1) % 5]
            d = cm ^ rol(cp, 1)
            vals = []
            for y in range(5):
                r = RHO[x + 5 * y]
                vals.append((row * ((2 * x + 3 * y) % 5) + 5 * s + y, _rol_lane(a[l][y] ^ d, r >= 32, r & 31)))
            new.append(vals)
        for l in range(20):  # lanes 20..31 never store
            for idx, v in new[l]:
                pis[idx] = v
        for l in range(32):
            s, x = min(l // 5, 3), l % 5
            o0, o1, o2 = 5 * s + x, 5 * s + (x + 1) % 5, 5 * s + (x + 2) % 5
            a[l] = [pis[o0 + row * y] ^ ((~pis[o1 + row * y] & M64) & pis[o2 + row * y]) for y in range(5)]
            if x == 0:
                a[l][0] ^= RC[rd]
    return [[a[5 * s + x][y] for y in range(5) for x in range(5)] for s in range(4)]


def test_round_constants_and_plain_keccak_match_hashlib():
    assert len(RC) == 24 and RC[0] == 1 and RC[23] == 0x8000000080008008
    st = [0] * 25
    blk = bytearray(136)
    blk[0] ^= 0x1F
    blk[135] ^= 0x80
    for i in range(17):
        st[i] ^= int.from_bytes(blk[8 * i:8 * i + 8], "little")
    out = b"".join(v.to_bytes(8, "little") for v in keccak_f(st)[:4])
    assert out == hashlib.shake_256(b"").digest(32)


def test_warp_cooperative_layout_is_keccak_f():
    rng = random.Random(1)
    for _ in range(3):
        st = [rng.getrandbits(64) for _ in range(25)]
        assert warp25(st) == keccak_f(st)


def test_column_layout_is_keccak_f_for_four_states():
    rng = random.Random(2)
    st = [[rng.getrandbits(64) for _ in range(25)] for _ in range(4)]
    got = col4(st)
    for s in range(4):
        assert [got[s][i] for i in range(25)] == keccak_f(st[s])


def _zetas():
    brv = lambda m: int(f"{m:08b}"[::-1], 2)  # noqa: E731
    return [pow(1753, brv(m), Q) for m in range(256)]


def _ntt_ref(w, Z):  # FIPS 204 Alg. 41
    w, m, ln = list(w), 0, 128
    while ln >= 1:
        for st in range(0, 256, 2 * ln):
            m += 1
            for j in range(st, st + ln):
                t = Z[m] * w[j + ln] % Q
                w[j + ln], w[j] = (w[j] - t) % Q, (w[j] + t) % Q
        ln //= 2
    return w


def _intt_ref(w, Z):  # FIPS 204 Alg. 42
    w, m, ln = list(w), 256, 1
    while ln < 256:
        for st in range(0, 256, 2 * ln):
            m -= 1
            z = -Z[m] % Q
            for j in range(st, st + ln):
                t = w[j]
                w[j], w[j + ln] = (t + w[j + ln]) % Q, z * (t - w[j + ln]) % Q
        ln *= 2
    return [x * 8347681 % Q for x in w]


def _montq(a, b):  # montq(): a b 2^-32 mod q for a, b in [0, q)
    x = a * b
    m = (x & 0xFFFFFFFF) * _const("MONT_QINV_NEG") & 0xFFFFFFFF
    t = (x + m * Q) >> 32
    assert t < 2 * Q
    return min(t, (t - Q) & 0xFFFFFFFF)


def _ntt4(w, ZR):  # ntt_w: radix 4, Montgomery twiddles
    w = list(w)
    for lg in (7, 5, 3, 1):
        ln, h = 1 << lg, 1 << (lg - 1)
        for uu in range(64):
            grp = uu >> (lg - 1)
            b = (grp << (lg + 1)) + (uu & (h - 1))
            z1, z2, z3 = ZR[(128 >> lg) + grp], ZR[(256 >> lg) + 2 * grp], ZR[(256 >> lg) + 2 * grp + 1]
            a0, a1, a2, a3 = w[b], w[b + h], w[b + ln], w[b + ln + h]
            t = _montq(z1, a2); a2, a0 = (a0 - t) % Q, (a0 + t) % Q  # noqa: E702
            t = _montq(z1, a3); a3, a1 = (a1 - t) % Q, (a1 + t) % Q  # noqa: E702
            t = _montq(z2, a1); a1, a0 = (a0 - t) % Q, (a0 + t) % Q  # noqa: E702
            t = _montq(z3, a3); a3, a2 = (a2 - t) % Q, (a2 + t) % Q  # noqa: E702
            w[b], w[b + h], w[b + ln], w[b + ln + h] = a0, a1, a2, a3
    return w


def _intt4(w, ZR):  # ntt_inv_w: radix 4, 256^-1 fused into the last pass
    w, F = list(w), _const("MONT_F")
    for lg in (0, 2, 4, 6):
        ln = 1 << lg
        for uu in range(64):
            g = uu >> lg
            b = (g << (lg + 2)) + (uu & (ln - 1))
            za, zb = Q - ZR[(256 >> lg) - 1 - 2 * g], Q - ZR[(256 >> lg) - 2 - 2 * g]
            zc = Q - ZR[(128 >> lg) - 1 - g]
            a0, a1, a2, a3 = w[b], w[b + ln], w[b + 2 * ln], w[b + 3 * ln]
            t = a0; a0, a1 = (t + a1) % Q, _montq(za, (t - a1) % Q)  # noqa: E702
            t = a2; a2, a3 = (t + a3) % Q, _montq(zb, (t - a3) % Q)  # noqa: E702
            t = a0; a0, a2 = (t + a2) % Q, _montq(zc, (t - a2) % Q)  # noqa: E702
            t = a1; a1, a3 = (t + a3) % Q, _montq(zc, (t - a3) % Q)  # noqa: E702
            if lg == 6:
                a0, a1, a2, a3 = (_montq(F, v) for v in (a0, a1, a2, a3))
            w[b], w[b + ln], w[b + 2 * ln], w[b + 3 * ln] = a0, a1, a2, a3
    return w


def test_montgomery_constants():
    R = 1 << 32
    assert _const("MONT_QINV_NEG") == (-pow(Q, -1, R)) % R
    assert int(re.search(r"MONT_R = (\d+);", SRC).group(1)) == R % Q
    assert _const("MONT_F") == pow(256, -1, Q) * R % Q
    rng = random.Random(3)
    for _ in range(20000):
        a, b = rng.randrange(Q), rng.randrange(Q)
        assert _montq(a * R % Q, b) == a * b % Q
    for a in (0, 1, Q - 1):
        for b in (0, 1, Q - 1):
            assert _montq(a * R % Q, b) == a * b % Q


def test_radix4_warp_ntt_is_alg41_and_alg42():
    Z = _zetas()
    ZR = [z * (1 << 32) % Q for z in Z]
    rng = random.Random(4)
    for _ in range(3):
        v = [rng.randrange(Q) for _ in range(256)]
        assert _ntt4(v, ZR) == _ntt_ref(v, Z)
        assert _intt4(v, ZR) == _intt_ref(v, Z)
        assert _intt_ref(_ntt_ref(v, Z), Z) == v
