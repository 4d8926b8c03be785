// mldsa.cuh -- NEXT-4: ML-DSA-44 signing of the HCT puzzles on the GPU (Alg. 1
// step 1, "sigma <- ML-DSA.Sign(sk_PSD, pi_theta)"; 2420-byte
// signature), written from FIPS 204 (August 2024): Keccak-f[1600]
// / SHAKE, ExpandA / ExpandS / ExpandMask, NTT mod q = 8380417, SampleInBall,
// Decompose / MakeHint, the encodings.  Deterministic variant (rnd = {0}^32),
// pure ML-DSA with an empty context: M' = 0x00 || 0x00 || pi_theta.
//
// Two kernels:
//   mldsa_keygen_kernel  (1 CTA)   -- KeyGen_internal(xi) into an MldsaKey in
//                                      global memory (A-hat, NTT(s1), NTT(s2),
//                                      NTT(t0), K, tr, pk), once per bind call;
//   mldsa_sign_kernel    (persistent warps, one record per warp at a time) --
//                                      Sign_internal of pi_theta; the 2420
//                                      signature bytes go to byte 597 of the
//                                      record's 3024-byte staging row (16-byte
//                                      aligned for the packing kernel).
// KeyGen's sponges run one per thread (byte-serial absorb / squeeze) and its
// polynomial arithmetic across the CTA; the signer's sponges and NTTs are
// warp-cooperative (see mldsa_sign_kernel).
#pragma once
#include <algorithm>
#include <cstdint>

#include "philox.cuh"

namespace qpir {
namespace mldsa {

constexpr int32_t Q = 8380417;
constexpr int32_t D_ = 13;
constexpr int32_t TAU = 39;
constexpr int32_t GAMMA1 = 1 << 17;
constexpr int32_t GAMMA2 = (Q - 1) / 88;
constexpr int K = 4, L = 4;
constexpr int32_t ETA = 2;
constexpr int32_t BETA = TAU * ETA;
constexpr int OMEGA = 80;
constexpr int PK_BYTES = 1312, SIG_BYTES = 2420;
constexpr int SIG_OFF = 597;      // record byte of the signature (560 spectrum + 37 puzzle)
constexpr int REC_STAGE = 3024;   // staging row: 3017 bytes rounded up to 16
constexpr int THREADS = 256;

struct MldsaKey {                 // expanded signing key (global memory); the four
  int32_t A[K][L][256];           // A-hat (NTT domain)      polynomial arrays end in
  int32_t s1[L][256];             // NTT(s1)                 Montgomery form (x 2^32 mod q)
  int32_t s2[K][256];             // NTT(s2)                 for the signer's montq
  int32_t t0[K][256];             // NTT(t0)
  uint8_t Kseed[32];
  uint8_t tr[64];
  uint8_t pk[PK_BYTES];
};

// ------------------------------------------------------------------ Keccak / SHAKE
static __constant__ uint64_t kRC[24] = {
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808aull, 0x8000000080008000ull,
    0x000000000000808bull, 0x0000000080000001ull, 0x8000000080008081ull, 0x8000000000008009ull,
    0x000000000000008aull, 0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000aull,
    0x000000008000808bull, 0x800000000000008bull, 0x8000000000008089ull, 0x8000000000008003ull,
    0x8000000000008002ull, 0x8000000000000080ull, 0x000000000000800aull, 0x800000008000000aull,
    0x8000000080008081ull, 0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};

__device__ __forceinline__ uint64_t rol64(uint64_t x, int s) { return (x << s) | (x >> (64 - s)); }

// Keccak-f[1600] (FIPS 202 Sec. 3.3): theta, rho + pi, chi, iota; 24 rounds.
static __device__ __noinline__ void keccak_f1600(uint64_t* A) {
  constexpr int rotc[24] = {1, 3, 6, 10, 15, 21, 28, 36, 45, 55, 2, 14, 27, 41, 56, 8, 25, 43, 62, 18, 39, 61, 20, 44};
  constexpr int piln[24] = {10, 7, 11, 17, 18, 3, 5, 16, 8, 21, 24, 4, 15, 23, 19, 13, 12, 2, 20, 14, 22, 9, 6, 1};
  uint64_t st[25];
#pragma unroll
  for (int i = 0; i < 25; ++i) st[i] = A[i];
#pragma unroll 1
  for (int r = 0; r < 24; ++r) {
    uint64_t bc[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) bc[i] = st[i] ^ st[i + 5] ^ st[i + 10] ^ st[i + 15] ^ st[i + 20];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const uint64_t t = bc[(i + 4) % 5] ^ rol64(bc[(i + 1) % 5], 1);
#pragma unroll
      for (int j = 0; j < 25; j += 5) st[j + i] ^= t;
    }
    uint64_t t = st[1];
#pragma unroll
    for (int i = 0; i < 24; ++i) {
      const int j = piln[i];
      const uint64_t b = st[j];
      st[j] = rol64(t, rotc[i]);
      t = b;
    }
#pragma unroll
    for (int j = 0; j < 25; j += 5) {
      uint64_t b[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) b[i] = st[j + i];
#pragma unroll
      for (int i = 0; i < 5; ++i) st[j + i] ^= (~b[(i + 1) % 5]) & b[(i + 2) % 5];
    }
    st[0] ^= kRC[r];
  }
#pragma unroll
  for (int i = 0; i < 25; ++i) A[i] = st[i];
}

// SHAKE128 (rate 168) / SHAKE256 (rate 136) sponge, one thread, byte-serial.
struct Shake {
  uint64_t A[25];
  uint32_t pos, rate;
  __device__ void init(uint32_t r) {
    for (int i = 0; i < 25; ++i) A[i] = 0;
    pos = 0;
    rate = r;
  }
  __device__ void absorb(const uint8_t* p, uint32_t n) {
    for (uint32_t i = 0; i < n; ++i) {
      A[pos >> 3] ^= (uint64_t)p[i] << (8 * (pos & 7));
      if (++pos == rate) {
        keccak_f1600(A);
        pos = 0;
      }
    }
  }
  __device__ void absorb_byte(uint8_t b) { absorb(&b, 1); }
  __device__ void finalize() {  // SHAKE domain bits 1111 + pad10*1 (FIPS 202)
    A[pos >> 3] ^= 0x1Full << (8 * (pos & 7));
    A[(rate - 1) >> 3] ^= 0x80ull << (8 * ((rate - 1) & 7));
    keccak_f1600(A);
    pos = 0;
  }
  __device__ uint8_t squeeze_byte() {
    if (pos == rate) {
      keccak_f1600(A);
      pos = 0;
    }
    const uint8_t b = (uint8_t)(A[pos >> 3] >> (8 * (pos & 7)));
    ++pos;
    return b;
  }
  __device__ void squeeze(uint8_t* out, uint32_t n) {
    for (uint32_t i = 0; i < n; ++i) out[i] = squeeze_byte();
  }
};

// Warp-cooperative Keccak-f[1600]: lane i < 25 holds state word A[x + 5y]
// (x = i % 5, y = i / 5); theta's column parities, pi's lane permutation and
// chi's row neighbours move through warp shuffles (FIPS 202 Sec. 3.2 steps).
// Lanes 25..31 take part in the shuffles with a dummy word.
__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src);
  const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t rolv(uint64_t x, int s) { return s ? (x << s) | (x >> (64 - s)) : x; }

// Per-lane constants of the warp-cooperative round (lane i < 25 holds A[x + 5y];
// lanes 25..31 shadow lane 0 and are never read).
// Built once per CTA into a shared table (k_lane_tab) so a permutation call
// loads them instead of re-deriving ~150 instructions of index arithmetic.
struct alignas(16) KLane {
  int c1, c2, c4;   // A[x][y+1], A[x][y+2]-partner, A[x][y+4]: theta's column sum in 3 shuffles
  int xm1, xp1;     // C[x-1], C[x+1]
  int p0, p1, p2;   // pi sources of B[x][y], B[x+1][y], B[x+2][y] (chi reads them directly)
  int sw, rr;       // rho offset r[x][y] = 32 sw + rr
  uint64_t rcmask;  // lane 0: iota applies
  __device__ __forceinline__ void init(int lane) {
    // rho offsets r[x][y] (FIPS 202 Table 2), indexed x + 5y
    constexpr uint32_t rho[25] = {0, 1, 62, 28, 27, 36, 44, 6, 55, 20, 3, 10, 43, 25, 39,
                                  41, 45, 15, 21, 8, 18, 2, 61, 56, 14};
    const int l = lane < 25 ? lane : 0;
    const int x = l % 5, y = l / 5;
    c1 = x + 5 * ((y + 1) % 5);
    c2 = x + 5 * ((y + 2) % 5);
    c4 = x + 5 * ((y + 4) % 5);
    xm1 = (x + 4) % 5 + 5 * y;
    xp1 = (x + 1) % 5 + 5 * y;
    // pi: B[X][Y] = A[x][y] with X = y, Y = 2x + 3y: lane (X, Y) reads source
    // x = 3 (Y - 3X) mod 5, y = X
    auto pisrc = [](int X, int Y) { return (3 * ((Y - 3 * X) % 5 + 10)) % 5 + 5 * X; };
    p0 = pisrc(x, y);
    p1 = pisrc((x + 1) % 5, y);
    p2 = pisrc((x + 2) % 5, y);
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 25; ++i) r = i == l ? rho[i] : r;  // no local-memory table
    sw = r >= 32;
    rr = r & 31;
    rcmask = lane == 0 ? ~0ull : 0ull;
  }
};

// rotate left by the lane's rho offset: a half swap, then two funnel shifts
__device__ __forceinline__ uint64_t rol_lane(uint64_t v, int sw, int rr) {
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  const uint32_t x0 = sw ? hi : lo, x1 = sw ? lo : hi;
  return ((uint64_t)__funnelshift_l(x0, x1, rr) << 32) | __funnelshift_l(x1, x0, rr);
}

// S independent states, one Keccak-f[1600] each (FIPS 202 Sec. 3.2 steps), their
// rounds interleaved so the shuffles of one state overlap the others' arithmetic.
// Per round and state 8 64-bit shuffles: theta's column sum as a 3-step chain,
// C[x -/+ 1], and B[x], B[x+1], B[x+2] straight from the rho-rotated words.
template <int S>
__device__ __forceinline__ void keccak_warp_n(uint64_t (&a)[S], const KLane& k) {
#pragma unroll 1
  for (int rd = 0; rd < 24; ++rd) {
    uint64_t c[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const uint64_t t4 = shfl64(a[s], k.c4);
      const uint64_t s1 = a[s] ^ shfl64(a[s], k.c1);      // A[y] ^ A[y+1]
      c[s] = s1 ^ shfl64(s1, k.c2) ^ t4;                   // ^ A[y+2] ^ A[y+3], ^ A[y+4]
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const uint64_t cm = shfl64(c[s], k.xm1), cp = shfl64(c[s], k.xp1);
      a[s] = rol_lane(a[s] ^ cm ^ rolv(cp, 1), k.sw, k.rr);  // theta, then rho
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const uint64_t b0 = shfl64(a[s], k.p0), b1 = shfl64(a[s], k.p1), b2 = shfl64(a[s], k.p2);
      a[s] = b0 ^ (~b1 & b2) ^ (kRC[rd] & k.rcmask);     // pi, chi, iota
    }
  }
}

static __shared__ KLane k_lane_tab[32];

static __device__ __noinline__ uint64_t keccak_warp(uint64_t a, int lane) {
  const KLane k = k_lane_tab[lane];
  uint64_t st[1] = {a};
  keccak_warp_n<1>(st, k);
  return st[0];
}

// Four independent states in column layout: lane 5s + x (s < 4, x < 5) holds
// column x of state s, a[y] = A[x][y]. theta's column sum is local, C[x -/+ 1]
// two shuffles; rho rotates in registers; pi and chi's row neighbours go through
// 864 bytes of shared memory (each lane stores its five rotated words at their
// pi destinations B[y][2x + 3y], then reads row Y of columns x, x+1, x+2).
// Per round for all four states: 4 shuffles, 5 stores, 15 loads, ~50 ALU
// instructions (the 25-lane layout above: 64 shuffles, ~120 ALU).
// Lanes 20..31 compute on garbage and never store. `pis`: 200 words per warp.
constexpr int KC_ROW = 22;  // pi buffer row stride in words (bank spread of the stores)
// Per-lane constants of the column layout, built once per CTA (k_col_tab).
struct alignas(16) KCol {
  int sw[5], rr[5];  // rho offsets r[x][y] = 32 sw + rr of the lane's column x
  int dst[5];        // pi destination word of A[x][y]: B[y][2x + 3y] at 22 Y + 5 s + X
  int o0, o1, o2;    // row-0 words of columns x, x+1, x+2 of the lane's state
  int xm1, xp1;      // C[x-1], C[x+1]
  uint64_t rcm;      // column 0: iota applies
  __device__ __forceinline__ void init(int lane) {
    constexpr uint32_t rho[25] = {0, 1, 62, 28, 27, 36, 44, 6, 55, 20, 3, 10, 43, 25, 39,
                                  41, 45, 15, 21, 8, 18, 2, 61, 56, 14};
    // lanes 20..31 shadow state 3 (same words: their loads broadcast, no conflicts)
    const int s = min(lane / 5, 3), x = lane % 5;
    xm1 = 5 * s + (x + 4) % 5;
    xp1 = 5 * s + (x + 1) % 5;
    for (int y = 0; y < 5; ++y) {
      const uint32_t r = rho[x + 5 * y];
      sw[y] = r >= 32;
      rr[y] = r & 31;
      dst[y] = KC_ROW * ((2 * x + 3 * y) % 5) + 5 * s + y;
    }
    o0 = 5 * s + x;  // row Y at + 22 Y: a warp's loads hit consecutive words
    o1 = 5 * s + (x + 1) % 5;
    o2 = 5 * s + (x + 2) % 5;
    rcm = x == 0 ? ~0ull : 0ull;
  }
};
static __shared__ KCol k_col_tab[32];

__device__ __forceinline__ void keccak_col4(uint64_t (&a)[5], uint64_t* pis, int lane) {
  const KCol& kt = k_col_tab[lane];
  int sw[5], rr[5], dst[5];
#pragma unroll
  for (int y = 0; y < 5; ++y) {
    sw[y] = kt.sw[y];
    rr[y] = kt.rr[y];
    dst[y] = kt.dst[y];
  }
  const int xm1 = kt.xm1, xp1 = kt.xp1;
  const uint64_t rcm = kt.rcm;
  const bool st = lane < 20;
  const uint64_t* r0 = pis + kt.o0;
  const uint64_t* r1 = pis + kt.o1;
  const uint64_t* r2 = pis + kt.o2;
#pragma unroll 1
  for (int rd = 0; rd < 24; ++rd) {
    const uint64_t c = a[0] ^ a[1] ^ a[2] ^ a[3] ^ a[4];
    const uint64_t cm = shfl64(c, xm1), cp = shfl64(c, xp1);
    const uint64_t d = cm ^ rolv(cp, 1);
#pragma unroll
    for (int y = 0; y < 5; ++y) {
      const uint64_t v = rol_lane(a[y] ^ d, sw[y], rr[y]);
      if (st) pis[dst[y]] = v;
    }
    __syncwarp();
#pragma unroll
    for (int y = 0; y < 5; ++y) a[y] = r0[KC_ROW * y] ^ (~r1[KC_ROW * y] & r2[KC_ROW * y]);
    a[0] ^= kRC[rd] & rcm;
    __syncwarp();
  }
}

// Warp sponge (SHAKE rate RATE): absorb p0 || p1 || p2 with the SHAKE padding;
// the whole warp calls it; scratch: RATE bytes, 8-byte aligned, per warp.
template <int RATE>
__device__ void wsp_absorb(uint64_t& a, const uint8_t* p0, int n0, const uint8_t* p1, int n1,
                           const uint8_t* p2, int n2, uint8_t* scratch, int lane) {
  const int total = n0 + n1 + n2;
  for (int off = 0;; off += RATE) {
    const int take = min(RATE, total - off);
    for (int i = lane; i < RATE; i += 32) {
      const int m = off + i;
      uint8_t v = 0;
      if (i < take) v = m < n0 ? p0[m] : m < n0 + n1 ? p1[m - n0] : p2[m - n0 - n1];
      if (take < RATE) {
        if (i == take) v ^= 0x1F;
        if (i == RATE - 1) v ^= 0x80;
      }
      scratch[i] = v;
    }
    __syncwarp();
    if (lane < RATE / 8) a ^= reinterpret_cast<const uint64_t*>(scratch)[lane];
    a = keccak_warp(a, lane);
    __syncwarp();
    if (take < RATE) return;
  }
}
template <int RATE>
__device__ __forceinline__ void wsp_out(uint64_t a, uint8_t* out, int lane) {  // RATE bytes
  if (lane < RATE / 8) reinterpret_cast<uint64_t*>(out)[lane] = a;
  __syncwarp();
}

// ------------------------------------------------------------------ arithmetic
__device__ __forceinline__ int32_t mulq(int32_t a, int32_t b) {  // a, b in [0, q)
  // Barrett: x < 2^46, qt = floor(x * floor(2^64 / q) / 2^64) is floor(x / q) or one less
  const uint64_t x = (uint64_t)(uint32_t)a * (uint32_t)b;
  const uint64_t qt = __umul64hi(x, 2201172575745ull);
  uint32_t r = (uint32_t)(x - qt * (uint64_t)Q);
  return (int32_t)(r >= (uint32_t)Q ? r - Q : r);
}
// Montgomery product a b 2^-32 mod q for a, b in [0, q) (one operand carries the
// factor 2^32: the signer's twiddles and key polynomials): x + m q is divisible
// by 2^32 with m = -x q^-1 mod 2^32, and (x + m q) / 2^32 < 2q.
constexpr uint32_t MONT_QINV_NEG = 4236238847u;  // -q^-1 mod 2^32
constexpr int32_t MONT_R = 4193792;              // 2^32 mod q
constexpr int32_t MONT_F = 16382;                // 256^-1 2^32 mod q = 2^24 mod q
__device__ __forceinline__ int32_t montq(int32_t a, int32_t b) {
  const uint64_t x = (uint64_t)(uint32_t)a * (uint32_t)b;
  const uint32_t m = (uint32_t)x * MONT_QINV_NEG;
  const uint32_t t = (uint32_t)((x + (uint64_t)m * (uint32_t)Q) >> 32);
  return (int32_t)min(t, t - (uint32_t)Q);
}
__device__ __forceinline__ int32_t addq(int32_t a, int32_t b) {
  int32_t s = a + b;
  return s >= Q ? s - Q : s;
}
__device__ __forceinline__ int32_t subq(int32_t a, int32_t b) {
  int32_t s = a - b;
  return s < 0 ? s + Q : s;
}
__device__ __forceinline__ int32_t modq(int32_t a) {  // any int32 -> [0, q)
  int32_t r = a % Q;
  return r < 0 ? r + Q : r;
}
__device__ __forceinline__ int32_t centered(int32_t a) {  // [0, q) -> a mod+- q
  return a > (Q - 1) / 2 ? a - Q : a;
}

// zetas[m] = 1753^brv8(m) mod q (FIPS 204 Alg. 41), computed once per CTA.
static __device__ void fill_zetas(int32_t* z) {
  for (int m = threadIdx.x; m < 256; m += blockDim.x) {
    int br = __brev((unsigned)m) >> 24;
    int64_t r = 1, b = 1753;
    for (int e = br; e; e >>= 1) {
      if (e & 1) r = r * b % Q;
      b = b * b % Q;
    }
    z[m] = (int32_t)r;
  }
}

// NTT (Alg. 41) of n polynomials p[i * 256 ..] in shared memory, CTA-wide.
static __device__ void ntt(int32_t* p, int n, const int32_t* zetas) {
  for (int len = 128, lg = 7; len >= 1; len >>= 1, --lg) {
    for (int t = threadIdx.x; t < n * 128; t += blockDim.x) {
      const int poly = t >> 7, b = t & 127;
      const int grp = b >> lg, j = (grp << (lg + 1)) + (b & (len - 1));
      const int32_t z = zetas[(256 / (2 * len)) + grp];  // m = 2^(7-lg) + grp
      int32_t* w = p + poly * 256;
      const int32_t tt = mulq(z, w[j + len]);
      const int32_t a = w[j];
      w[j + len] = subq(a, tt);
      w[j] = addq(a, tt);
    }
    __syncthreads();
  }
}

// NTT^-1 (Alg. 42), then multiplication by 256^-1.
static __device__ void ntt_inv(int32_t* p, int n, const int32_t* zetas) {
  for (int len = 1, lg = 0; len < 256; len <<= 1, ++lg) {
    for (int t = threadIdx.x; t < n * 128; t += blockDim.x) {
      const int poly = t >> 7, b = t & 127;
      const int grp = b >> lg, j = (grp << (lg + 1)) + (b & (len - 1));
      // m runs 255 .. down: the group index within this layer counts from the top
      const int32_t z = Q - zetas[(256 / len) - 1 - grp];
      int32_t* w = p + poly * 256;
      const int32_t a = w[j], c = w[j + len];
      w[j] = addq(a, c);
      w[j + len] = mulq(z, subq(a, c));
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < n * 256; t += blockDim.x) p[t] = mulq(8347681, p[t]);
  __syncthreads();
}

// Decompose (Alg. 36) of r in [0, q): r1 in [0, 43], r0 centred.
__device__ __forceinline__ void decompose(int32_t r, int32_t& r1, int32_t& r0) {
  int32_t a0 = r % (2 * GAMMA2);
  if (a0 > GAMMA2) a0 -= 2 * GAMMA2;
  if (r - a0 == Q - 1) {
    r1 = 0;
    r0 = a0 - 1;
  } else {
    r1 = (r - a0) / (2 * GAMMA2);
    r0 = a0;
  }
}

// ------------------------------------------------------------------ key generation
// KeyGen_internal (Alg. 6) for seed xi into *key (one CTA of THREADS threads).
static __global__ void __launch_bounds__(THREADS) mldsa_keygen_kernel(const uint8_t* __restrict__ xi,
                                                               MldsaKey* __restrict__ key) {
  __shared__ int32_t zetas[256];
  __shared__ uint8_t seed[128];  // rho || rho' || K
  __shared__ int32_t s1[L][256], s2[K][256], t[K][256];
  __shared__ uint8_t pk[PK_BYTES];
  fill_zetas(zetas);
  if (threadIdx.x == 0) {
    Shake h;
    h.init(136);
    h.absorb(xi, 32);
    h.absorb_byte(K);
    h.absorb_byte(L);
    h.finalize();
    h.squeeze(seed, 128);
  }
  __syncthreads();
  const uint8_t* rho = seed;
  const uint8_t* rhop = seed + 32;
  const int tid = threadIdx.x;
  if (tid < K * L) {  // ExpandA (Alg. 32): A[r][s] = RejNTTPoly(rho || s || r)
    const int r = tid / L, s = tid % L;
    Shake g;
    g.init(168);
    g.absorb(rho, 32);
    g.absorb_byte((uint8_t)s);
    g.absorb_byte((uint8_t)r);
    g.finalize();
    for (int j = 0; j < 256;) {
      const uint32_t b0 = g.squeeze_byte(), b1 = g.squeeze_byte(), b2 = g.squeeze_byte();
      const int32_t z = (int32_t)(((b2 & 127u) << 16) | (b1 << 8) | b0);
      if (z < Q) key->A[r][s][j++] = z;
    }
  } else if (tid >= 32 && tid < 32 + K + L) {  // ExpandS (Alg. 33, RejBoundedPoly eta = 2)
    const int r = tid - 32;
    int32_t* out = r < L ? s1[r] : s2[r - L];
    Shake h;
    h.init(136);
    h.absorb(rhop, 64);
    h.absorb_byte((uint8_t)r);
    h.absorb_byte(0);
    h.finalize();
    for (int j = 0; j < 256;) {
      const uint32_t z = h.squeeze_byte();
      const uint32_t z0 = z & 15u, z1 = z >> 4;
      if (z0 < 15) out[j++] = modq(2 - (int32_t)(z0 % 5));
      if (z1 < 15 && j < 256) out[j++] = modq(2 - (int32_t)(z1 % 5));
    }
  }
  __syncthreads();
  ntt(&s1[0][0], L, zetas);
  // A-hat o s1-hat, then NTT^-1, + s2
  for (int c = tid; c < 256; c += blockDim.x)
    for (int i = 0; i < K; ++i) {
      int32_t acc = 0;
      for (int j = 0; j < L; ++j) acc = addq(acc, mulq(key->A[i][j][c], s1[j][c]));
      t[i][c] = acc;
    }
  __syncthreads();
  ntt_inv(&t[0][0], K, zetas);
  for (int e = tid; e < K * 256; e += blockDim.x) {
    const int i = e >> 8, c = e & 255;
    const int32_t tv = addq(t[i][c], s2[i][c]);
    int32_t r0 = tv & ((1 << D_) - 1);  // Power2Round (Alg. 35)
    if (r0 > (1 << (D_ - 1))) r0 -= (1 << D_);
    t[i][c] = (tv - r0) >> D_;          // t1
    key->t0[i][c] = modq(r0);           // t0 (NTT below)
  }
  __syncthreads();
  // pkEncode (Alg. 22): rho || SimpleBitPack(t1, 10 bits)
  for (int i = tid; i < 32; i += blockDim.x) pk[i] = rho[i];
  for (int e = tid; e < K * 64; e += blockDim.x) {  // 4 coefficients -> 5 bytes
    const int i = e >> 6, q4 = e & 63;
    uint64_t v = 0;
    for (int k = 0; k < 4; ++k) v |= (uint64_t)t[i][4 * q4 + k] << (10 * k);
    for (int b = 0; b < 5; ++b) pk[32 + i * 320 + q4 * 5 + b] = (uint8_t)(v >> (8 * b));
  }
  __syncthreads();
  for (int i = tid; i < PK_BYTES; i += blockDim.x) key->pk[i] = pk[i];
  if (tid == 0) {
    Shake h;  // tr = H(pk, 64)
    h.init(136);
    h.absorb(pk, PK_BYTES);
    h.finalize();
    h.squeeze(key->tr, 64);
    for (int i = 0; i < 32; ++i) key->Kseed[i] = seed[96 + i];
  }
  // NTT(s1) already in s1; NTT(s2), NTT(t0)
  __syncthreads();
  for (int e = tid; e < K * 256; e += blockDim.x) t[e >> 8][e & 255] = key->t0[e >> 8][e & 255];
  __syncthreads();
  ntt(&s2[0][0], K, zetas);
  ntt(&t[0][0], K, zetas);
  for (int e = tid; e < L * 256; e += blockDim.x) key->s1[e >> 8][e & 255] = s1[e >> 8][e & 255];
  for (int e = tid; e < K * 256; e += blockDim.x) {
    key->s2[e >> 8][e & 255] = s2[e >> 8][e & 255];
    key->t0[e >> 8][e & 255] = t[e >> 8][e & 255];
  }
  __syncthreads();
  // Montgomery form for the signer: every product it takes has one key operand
  for (int e = tid; e < K * L * 256; e += blockDim.x) (&key->A[0][0][0])[e] = mulq((&key->A[0][0][0])[e], MONT_R);
  for (int e = tid; e < L * 256; e += blockDim.x) (&key->s1[0][0])[e] = mulq((&key->s1[0][0])[e], MONT_R);
  for (int e = tid; e < K * 256; e += blockDim.x) {
    (&key->s2[0][0])[e] = mulq((&key->s2[0][0])[e], MONT_R);
    (&key->t0[0][0])[e] = mulq((&key->t0[0][0])[e], MONT_R);
  }
}

// ------------------------------------------------------------------ signing
struct SignArgs {
  const MldsaKey* key;
  uint64_t theta0, n;
  uint64_t seed_psd;   // the puzzles' nonce key (DESIGN R21)
  uint32_t kappa, n_l;
  uint8_t* out;        // n rows of REC_STAGE bytes; signature at SIG_OFF
  uint32_t* ticket;    // zeroed before the launch: the warps' record counter
};

// nonce block blk (16 bytes) of pi_theta: Philox(key = seed_psd, ctr = (theta_lo,
// theta_hi, blk, 0x48)) -- the same words as the puzzle generator (DESIGN R21)
__device__ __forceinline__ uint4 philox_nonce_block(uint64_t seed, uint64_t theta, uint32_t blk) {
  return philox4x32_10(make_uint4((uint32_t)theta, (uint32_t)(theta >> 32), blk, 0x48u),
                       make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}

// One signature per warp (WPB warps per CTA): the single sponges (mu, rho'', c~,
// SampleInBall) run warp-cooperatively on 25 lanes, the four ExpandMask streams in
// column layout on 20 lanes, the polynomial work across the 32 lanes, __syncwarp
// between steps -- many signatures in flight per SM hide the serial Keccak
// latency (one signature per 256-thread CTA ran at 319 k/s on C2).
struct SignSmem {                   // per warp (y / z live in registers: 32 per lane)
  union alignas(8) {
    int32_t tmp[K][256];            // NTT(y), then c.s1 / c.s2 / c.t0 products
    uint8_t w1enc[K * 192];         // w1Encode(w1), hashed before tmp is reused
  };
  union alignas(8) {
    int32_t w[K][256];              // w, then w - c s2, then the hint bits
    uint8_t ymask[L * 576];         // ExpandMask bytes, unpacked before w is computed
  };
  int32_t c[256];
  alignas(8) uint8_t scratch[1][136];  // sponge block staging
  alignas(8) uint8_t mu[64];
  alignas(8) uint8_t rhopp[64];
  alignas(8) uint8_t ctilde[32];
  uint8_t msg[40], zeros[32];
  int count[K];
};
constexpr int WPB = 4;  // ~10 KB of shared memory per warp: 5 CTAs x 4 warps per SM

// Warp NTT / NTT^-1 of N polynomials in shared memory, two layers per pass
// (radix 4: each lane loads 4 coefficients, applies both butterfly layers,
// stores them back -- half the shared-memory traffic of one layer per pass).
// Same butterflies, zeta indices and order of operations per coefficient as
// Alg. 41 / 42; the twiddles are in Montgomery form (x 2^32 mod q).
template <int N>
static __device__ __noinline__ void ntt_w(int32_t* p, const int32_t* zetas, int lane) {
#pragma unroll 1
  for (int lg = 7; lg >= 1; lg -= 2) {  // layers (len, len / 2), len = 2^lg
    const int len = 1 << lg, h = len >> 1;
#pragma unroll 1
    for (int k = 0; k < 2 * N; ++k) {
      const int u = lane + 32 * k, uu = u & 63;
      const int grp = uu >> (lg - 1);                       // block of the len layer
      int32_t* w = p + (u >> 6) * 256 + (grp << (lg + 1)) + (uu & (h - 1));
      const int32_t z1 = zetas[(128 >> lg) + grp];          // m = 256 / (2 len) + grp
      const int32_t z2 = zetas[(256 >> lg) + 2 * grp];      // the two len / 2 blocks
      const int32_t z3 = zetas[(256 >> lg) + 2 * grp + 1];
      int32_t a0 = w[0], a1 = w[h], a2 = w[len], a3 = w[len + h];
      int32_t t = montq(z1, a2);
      a2 = subq(a0, t);
      a0 = addq(a0, t);
      t = montq(z1, a3);
      a3 = subq(a1, t);
      a1 = addq(a1, t);
      t = montq(z2, a1);
      a1 = subq(a0, t);
      a0 = addq(a0, t);
      t = montq(z3, a3);
      a3 = subq(a2, t);
      a2 = addq(a2, t);
      w[0] = a0;
      w[h] = a1;
      w[len] = a2;
      w[len + h] = a3;
    }
    __syncwarp();
  }
}

// NTT^-1 (Alg. 42), the multiplication by 256^-1 fused into the last pass.
template <int N>
static __device__ __noinline__ void ntt_inv_w(int32_t* p, const int32_t* zetas, int lane) {
#pragma unroll 1
  for (int lg = 0; lg <= 6; lg += 2) {  // layers (len, 2 len), len = 2^lg
    const int len = 1 << lg;
#pragma unroll 1
    for (int k = 0; k < 2 * N; ++k) {
      const int u = lane + 32 * k, uu = u & 63;
      const int g = uu >> lg;                               // block of the 2 len layer
      int32_t* w = p + (u >> 6) * 256 + (g << (lg + 2)) + (uu & (len - 1));
      const int32_t za = Q - zetas[(256 >> lg) - 1 - 2 * g];  // len blocks 2g, 2g + 1
      const int32_t zb = Q - zetas[(256 >> lg) - 2 - 2 * g];
      const int32_t zc = Q - zetas[(128 >> lg) - 1 - g];      // 2 len block g
      int32_t a0 = w[0], a1 = w[len], a2 = w[2 * len], a3 = w[3 * len];
      int32_t t = a0;
      a0 = addq(t, a1);
      a1 = montq(za, subq(t, a1));
      t = a2;
      a2 = addq(t, a3);
      a3 = montq(zb, subq(t, a3));
      t = a0;
      a0 = addq(t, a2);
      a2 = montq(zc, subq(t, a2));
      t = a1;
      a1 = addq(t, a3);
      a3 = montq(zc, subq(t, a3));
      if (lg == 6) {
        a0 = montq(MONT_F, a0);
        a1 = montq(MONT_F, a1);
        a2 = montq(MONT_F, a2);
        a3 = montq(MONT_F, a3);
      }
      w[0] = a0;
      w[len] = a1;
      w[2 * len] = a2;
      w[3 * len] = a3;
    }
    __syncwarp();
  }
}

// Sign_internal (Alg. 7) of M' = 0 || 0 || pi_theta, rnd = {0}^32, for record
// i_rec; the whole warp calls it.
static __device__ __forceinline__ void sign_one(const SignArgs& a, SignSmem& S, const int32_t* zetas,
                                                uint64_t i_rec, int lane) {
  const uint64_t theta = a.theta0 + i_rec;
  const MldsaKey* key = a.key;
  S.zeros[lane] = 0;
  if (lane < 2) {  // the message pi_theta: n_s (Philox, R21) || kappa || n_l
    const uint4 r = philox_nonce_block(a.seed_psd, theta, lane);
    const uint32_t wds[4] = {r.x, r.y, r.z, r.w};
    for (int k = 0; k < 16; ++k) S.msg[2 + 16 * lane + k] = (uint8_t)(wds[k >> 2] >> (8 * (k & 3)));
  } else if (lane == 2) {
    S.msg[0] = 0;  // M' = IntegerToBytes(0, 1) || IntegerToBytes(|ctx| = 0, 1) || M
    S.msg[1] = 0;
    for (int k = 0; k < 4; ++k) S.msg[34 + k] = (uint8_t)(a.kappa >> (8 * k));
    S.msg[38] = (uint8_t)a.n_l;
  }
  __syncwarp();
  {
    uint64_t h = 0;  // mu = H(tr || M', 64)
    wsp_absorb<136>(h, key->tr, 64, S.msg, 39, nullptr, 0, S.scratch[0], lane);
    wsp_out<136>(h, S.scratch[0], lane);
    for (int k = lane; k < 64; k += 32) S.mu[k] = S.scratch[0][k];
    __syncwarp();
    uint64_t h2 = 0;  // rho'' = H(K || rnd || mu, 64), rnd = {0}^32
    wsp_absorb<136>(h2, key->Kseed, 32, S.zeros, 32, S.mu, 64, S.scratch[0], lane);
    wsp_out<136>(h2, S.scratch[0], lane);
    for (int k = lane; k < 64; k += 32) S.rhopp[k] = S.scratch[0][k];
    __syncwarp();
  }
  int32_t yr[32];  // y, then z: coefficient lane + 32 j of the four polynomials
  for (uint32_t kappa_ctr = 0;; kappa_ctr += L) {
    // ExpandMask (Alg. 34): y[r] = BitUnpack(H(rho'' || (kappa + r), 576), gamma1 - 1, gamma1)
    {
      // the four streams H(rho'' || IntegerToBytes(kappa + r, 2)), one per lane
      // group (column layout): one padded block each (66 message bytes < 136),
      // then 5 output blocks; tmp (free until y is unpacked) holds the pi buffer
      const int sg = lane / 5, x = lane % 5;
      const uint32_t idx = kappa_ctr + (uint32_t)min(sg, L - 1);
      uint64_t st[5];
#pragma unroll
      for (int y = 0; y < 5; ++y) {
        const int i = x + 5 * y;
        uint64_t v = 0;
        if (i < 8) v = reinterpret_cast<const uint64_t*>(S.rhopp)[i];
        if (i == 8) v = (uint64_t)(idx & 0xFFFFu) | (0x1Full << 16);
        if (i == 16) v = 0x80ull << 56;
        st[y] = v;
      }
      uint64_t* pis = reinterpret_cast<uint64_t*>(&S.tmp[0][0]);
      for (int o = 0; o < 576; o += 136) {  // 5 blocks (680 >= 576 bytes)
        keccak_col4(st, pis, lane);
        const int nw = min(17, (576 - o) / 8);
        if (lane < 5 * L) {
#pragma unroll
          for (int y = 0; y < 4; ++y)
            if (x + 5 * y < nw) reinterpret_cast<uint64_t*>(S.ymask + sg * 576 + o)[x + 5 * y] = st[y];
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) {  // coefficient lane + 32 j of the flattened y
      const int r = j >> 3, cidx = lane + 32 * (j & 7);
      const int bit = 18 * cidx, b = bit >> 3;
      const uint8_t* v = S.ymask + r * 576 + b;
      uint32_t word = v[0] | ((uint32_t)v[1] << 8) | ((uint32_t)v[2] << 16);
      if (b + 3 < 576) word |= (uint32_t)v[3] << 24;
      const uint32_t f = (word >> (bit & 7)) & 0x3FFFFu;
      yr[j] = modq(GAMMA1 - (int32_t)f);
      S.tmp[r][cidx] = yr[j];
    }
    __syncwarp();
    ntt_w<L>(&S.tmp[0][0], zetas, lane);
    for (int cc = lane; cc < 256; cc += 32)
      for (int i = 0; i < K; ++i) {
        int32_t acc = 0;
        for (int j = 0; j < L; ++j) acc = addq(acc, montq(key->A[i][j][cc], S.tmp[j][cc]));
        S.w[i][cc] = acc;
      }
    __syncwarp();
    ntt_inv_w<K>(&S.w[0][0], zetas, lane);
    // w1Encode (Alg. 28): HighBits, 6 bits per coefficient, 4 coefficients -> 3 bytes
    for (int e = lane; e < K * 64; e += 32) {
      const int i = e >> 6, g4 = e & 63;
      uint32_t v = 0;
      for (int k = 0; k < 4; ++k) {
        int32_t r1, r0;
        decompose(S.w[i][4 * g4 + k], r1, r0);
        v |= (uint32_t)r1 << (6 * k);
      }
      S.w1enc[i * 192 + g4 * 3 + 0] = (uint8_t)v;
      S.w1enc[i * 192 + g4 * 3 + 1] = (uint8_t)(v >> 8);
      S.w1enc[i * 192 + g4 * 3 + 2] = (uint8_t)(v >> 16);
    }
    for (int k = lane; k < 256; k += 32) S.c[k] = 0;
    __syncwarp();
    {
      uint64_t h = 0;  // c~ = H(mu || w1Encode(w1), 32)
      uint8_t* sc = S.scratch[0];
      {
        // mu (8 words) || w1Encode (96 words) is word-aligned: each of the 7
        // rate blocks is absorbed as 17 u64 loads, SHAKE padding on the words
        constexpr int NW = (64 + K * 192) / 8, NB = NW / 17 + 1;
        static_assert(NW % 17 != 0 && NB == 7, "mu || w1Encode: 6 full blocks + 2 words");
        const uint64_t* mu64 = reinterpret_cast<const uint64_t*>(S.mu);
        const uint64_t* w64 = reinterpret_cast<const uint64_t*>(S.w1enc);
        for (int blk = 0; blk < NB; ++blk) {
          if (lane < 17) {
            const int m = 17 * blk + lane;
            uint64_t v = m < 8 ? mu64[m] : m < NW ? w64[m - 8] : 0ull;
            if (m == NW) v ^= 0x1Full;
            if (blk == NB - 1 && lane == 16) v ^= 0x80ull << 56;
            h ^= v;
          }
          h = keccak_warp(h, lane);
        }
      }
      wsp_out<136>(h, sc, lane);
      if (lane < 32) S.ctilde[lane] = sc[lane];
      __syncwarp();
      // SampleInBall (Alg. 29): lane 0 samples, the warp squeezes further blocks
      uint64_t sb = 0;  // H(c~): one block, c~ as 4 words, then the SHAKE padding
      if (lane < 4) sb = reinterpret_cast<const uint64_t*>(S.ctilde)[lane];
      if (lane == 4) sb = 0x1Full;
      if (lane == 16) sb = 0x80ull << 56;
      sb = keccak_warp(sb, lane);
      wsp_out<136>(sb, sc, lane);
      uint64_t hb = 0;
      for (int k = 0; k < 8; ++k) hb |= (uint64_t)sc[k] << (8 * k);
      int i = 256 - TAU, pos = 8;
      while (true) {
        if (lane == 0) {
          while (i < 256 && pos < 136) {
            const int j = sc[pos++];
            if (j > i) continue;
            S.c[i] = S.c[j];
            S.c[j] = ((hb >> (i + TAU - 256)) & 1) ? Q - 1 : 1;
            ++i;
          }
        }
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i == 256) break;
        sb = keccak_warp(sb, lane);
        __syncwarp();
        wsp_out<136>(sb, sc, lane);
        pos = 0;
      }
      __syncwarp();
    }
    ntt_w<1>(S.c, zetas, lane);
    // z = y + NTT^-1(c o s1); checked against gamma1 - beta
    for (int e = lane; e < L * 256; e += 32) S.tmp[e >> 8][e & 255] = montq(S.c[e & 255], key->s1[e >> 8][e & 255]);
    __syncwarp();
    ntt_inv_w<L>(&S.tmp[0][0], zetas, lane);
    int bad = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int e = lane + 32 * j;
      const int32_t z = addq(yr[j], S.tmp[e >> 8][e & 255]);
      yr[j] = z;  // y now holds z
      const int32_t zc = centered(z);
      if (zc >= GAMMA1 - BETA || zc <= -(GAMMA1 - BETA)) bad = 1;
    }
    // r0 = LowBits(w - c s2), checked against gamma2 - beta; w <- w - c s2
    for (int e = lane; e < K * 256; e += 32) S.tmp[e >> 8][e & 255] = montq(S.c[e & 255], key->s2[e >> 8][e & 255]);
    __syncwarp();
    ntt_inv_w<K>(&S.tmp[0][0], zetas, lane);
    for (int e = lane; e < K * 256; e += 32) {
      const int32_t v = subq(S.w[e >> 8][e & 255], S.tmp[e >> 8][e & 255]);
      S.w[e >> 8][e & 255] = v;
      int32_t r1, r0;
      decompose(v, r1, r0);
      if (r0 >= GAMMA2 - BETA || r0 <= -(GAMMA2 - BETA)) bad = 1;
    }
    if (__any_sync(0xffffffffu, bad)) continue;
    // c t0; h = MakeHint(-ct0, w - cs2 + ct0); ||ct0|| < gamma2, #h <= omega
    for (int e = lane; e < K * 256; e += 32) S.tmp[e >> 8][e & 255] = montq(S.c[e & 255], key->t0[e >> 8][e & 255]);
    __syncwarp();
    ntt_inv_w<K>(&S.tmp[0][0], zetas, lane);
    int cnt[K] = {0, 0, 0, 0};
    for (int e = lane; e < K * 256; e += 32) {
      const int32_t ct0 = S.tmp[e >> 8][e & 255];
      const int32_t cc = centered(ct0);
      if (cc >= GAMMA2 || cc <= -GAMMA2) bad = 1;
      const int32_t r = addq(S.w[e >> 8][e & 255], ct0);  // w - cs2 + ct0
      int32_t h1, h0, v1, v0;
      decompose(r, h1, h0);
      decompose(subq(r, ct0), v1, v0);                     // r + (-ct0)
      const int hint = h1 != v1;
      S.w[e >> 8][e & 255] = hint;  // w now holds the hint bits
      cnt[e >> 8] += hint;
    }
    if (__any_sync(0xffffffffu, bad)) continue;
    int total = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int ci = __reduce_add_sync(0xffffffffu, cnt[i]);
      if (lane == 0) S.count[i] = ci;
      total += ci;
    }
    if (total > OMEGA) continue;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) {  // z (centred) into tmp for the packing
      const int e = lane + 32 * j;
      S.tmp[e >> 8][e & 255] = centered(yr[j]);
    }
    __syncwarp();
    // sigEncode (Alg. 26): c~ || BitPack(z, gamma1 - 1, gamma1) || HintBitPack(h)
    uint8_t* sig = a.out + i_rec * REC_STAGE + SIG_OFF;
    if (lane < 8)
      for (int k = 0; k < 4; ++k) sig[4 * lane + k] = S.ctilde[4 * lane + k];
    for (int e = lane; e < L * 64; e += 32) {  // 4 coefficients -> 9 bytes
      const int r = e >> 6, g4 = e & 63;
      uint64_t lo = 0;
      uint32_t hi = 0;
      for (int k = 0; k < 4; ++k) {
        const uint32_t f = (uint32_t)(GAMMA1 - S.tmp[r][4 * g4 + k]);  // 18 bits
        const int bit = 18 * k;
        lo |= (uint64_t)f << bit;
        if (bit + 18 > 64) hi |= f >> (64 - bit);
      }
      uint8_t* o = sig + 32 + r * 576 + g4 * 9;
      for (int b = 0; b < 8; ++b) o[b] = (uint8_t)(lo >> (8 * b));
      o[8] = (uint8_t)hi;
    }
    {  // HintBitPack (Alg. 20): the indices of each poly's hints in increasing order,
       // 32 coefficients per ballot, each hint's slot from the popcount below it
      uint8_t* hp = sig + 32 + L * 576;
      int index = 0;
      for (int i = 0; i < K; ++i) {
        for (int c = 0; c < 8; ++c) {
          const bool hbit = S.w[i][32 * c + lane] != 0;
          const uint32_t mk = __ballot_sync(0xffffffffu, hbit);
          if (hbit) hp[index + __popc(mk & ((1u << lane) - 1u))] = (uint8_t)(32 * c + lane);
          index += __popc(mk);
        }
        if (lane == 0) hp[OMEGA + i] = (uint8_t)index;
      }
      for (int k = index + lane; k < OMEGA; k += 32) hp[k] = 0;
    }
    return;
  }
}

// Persistent warps: each warp takes the next record from a.ticket until all n
// are signed. The rejection loop's iteration count is geometric (FIPS 204: ~4.25
// expected for ML-DSA-44), so warps finish at different times; one record per
// warp with CTAs of WPB warps kept each CTA resident until its slowest
// signature was done (ncu: 15 % warps active of a 31 % occupancy limit).
static __global__ void __launch_bounds__(32 * WPB, 5) mldsa_sign_kernel(SignArgs a) {
  __shared__ int32_t zetas[256];
  extern __shared__ __align__(16) uint8_t dsm[];
  fill_zetas(zetas);
  if (threadIdx.x < 32) {
    k_lane_tab[threadIdx.x].init(threadIdx.x);
    k_col_tab[threadIdx.x].init(threadIdx.x);
  }
  __syncthreads();
  for (int m = threadIdx.x; m < 256; m += blockDim.x) zetas[m] = mulq(zetas[m], MONT_R);  // Montgomery form
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  SignSmem& S = reinterpret_cast<SignSmem*>(dsm)[wid];
  for (;;) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1u);
    const uint64_t i_rec = __shfl_sync(0xffffffffu, t, 0);
    if (i_rec >= a.n) return;
    sign_one(a, S, zetas, i_rec, lane);
    __syncwarp();
  }
}

// host launchers (the caller owns `key`, `xi_dev` (32 bytes) and `stage`)
static inline cudaError_t keygen(const uint8_t* xi_dev, MldsaKey* key, cudaStream_t st) {
  mldsa_keygen_kernel<<<1, THREADS, 0, st>>>(xi_dev, key);
  return cudaGetLastError();
}
// `ticket`: one device u32 the launcher zeroes on `st` (n < 2^32 per launch).
static inline cudaError_t sign_records(const MldsaKey* key, uint64_t theta0, uint64_t n, uint64_t seed_psd,
                                       uint32_t kappa, uint32_t n_l, uint8_t* stage, uint32_t* ticket,
                                       cudaStream_t st) {
  SignArgs a;
  a.key = key;
  a.theta0 = theta0;
  a.n = n;
  a.seed_psd = seed_psd;
  a.kappa = kappa;
  a.n_l = n_l;
  a.out = stage;
  a.ticket = ticket;
  const size_t sm = WPB * sizeof(SignSmem);
  cudaError_t e = cudaFuncSetAttribute(mldsa_sign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int dev = 0, n_sm = 0, per_sm = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mldsa_sign_kernel, 32 * WPB, sm)) != cudaSuccess)
    return e;
  const uint64_t blocks = std::min<uint64_t>((n + WPB - 1) / WPB, (uint64_t)n_sm * std::max(per_sm, 1));
  if ((e = cudaMemsetAsync(ticket, 0, sizeof(uint32_t), st)) != cudaSuccess) return e;
  mldsa_sign_kernel<<<(uint32_t)blocks, 32 * WPB, sm, st>>>(a);
  return cudaGetLastError();
}

}  // namespace mldsa
}  // namespace qpir
