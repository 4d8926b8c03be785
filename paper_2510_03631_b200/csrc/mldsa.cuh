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
//   mldsa_sign_kernel    (1 CTA per record) -- Sign_internal of pi_theta; the
//                                      2420 signature bytes go to byte 597 of the
//                                      record's 3024-byte staging row (16-byte
//                                      aligned for the packing kernel).
// The sponges run one per thread (byte-serial absorb / squeeze); polynomial
// arithmetic runs across the CTA (256 threads: one coefficient or one NTT
// butterfly per thread per step).
#pragma once
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

struct MldsaKey {                 // expanded signing key (global memory)
  int32_t A[K][L][256];           // A-hat (NTT domain)
  int32_t s1[L][256];             // NTT(s1)
  int32_t s2[K][256];             // NTT(s2)
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

// ------------------------------------------------------------------ arithmetic
__device__ __forceinline__ int32_t mulq(int32_t a, int32_t b) {
  return (int32_t)(((int64_t)a * b) % Q);  // a, b in [0, q)
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
}

// ------------------------------------------------------------------ signing
struct SignArgs {
  const MldsaKey* key;
  uint64_t theta0, n;
  uint64_t seed_psd;   // the puzzles' nonce key (DESIGN R21)
  uint32_t kappa, n_l;
  uint8_t* out;        // n rows of REC_STAGE bytes; signature at SIG_OFF
};

// nonce block blk (16 bytes) of pi_theta: Philox(key = seed_psd, ctr = (theta_lo,
// theta_hi, blk, 0x48)) -- the same words as the puzzle generator (DESIGN R21)
__device__ __forceinline__ uint4 philox_nonce_block(uint64_t seed, uint64_t theta, uint32_t blk) {
  return philox4x32_10(make_uint4((uint32_t)theta, (uint32_t)(theta >> 32), blk, 0x48u),
                       make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}

// Sign_internal (Alg. 7) of M' = 0 || 0 || pi_theta, rnd = {0}^32.
static __global__ void __launch_bounds__(THREADS) mldsa_sign_kernel(SignArgs a) {
  __shared__ int32_t zetas[256];
  __shared__ int32_t y[L][256];     // y (normal domain)
  __shared__ int32_t tmp[K][256];   // NTT(y), then c.s1 / c.s2 / c.t0 products
  __shared__ int32_t w[K][256];     // w = NTT^-1(A-hat o NTT(y))
  __shared__ int32_t c[256];
  __shared__ uint8_t buf[K * 192];  // ExpandMask bytes (4 x 576 > 768) / w1Encode (768)
  __shared__ uint8_t ymask[L * 576];
  __shared__ uint8_t mu[64], rhopp[64], ctilde[32], msg[39];
  __shared__ int s_count[K];
  const int tid = threadIdx.x;
  const uint64_t i_rec = blockIdx.x;
  if (i_rec >= a.n) return;
  const uint64_t theta = a.theta0 + i_rec;
  const MldsaKey* key = a.key;
  fill_zetas(zetas);
  if (tid < 2) {  // the message pi_theta: n_s (Philox, R21) || kappa || n_l
    const uint4 r = philox_nonce_block(a.seed_psd, theta, tid);
    const uint32_t wds[4] = {r.x, r.y, r.z, r.w};
    for (int k = 0; k < 16; ++k) msg[2 + 16 * tid + k] = (uint8_t)(wds[k >> 2] >> (8 * (k & 3)));
  } else if (tid == 2) {
    msg[0] = 0;  // M' = IntegerToBytes(0, 1) || IntegerToBytes(|ctx| = 0, 1) || M
    msg[1] = 0;
    for (int k = 0; k < 4; ++k) msg[34 + k] = (uint8_t)(a.kappa >> (8 * k));
    msg[38] = (uint8_t)a.n_l;
  }
  __syncthreads();
  if (tid == 0) {
    Shake h;  // mu = H(tr || M', 64)
    h.init(136);
    h.absorb(key->tr, 64);
    h.absorb(msg, 39);
    h.finalize();
    h.squeeze(mu, 64);
    Shake h2;  // rho'' = H(K || rnd || mu, 64)
    h2.init(136);
    h2.absorb(key->Kseed, 32);
    for (int k = 0; k < 32; ++k) h2.absorb_byte(0);
    h2.absorb(mu, 64);
    h2.finalize();
    h2.squeeze(rhopp, 64);
  }
  __syncthreads();
  for (uint32_t kappa_ctr = 0;; kappa_ctr += L) {
    // ExpandMask (Alg. 34): y[r] = BitUnpack(H(rho'' || (kappa + r), 576), gamma1 - 1, gamma1)
    if (tid < L) {
      Shake h;
      h.init(136);
      h.absorb(rhopp, 64);
      const uint32_t idx = kappa_ctr + tid;
      h.absorb_byte((uint8_t)(idx & 255));
      h.absorb_byte((uint8_t)(idx >> 8));
      h.finalize();
      h.squeeze(ymask + tid * 576, 576);
    }
    __syncthreads();
    for (int e = tid; e < L * 64; e += blockDim.x) {  // 4 coefficients per 9 bytes
      const int r = e >> 6, g4 = e & 63;
      const uint8_t* v = ymask + r * 576 + g4 * 9;
      uint64_t lo = 0;
      for (int b = 0; b < 8; ++b) lo |= (uint64_t)v[b] << (8 * b);
      const uint64_t hi = v[8];
      for (int k = 0; k < 4; ++k) {
        const int bit = 18 * k;
        uint32_t f;
        if (bit + 18 <= 64) f = (uint32_t)(lo >> bit) & 0x3FFFFu;
        else f = (uint32_t)((lo >> bit) | (hi << (64 - bit))) & 0x3FFFFu;
        const int32_t yv = GAMMA1 - (int32_t)f;
        y[r][4 * g4 + k] = modq(yv);
        tmp[r][4 * g4 + k] = modq(yv);
      }
    }
    __syncthreads();
    ntt(&tmp[0][0], L, zetas);
    for (int cc = tid; cc < 256; cc += blockDim.x)
      for (int i = 0; i < K; ++i) {
        int32_t acc = 0;
        for (int j = 0; j < L; ++j) acc = addq(acc, mulq(key->A[i][j][cc], tmp[j][cc]));
        w[i][cc] = acc;
      }
    __syncthreads();
    ntt_inv(&w[0][0], K, zetas);
    // w1Encode (Alg. 28): HighBits, 6 bits per coefficient, 4 coefficients -> 3 bytes
    for (int e = tid; e < K * 64; e += blockDim.x) {
      const int i = e >> 6, g4 = e & 63;
      uint32_t v = 0;
      for (int k = 0; k < 4; ++k) {
        int32_t r1, r0;
        decompose(w[i][4 * g4 + k], r1, r0);
        v |= (uint32_t)r1 << (6 * k);
      }
      buf[i * 192 + g4 * 3 + 0] = (uint8_t)v;
      buf[i * 192 + g4 * 3 + 1] = (uint8_t)(v >> 8);
      buf[i * 192 + g4 * 3 + 2] = (uint8_t)(v >> 16);
    }
    __syncthreads();
    if (tid == 0) {
      Shake h;  // c~ = H(mu || w1Encode(w1), 32)
      h.init(136);
      h.absorb(mu, 64);
      h.absorb(buf, K * 192);
      h.finalize();
      h.squeeze(ctilde, 32);
      // SampleInBall (Alg. 29)
      for (int k = 0; k < 256; ++k) c[k] = 0;
      Shake s;
      s.init(136);
      s.absorb(ctilde, 32);
      s.finalize();
      uint64_t hb = 0;
      for (int k = 0; k < 8; ++k) hb |= (uint64_t)s.squeeze_byte() << (8 * k);
      for (int i = 256 - TAU; i < 256; ++i) {
        int j = s.squeeze_byte();
        while (j > i) j = s.squeeze_byte();
        c[i] = c[j];
        c[j] = ((hb >> (i + TAU - 256)) & 1) ? Q - 1 : 1;
      }
    }
    __syncthreads();
    ntt(c, 1, zetas);
    // z = y + NTT^-1(c o s1); checked against gamma1 - beta
    for (int e = tid; e < L * 256; e += blockDim.x) tmp[e >> 8][e & 255] = mulq(c[e & 255], key->s1[e >> 8][e & 255]);
    __syncthreads();
    ntt_inv(&tmp[0][0], L, zetas);
    int bad = 0;
    for (int e = tid; e < L * 256; e += blockDim.x) {
      const int32_t z = addq(y[e >> 8][e & 255], tmp[e >> 8][e & 255]);
      y[e >> 8][e & 255] = z;  // y now holds z
      const int32_t zc = centered(z);
      if (zc >= GAMMA1 - BETA || zc <= -(GAMMA1 - BETA)) bad = 1;
    }
    // r0 = LowBits(w - c s2), checked against gamma2 - beta; w <- w - c s2
    for (int e = tid; e < K * 256; e += blockDim.x) tmp[e >> 8][e & 255] = mulq(c[e & 255], key->s2[e >> 8][e & 255]);
    __syncthreads();
    ntt_inv(&tmp[0][0], K, zetas);
    for (int e = tid; e < K * 256; e += blockDim.x) {
      const int32_t v = subq(w[e >> 8][e & 255], tmp[e >> 8][e & 255]);
      w[e >> 8][e & 255] = v;
      int32_t r1, r0;
      decompose(v, r1, r0);
      if (r0 >= GAMMA2 - BETA || r0 <= -(GAMMA2 - BETA)) bad = 1;
    }
    if (__syncthreads_or(bad)) continue;
    // c t0; h = MakeHint(-ct0, w - cs2 + ct0); ||ct0|| < gamma2, #h <= omega
    for (int e = tid; e < K * 256; e += blockDim.x) tmp[e >> 8][e & 255] = mulq(c[e & 255], key->t0[e >> 8][e & 255]);
    __syncthreads();
    ntt_inv(&tmp[0][0], K, zetas);
    int ones = 0;
    for (int e = tid; e < K * 256; e += blockDim.x) {
      const int32_t ct0 = tmp[e >> 8][e & 255];
      const int32_t cc = centered(ct0);
      if (cc >= GAMMA2 || cc <= -GAMMA2) bad = 1;
      const int32_t r = addq(w[e >> 8][e & 255], ct0);  // w - cs2 + ct0
      const int32_t zz = subq(0, ct0);                    // -ct0
      int32_t h1, h0, v1, v0;
      decompose(r, h1, h0);
      decompose(addq(r, zz), v1, v0);
      const int hint = h1 != v1;
      w[e >> 8][e & 255] = hint;  // w now holds the hint bits
      ones += hint;
    }
    if (__syncthreads_or(bad)) continue;
    // count hint ones per polynomial
    if (tid < K) s_count[tid] = 0;
    __syncthreads();
    if (ones) {
      for (int e = tid; e < K * 256; e += blockDim.x)
        if (w[e >> 8][e & 255]) atomicAdd(&s_count[e >> 8], 1);
    }
    __syncthreads();
    if (s_count[0] + s_count[1] + s_count[2] + s_count[3] > OMEGA) {
      __syncthreads();
      continue;
    }
    // sigEncode (Alg. 26): c~ || BitPack(z, gamma1 - 1, gamma1) || HintBitPack(h)
    uint8_t* sig = a.out + i_rec * REC_STAGE + SIG_OFF;
    for (int k = tid; k < 32; k += blockDim.x) sig[k] = ctilde[k];
    for (int e = tid; e < L * 64; e += blockDim.x) {  // 4 coefficients -> 9 bytes
      const int r = e >> 6, g4 = e & 63;
      uint64_t lo = 0;
      uint32_t hi = 0;
      for (int k = 0; k < 4; ++k) {
        const uint32_t f = (uint32_t)(GAMMA1 - centered(y[r][4 * g4 + k]));  // 18 bits
        const int bit = 18 * k;
        lo |= (uint64_t)f << bit;
        if (bit + 18 > 64) hi |= f >> (64 - bit);
      }
      uint8_t* o = sig + 32 + r * 576 + g4 * 9;
      for (int b = 0; b < 8; ++b) o[b] = (uint8_t)(lo >> (8 * b));
      o[8] = (uint8_t)hi;
    }
    if (tid < K) {  // HintBitPack (Alg. 20): indices of poly tid after the previous polys'
      uint8_t* hp = sig + 32 + L * 576;
      int index = 0;
      for (int i = 0; i < tid; ++i) index += s_count[i];
      for (int j = 0; j < 256; ++j)
        if (w[tid][j]) hp[index++] = (uint8_t)j;
      hp[OMEGA + tid] = (uint8_t)index;
      if (tid == K - 1)
        for (int k = index; k < OMEGA; ++k) hp[k] = 0;
    }
    return;
  }
}

// host launchers (the caller owns `key`, `xi_dev` (32 bytes) and `stage`)
static inline cudaError_t keygen(const uint8_t* xi_dev, MldsaKey* key, cudaStream_t st) {
  mldsa_keygen_kernel<<<1, THREADS, 0, st>>>(xi_dev, key);
  return cudaGetLastError();
}
static inline cudaError_t sign_records(const MldsaKey* key, uint64_t theta0, uint64_t n, uint64_t seed_psd,
                                       uint32_t kappa, uint32_t n_l, uint8_t* stage, cudaStream_t st) {
  SignArgs a;
  a.key = key;
  a.theta0 = theta0;
  a.n = n;
  a.seed_psd = seed_psd;
  a.kappa = kappa;
  a.n_l = n_l;
  a.out = stage;
  mldsa_sign_kernel<<<(uint32_t)n, THREADS, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace mldsa
}  // namespace qpir
