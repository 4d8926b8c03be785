/*
 * qpir_oracle.c -- plain, slow, obviously-correct CPU oracle for the LWE-PIR
 * answer path of QPADL (arXiv 2510.03631).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may link, load or
 * call this file: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs.  It shares no code with
 * paper_2510_03631_b200/ (the CUDA path) and includes none of its headers.
 *
 * Citation keys: P:NNN = PAPER.md line, S:NNN = SPEC.md line, SURVEY = SURVEY.md
 * section, DESIGN = DESIGN.md "Readings" table (R1..R21).
 *
 * What is computed (plain definitions, DESIGN R1..R21 for everything the paper
 * leaves open):
 *   - the PIR response rho <- PIR.Query.Response(q, DB)  (Def. 1, P:241;
 *     Alg. 1 step 18) read as the LWE answer ans = D.qu mod 2^32,
 *     which is the same "q.DB mod q" contraction as Alg. 4 steps 14-15
 *      with the modulus fixed to q = 2^32 (DESIGN R2);
 *   - the multi-request form (Alg. 3/4 "multiple requests"):
 *     ANS[b] = D.Q[b] mod 2^32;
 *   - the offline precomputation (Offline-online mode) read as
 *     the LWE hint H = D.A mod 2^32 (DESIGN R7);
 *   - client side (Def. 1 Client.Query / BlockReconst):
 *     keygen, query, decode of a Regev-LWE PIR (DESIGN R1, R4-R8);
 *   - the NEXT rows: Chor XOR PIR (Alg. 3, R15/R16), Goldberg PIR over F_p
 *     with Lagrange and Berlekamp-Welch reconstruction (Alg. 4, R17/R18),
 *     CIP-PIR offline/online (R19), HCT Puzzle.Gen / Puzzle.Bind (Alg. 1
 *     step 1, R21; the ML-DSA-44 signatures are in oracle/mldsa.py).
 *
 * Every server-side result is the plain modular matrix product in Z_{2^32};
 * the loops below are the textbook triple loops in uint32_t arithmetic
 * (unsigned overflow wraps mod 2^32 by the C standard, C11 6.2.5p9).
 * No blocking, no reordering beyond an OpenMP split over independent rows.
 *
 * Pins (tests/test_oracle_*.py): Philox KATs from Random123; numpy/torch
 * library matmuls; closed forms (unit, all-ones, all-0xFFFFFFFF, constant,
 * top-limb queries); linearity; the exact LWE identity; brute-force decode of
 * every record of the tiny DB; the GF(2) link to Chor PIR (Alg. 3).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11, "Parallel random   */
/* numbers: as easy as 1, 2, 3", Fig. 2 / Random123 philox.h).          */
/* DESIGN R7: the LWE public matrix A and all client randomness are     */
/* drawn from it.                                                       */
/* ------------------------------------------------------------------ */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void qo_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                      uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { /* key schedule: bump before every round but the first */
      k0 += PHILOX_W0;
      k1 += PHILOX_W1;
    }
    uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c0;
    uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Domain tags in ctr[3] (DESIGN R7): 'A' public matrix, 'S' secret, 'E' error. */
#define QO_DOMAIN_A 0x41u
#define QO_DOMAIN_S 0x53u
#define QO_DOMAIN_E 0x45u

static void key_from_seed(uint64_t seed, uint32_t key[2]) {
  key[0] = (uint32_t)(seed & 0xFFFFFFFFu);
  key[1] = (uint32_t)(seed >> 32);
}

/* A[c][j] = Philox(key = seed_A, ctr = (c, j>>2, 0, 'A'))[j & 3]  (DESIGN R7).
 * A is m x n, row-major (cell-major): A[c*n + j]. */
void qo_expand_A(uint64_t seed_A, uint64_t m, uint32_t n, uint32_t *A) {
  uint32_t key[2];
  key_from_seed(seed_A, key);
  for (uint64_t c = 0; c < m; ++c) {
    for (uint32_t j = 0; j < n; ++j) {
      uint32_t ctr[4] = {(uint32_t)c, j >> 2, 0u, QO_DOMAIN_A};
      uint32_t out[4];
      qo_philox4x32_10(ctr, key, out);
      A[c * (uint64_t)n + j] = out[j & 3u];
    }
  }
}

/* ------------------------------------------------------------------ */
/* DB layout (DESIGN R9/R10; "DB is modeled as a matrix", S:51  */
/* row-major DB.Index, P:1107 multiple-block retrieval).              */
/* theta = cell * n_ch + ch ;  record bytes rec_theta[0..d)            */
/* blk = cell / m, col = cell % m, row = (blk * n_ch + ch) * d + b     */
/* ell = ceil(n_cells / m) * n_ch * d.  Unused slots hold 0.           */
/* ------------------------------------------------------------------ */
uint64_t qo_ell(uint64_t n_cells, uint64_t n_ch, uint64_t d, uint64_t m) {
  uint64_t n_blk = (n_cells + m - 1) / m;
  return n_blk * n_ch * d;
}

void qo_position(uint64_t n_ch, uint64_t d, uint64_t m, uint64_t theta,
                 uint64_t b, uint64_t *row, uint64_t *col) {
  uint64_t cell = theta / n_ch;
  uint64_t ch = theta % n_ch;
  uint64_t blk = cell / m;
  *col = cell % m;
  *row = (blk * n_ch + ch) * d + b;
}

/* D is ell x m, row-major, plain (the oracle's own layout). */
void qo_pack(const uint8_t *records, uint64_t n_cells, uint64_t n_ch,
             uint64_t d, uint64_t m, uint8_t *D) {
  uint64_t ell = qo_ell(n_cells, n_ch, d, m);
  memset(D, 0, (size_t)(ell * m));
  uint64_t n_rec = n_cells * n_ch;
  for (uint64_t theta = 0; theta < n_rec; ++theta) {
    for (uint64_t b = 0; b < d; ++b) {
      uint64_t row, col;
      qo_position(n_ch, d, m, theta, b, &row, &col);
      D[row * m + col] = records[theta * d + b];
    }
  }
}

/* ------------------------------------------------------------------ */
/* Server side.                                                        */
/* ------------------------------------------------------------------ */

/* ans[r] = sum_c D[r][c] * qu[c] mod 2^32, r < rows.  (Def. 1 Response,
 * P:241; Alg. 4 steps 14-15, modulus 2^32 per DESIGN R2.)
 * D may be any set of rows (rows x m, row-major). */
void qo_answer(const uint8_t *D, uint64_t rows, uint64_t m, const uint32_t *qu,
               uint32_t *ans) {
  int64_t R = (int64_t)rows;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; ++r) {
    uint32_t acc = 0;
    const uint8_t *Dr = D + (uint64_t)r * m;
    for (uint64_t c = 0; c < m; ++c) acc += (uint32_t)Dr[c] * qu[c];
    ans[r] = acc;
  }
}

/* ANS[b][r] = sum_c D[r][c] * Q[b][c] mod 2^32.  Q is B x m (query-major),
 * ANS is B x rows (query-major).  Multi-request form. */
void qo_answer_batch(const uint8_t *D, uint64_t rows, uint64_t m,
                     const uint32_t *Q, uint64_t B, uint32_t *ANS) {
  int64_t R = (int64_t)rows;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; ++r) {
    const uint8_t *Dr = D + (uint64_t)r * m;
    for (uint64_t b = 0; b < B; ++b) {
      const uint32_t *Qb = Q + b * m;
      uint32_t acc = 0;
      for (uint64_t c = 0; c < m; ++c) acc += (uint32_t)Dr[c] * Qb[c];
      ANS[b * rows + (uint64_t)r] = acc;
    }
  }
}

/* H[r][j] = sum_c D[r][c] * A[c][j] mod 2^32.  A is m x n (cell-major), H is
 * rows x n row-major.  Offline precomputation, DESIGN R7. */
void qo_hint(const uint8_t *D, uint64_t rows, uint64_t m, const uint32_t *A,
             uint32_t n, uint32_t *H) {
  int64_t R = (int64_t)rows;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; ++r) {
    const uint8_t *Dr = D + (uint64_t)r * m;
    uint32_t *Hr = H + (uint64_t)r * n;
    for (uint32_t j = 0; j < n; ++j) Hr[j] = 0;
    /* same sum, c outer so that A is read row by row */
    for (uint64_t c = 0; c < m; ++c) {
      const uint32_t dv = Dr[c];
      const uint32_t *Ac = A + c * (uint64_t)n;
      for (uint32_t j = 0; j < n; ++j) Hr[j] += dv * Ac[j];
    }
  }
}

/* ------------------------------------------------------------------ */
/* Client side (Def. 1 Client.Query / BlockReconst),     */
/* Regev-LWE with q = 2^32, p = 2^8, Delta = 2^24 (DESIGN R2-R8).      */
/* ------------------------------------------------------------------ */

/* s[j] = Philox(key = seed_s, ctr = (j>>2, 0, 0, 'S'))[j & 3]: uniform Z_q^n. */
void qo_keygen(uint64_t seed_s, uint32_t n, uint32_t *s) {
  uint32_t key[2];
  key_from_seed(seed_s, key);
  for (uint32_t j = 0; j < n; ++j) {
    uint32_t ctr[4] = {j >> 2, 0u, 0u, QO_DOMAIN_S};
    uint32_t out[4];
    qo_philox4x32_10(ctr, key, out);
    s[j] = out[j & 3u];
  }
}

/* e_c = round(sigma * z), z = sqrt(-2 ln u1) cos(2 pi u2) (Box-Muller),
 * u1 = (w0 + 1) / 2^32 in (0, 1], u2 = w1 / 2^32,
 * (w0, w1) = Philox(key = seed_e, ctr = (c, qidx, 0, 'E'))[0..1].  DESIGN R5. */
void qo_sample_error(uint64_t seed_e, uint32_t qidx, uint64_t m, double sigma,
                     int32_t *e) {
  uint32_t key[2];
  key_from_seed(seed_e, key);
  const double two32 = 4294967296.0;
  const double two_pi = 6.283185307179586476925286766559;
  for (uint64_t c = 0; c < m; ++c) {
    uint32_t ctr[4] = {(uint32_t)c, qidx, 0u, QO_DOMAIN_E};
    uint32_t out[4];
    qo_philox4x32_10(ctr, key, out);
    double u1 = ((double)out[0] + 1.0) / two32;
    double u2 = (double)out[1] / two32;
    double z = sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
    e[c] = (int32_t)llround(sigma * z);
  }
}

/* qu[c] = (sum_j A[c][j] s[j] + e_c + Delta * [c == col_star]) mod 2^32.
 * Client.Query(theta) (Def. 1; Alg. 1 step 7), DESIGN R1.
 * e is written to e_out (may be NULL) so that tests can check the exact
 * LWE identity.  A: m x n cell-major. */
void qo_query(const uint32_t *A, uint64_t m, uint32_t n, const uint32_t *s,
              uint64_t seed_e, uint32_t qidx, double sigma, uint64_t col_star,
              uint32_t *qu, int32_t *e_out, int32_t *e_scratch) {
  int32_t *e = e_out ? e_out : e_scratch;
  qo_sample_error(seed_e, qidx, m, sigma, e);
  const uint32_t Delta = 1u << 24;
  for (uint64_t c = 0; c < m; ++c) {
    uint32_t acc = 0;
    for (uint32_t j = 0; j < n; ++j) acc += A[c * (uint64_t)n + j] * s[j];
    acc += (uint32_t)e[c];
    if (c == col_star) acc += Delta;
    qu[c] = acc;
  }
}

/* BlockReconst (Def. 1) for a set of rows:
 * x_r = (ans[r] - sum_j H[r][j] s[j]) mod 2^32, out = ((x_r + 2^23) >> 24) & 0xFF.
 * rows[i] indexes both ans and H (H row-major, n wide).  DESIGN R8. */
void qo_decode(const uint32_t *ans, const uint32_t *H, uint32_t n,
               const uint32_t *s, const uint64_t *rows, uint64_t n_rows,
               uint8_t *out) {
  for (uint64_t i = 0; i < n_rows; ++i) {
    uint64_t r = rows[i];
    uint32_t hs = 0;
    for (uint32_t j = 0; j < n; ++j) hs += H[r * n + j] * s[j];
    uint32_t x = ans[r] - hs;
    out[i] = (uint8_t)(((x + (1u << 23)) >> 24) & 0xFFu);
  }
}

/* Threads the OpenMP loops above use (reported as cpu_baseline.cores). */
int qo_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void qo_set_num_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

/* ------------------------------------------------------------------ */
/* NEXT-1: QPADL-ENS = Chor et al. multi-server XOR PIR (P:736;        */
/* Lemma 1 proof; Alg. 3 "Multi-request Parallel Chor-PIR",    */
/* P:972-1000).  DB = r records (rows) of d bytes = b = 8d bits over   */
/* GF(2).  Bit t of an r-bit vector lives at byte t >> 3, bit t & 7.   */
/* ------------------------------------------------------------------ */
#define QO_DOMAIN_C 0x43u

/* Client.Query (Lemma 1 proof): rho_1..rho_{l-1} uniform r-bit strings,
 * rho_l = XOR_{i<l} rho_i XOR e_theta.  Share i's byte w is byte (w & 3) of
 * word 0 of Philox(key = seed, ctr = (w >> 2, i, theta_lo, 'C')) (DESIGN R15);
 * bits at positions >= r are 0.  shares: l x ceil(r/8) bytes. */
void qo_ens_query(uint64_t theta, uint64_t r, uint32_t l, uint64_t seed, uint8_t *shares) {
  uint64_t nb = (r + 7) / 8;
  uint32_t key[2];
  key_from_seed(seed, key);
  uint8_t *last = shares + (uint64_t)(l - 1) * nb;
  memset(last, 0, (size_t)nb);
  for (uint32_t i = 0; i + 1 < l; ++i) {
    uint8_t *sh = shares + (uint64_t)i * nb;
    for (uint64_t w = 0; w < nb; ++w) {
      uint32_t ctr[4] = {(uint32_t)(w >> 2), i, (uint32_t)theta, QO_DOMAIN_C};
      uint32_t out[4];
      qo_philox4x32_10(ctr, key, out);
      sh[w] = (uint8_t)((out[0] >> (8 * (w & 3))) & 0xFFu);
    }
    if (r % 8) sh[nb - 1] &= (uint8_t)((1u << (r % 8)) - 1u);
    for (uint64_t w = 0; w < nb; ++w) last[w] ^= sh[w];
  }
  last[theta >> 3] ^= (uint8_t)(1u << (theta & 7));
}

/* DB.Query.Response (Def. 1; Alg. 3 steps 8-9): out = XOR of the rows
 * theta whose share bit is 1.  records: r x d, row-major. */
void qo_ens_respond(const uint8_t *records, uint64_t r, uint64_t d, const uint8_t *share,
                    uint8_t *out) {
  memset(out, 0, (size_t)d);
  for (uint64_t t = 0; t < r; ++t) {
    if ((share[t >> 3] >> (t & 7)) & 1u) {
      const uint8_t *row = records + t * d;
      for (uint64_t j = 0; j < d; ++j) out[j] ^= row[j];
    }
  }
}

/* Multi-request form (Alg. 3): B shares (B x ceil(r/8)) -> B x d. */
void qo_ens_respond_batch(const uint8_t *records, uint64_t r, uint64_t d, const uint8_t *Q,
                          uint64_t B, uint8_t *out) {
  uint64_t nb = (r + 7) / 8;
  int64_t BB = (int64_t)B;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < BB; ++b)
    qo_ens_respond(records, r, d, Q + (uint64_t)b * nb, out + (uint64_t)b * d);
}

/* BlockReconst (Def. 1; Lemma 1 proof -- read as the XOR of the l
 * responses, DESIGN R16): out = XOR_i resp_i.  resp: l x d. */
void qo_ens_reconstruct(const uint8_t *resp, uint32_t l, uint64_t d, uint8_t *out) {
  memset(out, 0, (size_t)d);
  for (uint32_t i = 0; i < l; ++i)
    for (uint64_t j = 0; j < d; ++j) out[j] ^= resp[(uint64_t)i * d + j];
}

/* ------------------------------------------------------------------ */
/* NEXT-2: QPADL-FTR = Goldberg robust multi-server PIR over a prime    */
/* field F_p (Lemma 1 proof; Alg. 4 "Multi-request       */
/* Parallel Goldberg-PIR").  DB = r records x s words;     */
/* one word = one record byte (DESIGN R17), p = 65537 by default        */
/* (SPEC S:196).  Server i evaluates at alpha_i = i + 1.   */
/* ------------------------------------------------------------------ */
#define QO_DOMAIN_F 0x46u

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) { return (a * b) % p; }

static uint64_t powmod(uint64_t a, uint64_t e, uint64_t p) {
  uint64_t r = 1 % p;
  a %= p;
  while (e) {
    if (e & 1) r = mulmod(r, a, p);
    a = mulmod(a, a, p);
    e >>= 1;
  }
  return r;
}

/* Client.Query (Lemma 1 proof): for each record index j a random
 * polynomial f_j of degree t with f_j(0) = e_theta[j]; server i receives
 * rho_i[j] = f_j(alpha_i), alpha_i = i + 1.  Coefficient a_k of f_j
 * (k = 1..t) = Philox(key = seed, ctr = (j, k, theta, 'F'))[0] mod p
 * (DESIGN R18).  shares: l x r u32.  p < 2^31 so products fit in u64. */
void qo_ftr_query(uint64_t theta, uint64_t r, uint32_t l, uint32_t t, uint32_t p,
                  uint64_t seed, uint32_t *shares) {
  uint32_t key[2];
  key_from_seed(seed, key);
  for (uint64_t j = 0; j < r; ++j) {
    for (uint32_t i = 0; i < l; ++i) {
      uint64_t x = (uint64_t)i + 1;
      uint64_t val = (j == theta) ? 1u : 0u; /* f_j(0) = e_theta[j] */
      uint64_t xk = 1;
      for (uint32_t k = 1; k <= t; ++k) {
        uint32_t ctr[4] = {(uint32_t)j, k, (uint32_t)theta, QO_DOMAIN_F};
        uint32_t out[4];
        qo_philox4x32_10(ctr, key, out);
        xk = mulmod(xk, x, p);
        val = (val + mulmod(out[0] % p, xk, p)) % p;
      }
      shares[(uint64_t)i * r + j] = (uint32_t)val;
    }
  }
}

/* DB.Query.Response (Lemma 1 proof "R_j := rho_j . DB"; Alg. 4 steps
 * 14-15): out[b] = sum_j rho[j] * DB[j][b] mod p.  records: r x s bytes. */
void qo_ftr_respond(const uint8_t *records, uint64_t r, uint64_t s, const uint32_t *rho,
                    uint32_t p, uint32_t *out) {
  for (uint64_t b = 0; b < s; ++b) {
    uint64_t acc = 0;
    for (uint64_t j = 0; j < r; ++j)
      acc = (acc + (uint64_t)rho[j] * records[j * s + b]) % p;
    out[b] = (uint32_t)acc;
  }
}

void qo_ftr_respond_batch(const uint8_t *records, uint64_t r, uint64_t s, const uint32_t *Q,
                          uint64_t B, uint32_t p, uint32_t *out) {
  int64_t BB = (int64_t)B;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < BB; ++b)
    qo_ftr_respond(records, r, s, Q + (uint64_t)b * r, p, out + (uint64_t)b * s);
}

/* BlockReconst (Def. 1): Lagrange interpolation at 0 of k responses
 * with evaluation points alpha (k distinct nonzero elements):
 * out[b] = sum_i lambda_i * resp[i][b] mod p,
 * lambda_i = prod_{m != i} alpha_m / (alpha_m - alpha_i).  Modular inverse by
 * Fermat's little theorem (p prime).  Returns -1 if two alphas coincide. */
int qo_ftr_reconstruct(const uint32_t *resp, const uint32_t *alpha, uint32_t k, uint64_t s,
                       uint32_t p, uint32_t *out) {
  for (uint64_t b = 0; b < s; ++b) out[b] = 0;
  for (uint32_t i = 0; i < k; ++i) {
    uint64_t num = 1, den = 1;
    for (uint32_t m = 0; m < k; ++m) {
      if (m == i) continue;
      uint64_t am = alpha[m] % p, ai = alpha[i] % p;
      if (am == ai) return -1;
      num = mulmod(num, am, p);
      den = mulmod(den, (am + p - ai) % p, p);
    }
    uint64_t lam = mulmod(num, powmod(den, p - 2, p), p);
    for (uint64_t b = 0; b < s; ++b)
      out[b] = (uint32_t)((out[b] + mulmod(lam, resp[(uint64_t)i * s + b], p)) % p);
  }
  return 0;
}

/* Robust BlockReconst ("nu-Byzantine fault tolerance"; Lemma 1 proof,
 * P:1227): Berlekamp-Welch unique decoding of the k
 * responses, which are evaluations y_i = F(alpha_i) of a polynomial F of
 * degree <= t (sum_j f_j(x) DB[j][b], each f_j of degree t) with up to
 * e = floor((k - t - 1) / 2) of them wrong.  Per word b, the textbook steps:
 *   1. unknowns: E(x) = x^e + E_{e-1} x^{e-1} + ... + E_0 (error locator, monic)
 *      and Q(x) = Q_0 + ... + Q_{e+t} x^{e+t};
 *   2. the k linear equations Q(alpha_i) = y_i E(alpha_i), i.e.
 *      sum_c Q_c alpha_i^c - y_i sum_{a<e} E_a alpha_i^a = y_i alpha_i^e,
 *      solved by Gaussian elimination over F_p (free unknowns set to 0: any
 *      solution gives Q = F E when at most e responses are wrong);
 *   3. F = Q / E by polynomial long division; the remainder must be 0 and
 *      deg F <= t;
 *   4. F must agree with at least k - e responses (else: more than e errors);
 *   5. the word is F(0) (= the record byte, since f_j(0) = e_theta[j]).
 * The paper's Guruswami-Sudan list decoder reaches nu < k - floor(sqrt(k t))
 * (P:1227); unique decoding stops at e (DESIGN R21).  bad[i] (if not NULL) is
 * set to 1 for every server whose response disagrees with F in some word.
 * Returns 0 on success, 1 if k <= t (too few responses), 2 if decoding fails
 * (more errors than e), -1 if two alphas coincide.  p prime, k <= 64. */
int qo_ftr_decode_bw(const uint32_t *resp, const uint32_t *alpha, uint32_t k, uint64_t s,
                     uint32_t t, uint32_t p, uint32_t *out, uint32_t *bad) {
  if (k <= t) return 1;
  if (k > 64) return 1;
  for (uint32_t i = 0; i < k; ++i)
    for (uint32_t m = i + 1; m < k; ++m)
      if (alpha[i] % p == alpha[m] % p) return -1;
  const uint32_t e = (k - t - 1) / 2;
  const uint32_t nq = e + t + 1, nu = nq + e; /* unknowns: Q_0..Q_{e+t}, E_0..E_{e-1} */
  uint64_t M[64][130];                        /* k x (nu + 1) augmented matrix */
  if (bad)
    for (uint32_t i = 0; i < k; ++i) bad[i] = 0;
  for (uint64_t b = 0; b < s; ++b) {
    /* step 2: the linear system */
    for (uint32_t i = 0; i < k; ++i) {
      const uint64_t a = alpha[i] % p, y = resp[(uint64_t)i * s + b] % p;
      uint64_t apow = 1;
      for (uint32_t c = 0; c < nq; ++c) {
        M[i][c] = apow;
        if (c < e) M[i][nq + c] = (p - mulmod(y, apow, p)) % p;
        apow = mulmod(apow, a, p);
      }
      M[i][nu] = mulmod(y, powmod(a, e, p), p);
    }
    /* Gaussian elimination to reduced row echelon form */
    uint32_t pivcol[64];
    uint32_t rank = 0;
    for (uint32_t c = 0; c < nu && rank < k; ++c) {
      uint32_t piv = rank;
      while (piv < k && M[piv][c] == 0) ++piv;
      if (piv == k) continue;
      for (uint32_t x = 0; x <= nu; ++x) {
        uint64_t tmp = M[rank][x];
        M[rank][x] = M[piv][x];
        M[piv][x] = tmp;
      }
      const uint64_t inv = powmod(M[rank][c], p - 2, p);
      for (uint32_t x = 0; x <= nu; ++x) M[rank][x] = mulmod(M[rank][x], inv, p);
      for (uint32_t i = 0; i < k; ++i) {
        if (i == rank || M[i][c] == 0) continue;
        const uint64_t f = M[i][c];
        for (uint32_t x = 0; x <= nu; ++x) M[i][x] = (M[i][x] + p - mulmod(f, M[rank][x], p)) % p;
      }
      pivcol[rank++] = c;
    }
    for (uint32_t i = rank; i < k; ++i)
      if (M[i][nu] != 0) return 2; /* inconsistent: more than e errors */
    uint64_t sol[129];
    for (uint32_t c = 0; c < nu; ++c) sol[c] = 0;
    for (uint32_t i = 0; i < rank; ++i) sol[pivcol[i]] = M[i][nu];
    /* step 3: F = Q / E, E monic of degree e */
    uint64_t Q[129], E[65], F[129];
    for (uint32_t c = 0; c < nq; ++c) Q[c] = sol[c];
    for (uint32_t a = 0; a < e; ++a) E[a] = sol[nq + a];
    E[e] = 1;
    for (uint32_t c = 0; c < nq; ++c) F[c] = 0;
    for (int32_t c = (int32_t)nq - 1; c >= (int32_t)e; --c) {
      const uint64_t q = Q[c]; /* leading coefficient / 1 */
      F[c - e] = q;
      for (uint32_t a = 0; a <= e; ++a)
        Q[c - e + a] = (Q[c - e + a] + p - mulmod(q, E[a], p)) % p;
    }
    for (uint32_t c = 0; c < e; ++c)
      if (Q[c] != 0) return 2; /* E does not divide Q */
    /* deg F <= t holds by construction (deg Q - e <= t) */
    /* step 4: agreement */
    uint32_t agree = 0;
    for (uint32_t i = 0; i < k; ++i) {
      const uint64_t a = alpha[i] % p;
      uint64_t v = 0;
      for (int32_t c = (int32_t)t; c >= 0; --c) v = (mulmod(v, a, p) + F[c]) % p;
      if (v == resp[(uint64_t)i * s + b] % p)
        ++agree;
      else if (bad)
        bad[i] = 1;
    }
    if (agree + e < k) return 2;
    out[b] = (uint32_t)F[0]; /* step 5 */
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* NEXT-3: QPADL-OOP = CIP-PIR offline-online (P:930-942;       */
/* Lemma 2 proof).  B blocks (records of d bytes) in n chunks  */
/* of k = B / n blocks; full replication t = n; server i's */
/* flip chunk is chunk i, its non-flip chunks in rotated order          */
/* chunk_{i+1}, ..., chunk_{i+n-1} (DESIGN R19).                        */
/* ------------------------------------------------------------------ */
#define QO_DOMAIN_O 0x4Fu

/* PRG(S, nbits) (DESIGN R19): bit p = bit (p & 31) of word w = p >> 5,
 * word w = Philox(key = S, ctr = (w >> 2, 0, 0, 'O'))[w & 3]. */
static uint32_t oop_prg_bit(uint64_t seed, uint64_t p) {
  uint32_t key[2];
  key_from_seed(seed, key);
  uint64_t w = p >> 5;
  uint32_t ctr[4] = {(uint32_t)(w >> 2), 0u, 0u, QO_DOMAIN_O};
  uint32_t out[4];
  qo_philox4x32_10(ctr, key, out);
  return (out[w & 3] >> (p & 31)) & 1u;
}

/* Non-flip position p in [0, k(n-1)) of server i -> block index theta. */
static uint64_t oop_nonflip_block(uint64_t p, uint64_t k, uint32_t n, uint32_t i) {
  uint64_t chunk = (i + 1 + p / k) % n;
  return chunk * k + p % k;
}

/* Offline preprocessing of server i (P:930 steps 1-3): q = PRG(S, k(n-1)),
 * A = XOR of the non-flip blocks whose bit in q is set.  out: d bytes. */
void qo_oop_preprocess(const uint8_t *records, uint64_t B, uint64_t d, uint32_t n, uint32_t i,
                       uint64_t seed, uint8_t *A) {
  uint64_t k = B / n;
  memset(A, 0, (size_t)d);
  for (uint64_t p = 0; p < k * (n - 1); ++p) {
    if (oop_prg_bit(seed, p)) {
      const uint8_t *row = records + oop_nonflip_block(p, k, n, i) * d;
      for (uint64_t j = 0; j < d; ++j) A[j] ^= row[j];
    }
  }
}

/* Client query: Q = e_theta (B bits); for every server j, XOR
 * PRG(S_j, k(n-1)) into the positions of j's non-flip blocks; q_j = Q
 * restricted to chunk j.  seeds: n; q: n x ceil(k/8) bytes (bit b of q_j =
 * block j*k + b). */
void qo_oop_query(uint64_t theta, uint64_t B, uint32_t n, const uint64_t *seeds, uint8_t *q) {
  uint64_t k = B / n, kb = (k + 7) / 8;
  memset(q, 0, (size_t)(n * kb));
  /* Q as one bit per block, built plainly */
  for (uint64_t blk = 0; blk < B; ++blk) {
    uint32_t bit = (blk == theta) ? 1u : 0u;
    for (uint32_t j = 0; j < n; ++j) {
      if (blk / k == j) continue; /* flip chunk of server j */
      uint64_t rot = (blk / k + n - j - 1) % n; /* position of this chunk in j's non-flip order */
      uint64_t p = rot * k + blk % k;
      bit ^= oop_prg_bit(seeds[j], p);
    }
    uint64_t owner = blk / k;
    uint64_t b = blk % k;
    if (bit) q[owner * kb + (b >> 3)] |= (uint8_t)(1u << (b & 7));
  }
}

/* Online response of server i (Lemma 2: R_i := A_i XOR q_i . chunk_flip):
 * touches only chunk i (1/n of the DB).  out: d bytes. */
void qo_oop_respond(const uint8_t *records, uint64_t B, uint64_t d, uint32_t n, uint32_t i,
                    const uint8_t *q_i, const uint8_t *A_i, uint8_t *out) {
  uint64_t k = B / n;
  memcpy(out, A_i, (size_t)d);
  for (uint64_t b = 0; b < k; ++b) {
    if ((q_i[b >> 3] >> (b & 7)) & 1u) {
      const uint8_t *row = records + ((uint64_t)i * k + b) * d;
      for (uint64_t j = 0; j < d; ++j) out[j] ^= row[j];
    }
  }
}

/* ------------------------------------------------------------------ */
/* NEXT-4: PSD.Puzzle.Bind with HCT puzzles (Alg. 1 step 1). */
/* ------------------------------------------------------------------ */
/* HCT.Puzzle.Gen(1^lambda, kappa): "randomly selects n_s <-$ {0,1}^lambda
 * and sets the number of leaves n_l based on the difficulty level kappa; the
 * puzzle is Pi = (h, n_s, kappa, n_l)".  Sizes: "a lambda-bit nonce
 * (n_s), a 4-byte difficulty (kappa), and a 1-byte level (n_l), totaling 37
 * bytes" -> lambda = 256.  Encoding (DESIGN R21): n_s || kappa (u32 LE) || n_l;
 * h (the hash function) is fixed by the system, not stored; n_l is the caller's
 * level byte (the paper gives no kappa -> n_l map).  Randomness (DESIGN R21):
 * n_s word w (w = 0..7, little-endian) = Philox4x32-10(key = seed_psd,
 * ctr = (theta_lo, theta_hi, w >> 2, 0x48))[w & 3]. */
void qo_hct_puzzle_gen(uint64_t seed_psd, uint64_t theta, uint32_t kappa, uint8_t n_l,
                       uint8_t out[37]) {
  uint32_t key[2];
  key_from_seed(seed_psd, key);
  for (uint32_t w = 0; w < 8; ++w) {
    uint32_t ctr[4] = {(uint32_t)(theta & 0xFFFFFFFFu), (uint32_t)(theta >> 32), w >> 2, 0x48u};
    uint32_t r[4];
    qo_philox4x32_10(ctr, key, r);
    for (int b = 0; b < 4; ++b) out[4 * w + b] = (uint8_t)(r[w & 3] >> (8 * b));
  }
  for (int b = 0; b < 4; ++b) out[32 + b] = (uint8_t)(kappa >> (8 * b));
  out[36] = n_l;
}

/* Puzzle.Bind over records theta0 .. theta0 + n - 1 (Alg. 1 step 1: for every
 * theta, pi_theta <- Puzzle.Gen; sigma <- ML-DSA.Sign(sk, pi_theta);
 * DB.Record(pi_theta, sigma)).  Record layout (DESIGN R11): bytes
 * [0, 560) spectrum data (the caller's, row theta - theta0 of `spectrum`,
 * stride spec_stride >= 560), [560, 597) pi_theta, [597, 3017) the ML-DSA
 * signature slot -- ML-DSA is not implemented (no FIPS 204 implementation or
 * KAT vectors in this environment), so the slot is left zero ("unsigned") --
 * and zero from 3017 to d.  Requires d >= 597.  out: n x d bytes. */
void qo_puzzle_bind_hct(const uint8_t *spectrum, uint64_t spec_stride, uint64_t theta0,
                        uint64_t n, uint64_t seed_psd, uint32_t kappa, uint8_t n_l,
                        uint64_t d, uint8_t *out) {
  for (uint64_t i = 0; i < n; ++i) {
    uint8_t *rec = out + i * d;
    memset(rec, 0, (size_t)d);
    memcpy(rec, spectrum + i * spec_stride, 560);
    qo_hct_puzzle_gen(seed_psd, theta0 + i, kappa, n_l, rec + 560);
  }
}
