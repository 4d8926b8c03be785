/*
 * qpir.h -- C ABI of the B200-native LWE-PIR answer engine (libqpir.so).
 *
 * The server side of the PIR of QPADL (arXiv 2510.03631) read as a Regev-LWE
 * PIR (R1): the spectrum database is a matrix D over Z_p (p = 2^8,
 * one record byte per entry), a client query is qu in Z_q^m (q = 2^32), and
 *   answer        ans = D . qu            mod 2^32   (Def. 1 "DB.Query.Response",
 *                                                     PAPER.md:241; Alg. 1 step 18,
 *                                                     PAPER.md:591)
 *   batch answer  ANS = D . Q             mod 2^32   (multi-request form, Alg. 3/4,
 *                                                     PAPER.md:981)
 *   hint          H   = D . A             mod 2^32   (offline precomputation,
 *                                                     PAPER.md:1091-1092; DESIGN R7)
 * All arithmetic is exact in Z_{2^32} (u32 wrap-around), so every result has a
 * unique correct value and is bit-identical across GPUs, shards, split factors
 * and streams.
 *
 * Conventions (SPEC.md:204 little-endian u32 elements; SPEC.md:93 DB immutable
 * after build; SPEC.md:248 output independent of worker count):
 *   - Geometry (DESIGN R9/R10): theta = cell * n_ch + ch indexes the N =
 *     n_cells * n_ch records of rec_bytes = d bytes each.  blk = cell / m,
 *     col = cell % m, row = (blk * n_ch + ch) * d + b holds byte b of record
 *     theta; ell = ceil(n_cells / m) * n_ch * d rows.  A context owns the row
 *     shard [row_begin, row_end) of [0, ell) ("ell_local" rows).
 *   - Buffers: every pointer argument may be host memory (pageable or pinned)
 *     or device memory of the context's device; the library detects which with
 *     cudaPointerGetAttributes.  The caller owns every buffer it passes; the
 *     context owns its device copy of the D shard and its scratch.
 *   - Lengths: every buffer comes with its element count, which must match the
 *     geometry exactly, else QPIR_E_DIMENSION and nothing is written.
 *   - Streams: `stream` is a cudaStream_t (NULL = legacy default stream).  Work
 *     is enqueued on it.  If any output is host memory the call synchronises
 *     the stream before returning; with device outputs it returns immediately.
 *     Host inputs are copied on a copy stream the library owns (per context
 *     and stream), which `stream` then waits on: pageable inputs may be reused
 *     as soon as the call returns; pinned inputs must stay unchanged until
 *     `stream` has passed the call (as with cudaMemcpyAsync on `stream`).
 *   - Concurrency: answer / batch / hint calls on one context may run
 *     concurrently on different streams (each stream gets its own scratch
 *     arena: staging buffers, split-K partials, tickets); calls on one stream
 *     are ordered by that stream.  qpir_db_write must not overlap any other
 *     call on the context.  The D shard is never modified by answer/hint calls.
 *   - CUDA graphs: answer / batch / hint calls with device buffers may be
 *     captured into a CUDA graph (relaxed or thread-local capture mode) once a
 *     first eager call on that stream has sized its scratch; the graph reads
 *     the caller's buffers at replay time.  Back-to-back GEMV answers (and ENS
 *     scans) are launched with programmatic dependent launch: the next one
 *     starts streaming D while the previous one drains, and waits for it
 *     before touching any buffer the previous one writes.
 *   - Errors: functions return QPIR_OK (0) or a QPIR_E_* code; no partial
 *     outputs on error.  qpir_last_error(ctx) (or qpir_last_error(NULL) for a
 *     failed qpir_setup) names the offending field, e.g. "m: 8191 != 8192".
 *
 * The cross-GPU gather of answer slices is not part of this ABI: each rank
 * calls it on its own shard and the Python layer gathers over NCCL.
 */
#ifndef QPIR_H
#define QPIR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QPIR_OK 0
#define QPIR_E_PARAM 1     /* unsupported parameter (log_q, log_p, lwe_n, ...) */
#define QPIR_E_DIMENSION 2 /* a length or the shard geometry does not match     */
#define QPIR_E_STATE 3     /* call not valid in the context's state             */
#define QPIR_E_OOM 4       /* device or host allocation failed                  */
#define QPIR_E_CUDA 5      /* a CUDA runtime call failed (message has details)  */

typedef struct qpir_ctx qpir_ctx;

typedef struct {
  uint64_t n_cells;   /* location cells (grid (l_x, l_y) flattened) */
  uint64_t n_ch;      /* channels per cell                                        */
  uint64_t rec_bytes; /* d: bytes per record (3072 for paper-shaped records)      */
  uint64_t m;         /* DB columns; 0 means m = n_cells                          */
  uint32_t lwe_n;     /* LWE dimension n (width of the hint), 1..65536            */
  uint32_t log_q;     /* must be 32 (q = 2^32, DESIGN R2)                          */
  uint32_t log_p;     /* must be 8  (p = 2^8,  DESIGN R3)                          */
  uint32_t reserved0; /* must be 0                                                */
  uint64_t seed_A;    /* public-matrix seed: A[c][j] = Philox4x32-10(key = seed_A,
                         ctr = (c, j >> 2, 0, 0x41))[j & 3]  (DESIGN R7)          */
  uint64_t row_begin; /* this context's shard [row_begin, row_end) of [0, ell);   */
  uint64_t row_end;   /* row_end = 0 means ell (the whole matrix)                 */
  int32_t device;     /* CUDA device ordinal                                      */
  int32_t flags;      /* 0 or QPIR_FLAG_STABLE_INPUTS                             */
} qpir_params;

/* Caller's promise: a device query / share buffer passed to an answer call is
 * never written by the kernel that immediately precedes that call on its
 * stream.  The answer kernels are launched with programmatic dependent launch
 * (they may start while the previous kernel on the stream drains, and that
 * kernel's writes are visible only after griddepcontrol.wait); with the flag
 * they read their inputs before the wait, overlapping the previous grid's
 * tail.  Without it only the DB is read before the wait (host inputs are staged
 * by the library and are always read early). */
#define QPIR_FLAG_STABLE_INPUTS 1

/* Create a context on params->device holding the D shard.  `records` is the
 * full theta-ordered record array (n_cells * n_ch * rec_bytes bytes, host or
 * device) or NULL for an all-zero DB to be filled with qpir_db_write.  Only the
 * records that land in the shard are read.  On success *out owns the device
 * memory; release it with qpir_destroy.  Parameters are validated before any
 * CUDA call (QPIR_E_PARAM / QPIR_E_DIMENSION without touching the device).
 * Setup step a1 "DB pack" (DB.Record). */
int qpir_setup(const qpir_params *params, const uint8_t *records,
               uint64_t records_len, void *stream, qpir_ctx **out);

/* Write records theta_begin .. theta_begin + n_records - 1 (n_records * d
 * bytes, theta order, host or device) into the shard; records outside the
 * shard's rows are skipped.  Lets a caller stream a DB larger than host or
 * device memory in chunks.  Not to be called concurrently with answers. */
int qpir_db_write(qpir_ctx *ctx, uint64_t theta_begin, uint64_t n_records,
                  const uint8_t *records, uint64_t records_len, void *stream);

/* NEXT-4: PSD.Puzzle.Bind with HCT puzzles, on the GPU (Alg. 1 step 1,
 * PAPER.md:553-566; HCT.Puzzle.Gen PAPER.md:855; record layout PAPER.md:1686,
 * DESIGN R11 / R21).  Builds records theta_begin .. theta_begin + n_records - 1
 * and writes them into the shard exactly as qpir_db_write would:
 *   record = spectrum row (its first 560 bytes) || pi_theta = n_s (32 B) ||
 *            kappa (u32 LE) || n_l (1 B) || sigma (2420 B) || zero padding
 * with the 256-bit nonce n_s word w = Philox4x32-10(key = seed_psd,
 * ctr = (theta_lo, theta_hi, w >> 2, 0x48))[w & 3], and sigma the ML-DSA-44
 * signature of the 37-byte pi_theta (FIPS 204, deterministic variant, empty
 * context) under the key generated from the 32-byte seed mldsa_seed (host or
 * device; KeyGen and Sign run on the GPU).  mldsa_seed == NULL leaves the
 * signature slot zero (unsigned DB).  mldsa_pk (1312 bytes, host or device, may
 * be NULL) receives the public key.
 * spectrum: n_records rows of spec_stride >= 560 bytes, host or device
 * (spectrum_len == n_records * spec_stride); requires rec_bytes >= 597 (>= 3017
 * when signing).
 * Device memory owned by the context (kept for later calls): a host spectrum is
 * staged in <= 64 MB chunks; signing stages up to 65536 signature rows of 3024
 * bytes (198 MB) per launch, plus the expanded key (~29 KB).
 * Errors: QPIR_E_DIMENSION (range, lengths, stride, rec_bytes), QPIR_E_PARAM
 * (NULL spectrum), QPIR_E_OOM / QPIR_E_CUDA.  Concurrency as qpir_db_write. */
int qpir_puzzle_bind_hct(qpir_ctx *ctx, uint64_t theta_begin, uint64_t n_records,
                         const uint8_t *spectrum, uint64_t spec_stride,
                         uint64_t spectrum_len, uint64_t seed_psd, uint32_t kappa,
                         uint8_t n_l, const uint8_t *mldsa_seed, uint8_t *mldsa_pk,
                         void *stream);

/* Geometry: ell (all rows), m (columns), ell_local (= row_end - row_begin),
 * row_begin.  Any output pointer may be NULL. */
int qpir_geometry(const qpir_ctx *ctx, uint64_t *ell, uint64_t *m,
                  uint64_t *ell_local, uint64_t *row_begin);

/* Single query (step a3):
 *   ans_local[i] = sum_{c < m} D[row_begin + i][c] * qu[c]  mod 2^32.
 * qu: m u32 (len must equal m).  ans_local: ell_local u32 (len == ell_local). */
int qpir_answer(qpir_ctx *ctx, const uint32_t *qu, uint64_t len_qu,
                uint32_t *ans_local, uint64_t len_ans, void *stream);

/* Batch of B queries (step a6):
 *   ans_local[b * ell_local + i] = sum_c D[row_begin + i][c] * Q[b * m + c] mod 2^32.
 * Q: B x m u32 query-major (len == B * m); ans_local: B x ell_local (len ==
 * B * ell_local).  1 <= B <= 4096.  u32 device pointers must be 4-byte aligned.
 * The byte-limb planes of Q are built in chunks of queries under a 2 GiB budget
 * (env QPIR_LIMB_BUDGET_MB), so B and m only bound the output size. */
int qpir_answer_batch(qpir_ctx *ctx, const uint32_t *Q, uint64_t B,
                      uint64_t len_Q, uint32_t *ans_local, uint64_t len_ans,
                      void *stream);

/* Batch over a prime field (NEXT-2, QPADL-FTR: Goldberg robust PIR,
 * PAPER.md:740; the "q . DB mod q" GEMM of Alg. 4):
 *   ans_local[b * ell_local + i] = (sum_c D[row_begin + i][c] * Q[b * m + c]) mod p,
 * exact for any u32 Q entries and any 2 <= p < 2^32 (results < p).  With
 * n_ch = 1 and n_cells = r records, row b of D is byte b of every record, so
 * row i of the answer is word i of the FTR response rho . DB (one word = one
 * record byte, DESIGN R17).  Same buffers and B range as qpir_answer_batch.
 * Internally the entries are reduced mod p first and split into 2 byte limbs
 * for p <= 65537 (the residue 65536 of p = 65537 is listed per query and added
 * back by the mod-p fixup), 3 for p <= 2^24, 4 otherwise: the cost falls with
 * p, the result does not depend on the path.  The 2-limb split normally runs
 * inside the GEMM (converter warps); on a stream that is being captured into a
 * CUDA graph it runs as a separate kernel instead, so the captured work replays
 * exactly (the fused form keeps per-launch state on the host). */
int qpir_answer_batch_modp(qpir_ctx *ctx, const uint32_t *Q, uint64_t B,
                           uint64_t len_Q, uint32_t p, uint32_t *ans_local,
                           uint64_t len_ans, void *stream);

/* Hint (step a7): H_local[i * n + j] = sum_c D[row_begin + i][c] * A[c][j]
 * mod 2^32 with A expanded from seed_A on the device (n = lwe_n).  H_local:
 * ell_local x n row-major (len == ell_local * n). */
int qpir_hint(qpir_ctx *ctx, uint32_t *H_local, uint64_t len_H, void *stream);

/* Number of kernels this context has launched so far (for launch accounting). */
uint64_t qpir_kernel_launches(const qpir_ctx *ctx);

/* Last error message of ctx, or of the calling thread's last failed
 * qpir_setup when ctx is NULL.  Never NULL; "" if no error. */
const char *qpir_last_error(const qpir_ctx *ctx);

/* Free the context and its device memory (NULL is a no-op). */
void qpir_destroy(qpir_ctx *ctx);

/* ===================================================================== */
/* QPADL-ENS: Chor multi-server XOR PIR (Lemma 1 proof,     */
/* PAPER.md:1227; Alg. 3 "Multi-request Parallel Chor-PIR"). */
/* The DB is r records of d bytes (b = 8d bits over GF(2)), theta-major.   */
/* A share is an r-bit vector, bit t at byte t >> 3, bit (t & 7); bits at  */
/* positions >= r are ignored.  The response to a share is the XOR of the  */
/* records whose bit is 1 (rho = q . DB over GF(2)); a client XORs the l   */
/* responses of l servers to rebuild its record.  Same buffer, length,     */
/* stream, error and concurrency conventions as above (per-stream scratch: */
/* calls on different streams may run concurrently).                       */
/* ===================================================================== */
typedef struct qpir_ens_ctx qpir_ens_ctx;

typedef struct {
  uint64_t n_records; /* r                                       */
  uint64_t rec_bytes; /* d, 1..16384                             */
  int32_t device;     /* CUDA device ordinal                     */
  int32_t flags;      /* 0 or QPIR_FLAG_STABLE_INPUTS (shares)   */
} qpir_ens_params;

/* Create an ENS context holding all r records (records may be NULL: zero DB). */
int qpir_ens_setup(const qpir_ens_params *params, const uint8_t *records,
                   uint64_t records_len, void *stream, qpir_ens_ctx **out);

/* Overwrite records theta_begin .. theta_begin + n_records - 1. */
int qpir_ens_db_write(qpir_ens_ctx *ctx, uint64_t theta_begin, uint64_t n_records,
                      const uint8_t *records, uint64_t records_len, void *stream);

/* NEXT-4 on an ENS context: as qpir_puzzle_bind_hct, the records written in
 * place (theta-major rows). */
int qpir_ens_puzzle_bind_hct(qpir_ens_ctx *ctx, uint64_t theta_begin, uint64_t n_records,
                             const uint8_t *spectrum, uint64_t spec_stride,
                             uint64_t spectrum_len, uint64_t seed_psd, uint32_t kappa,
                             uint8_t n_l, const uint8_t *mldsa_seed, uint8_t *mldsa_pk,
                             void *stream);

/* Response to one share (len_share == ceil(r/8)) -> out: d bytes (len_out == d).
 * A 4-byte-aligned device share may be read in whole 32-bit words (up to 3
 * bytes past len_share, within the allocation granularity of cudaMalloc). */
int qpir_ens_answer(qpir_ens_ctx *ctx, const uint8_t *share, uint64_t len_share,
                    uint8_t *out, uint64_t len_out, void *stream);

/* Responses to B shares (B x ceil(r/8), share-major) -> out: B x d bytes.
 * 1 <= B <= 65536 (Alg. 3 multi-request form).  For B >= 32
 * the GF(2) product runs on tensor cores (records read once in place and
 * expanded on chip; the shares take B * r bytes of scratch as 0/1 bytes);
 * smaller B use a CUDA-core XOR kernel.  qpir_ens_last_path reports which. */
int qpir_ens_answer_batch(qpir_ens_ctx *ctx, const uint8_t *shares, uint64_t B,
                          uint64_t len_shares, uint8_t *out, uint64_t len_out,
                          void *stream);

/* QPADL-OOP = CIP-PIR offline-online on the same context (NEXT-3; PAPER.md:744,
 * PAPER.md:930-942; Lemma 2 proof).  The r records form n_chunks
 * chunks of k = r / n_chunks blocks (n_chunks must divide r); full replication,
 * server i's flip chunk is chunk i, its non-flip chunks in rotated order
 * chunk_{i+1}, ..., chunk_{i+n-1} (DESIGN R19).
 * Offline: for each seed S, q = PRG(S, k(n-1)) over the non-flip blocks,
 *   A = XOR of the selected blocks (A_out: n_seeds x d bytes).  PRG word w =
 *   Philox4x32-10(key = S, ctr = (w >> 2, 0, 0, 0x4F))[w & 3], bit p of the
 *   stream = bit (p & 31) of word p >> 5.
 * Online: R_i = A_i XOR q_i . chunk_i, q_i: k bits (ceil(k/8) bytes), touching
 *   only chunk i (1/n of the DB).  1 <= n_seeds <= 65535. */
int qpir_oop_preprocess(qpir_ens_ctx *ctx, uint32_t n_chunks, uint32_t server,
                        const uint64_t *seeds, uint64_t n_seeds, uint8_t *A_out,
                        uint64_t len_A, void *stream);
int qpir_oop_answer(qpir_ens_ctx *ctx, uint32_t n_chunks, uint32_t server,
                    const uint8_t *q, uint64_t len_q, const uint8_t *A, uint64_t len_A,
                    uint8_t *out, uint64_t len_out, void *stream);

uint64_t qpir_ens_kernel_launches(const qpir_ens_ctx *ctx);

/* Which kernel path the last ENS/OOP call of this context took (for reports). */
#define QPIR_ENS_PATH_NONE 0       /* no call yet                              */
#define QPIR_ENS_PATH_SCAN 1       /* single-share scan (answer / OOP online)  */
#define QPIR_ENS_PATH_CUDA_CORES 2 /* multi-request XOR kernel on CUDA cores   */
#define QPIR_ENS_PATH_TENSOR 3     /* multi-request GF(2) product on tcgen05   */
int qpir_ens_last_path(const qpir_ens_ctx *ctx);
const char *qpir_ens_last_error(const qpir_ens_ctx *ctx);
void qpir_ens_destroy(qpir_ens_ctx *ctx);

/* ===================================================================== */
/* Cross-rank combine of record-sharded NEXT rows (dist.py, one process per */
/* GPU): after an all-gather of the n_parts per-rank partial responses     */
/* (rank-major, n_parts x len), fold them on the device.  parts and out    */
/* must be device memory of one device (QPIR_E_PARAM otherwise: there is   */
/* no host fallback); the kernel is queued on `stream`, no sync.           */
/* ===================================================================== */
/* ENS / OOP (GF(2); Lemma 1 proof PAPER.md:1227, Alg. 3):
 * out[i] = XOR over r of parts[r * len + i]  (len bytes). */
int qpir_xor_fold(const uint8_t *parts, uint64_t n_parts, uint64_t len, uint8_t *out,
                  void *stream);
/* FTR (F_p; Lemma 1 proof "R_j := rho_j . DB", Alg. 4):
 * out[i] = (sum over r of parts[r * len + i]) mod p, summed exactly in 64 bits;
 * 1 <= n_parts <= 2^32, p >= 2. */
int qpir_sum_mod_p(const uint32_t *parts, uint64_t n_parts, uint64_t len, uint32_t p,
                   uint32_t *out, void *stream);
/* Message of the last failed combine call of this thread ("" if none). */
const char *qpir_combine_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* QPIR_H */
