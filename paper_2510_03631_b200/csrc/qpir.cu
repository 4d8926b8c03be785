// qpir.cu -- C ABI (include/qpir.h) of the B200-native LWE-PIR answer engine.
//
// Host side: parameter validation (before any CUDA call), context + device
// memory ownership, host/device buffer detection, kernel dispatch.  Every step
// of the path runs in the kernels of gemv.cuh / mma.cuh / aux_kernels.cuh; there
// is no CPU fallback -- a missing device is an error.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <map>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/qpir.h"
#include "aux_kernels.cuh"
#include "gemv.cuh"
#include "host_common.h"
#include "mma_launch.cuh"
#include "puzzle.cuh"
#include "mldsa.cuh"

using namespace qpir;
using namespace qpir_host;

namespace {

thread_local std::string g_setup_error;

struct Geometry {
  uint64_t n_cells, n_ch, d, m, ell, row_begin, row_end, ell_local;
  uint64_t m_pad, G, L;
  uint32_t lwe_n;
  uint64_t seed_A;
};

}  // namespace

// Host-input staging ring: the H2D copy of call i + 1's query runs on the
// arena's own copy stream while call i's kernels run; the compute stream waits
// only on that copy's event (two slots, each reused once the kernels that read
// it have finished).
struct InRing {
  void* buf[2] = {nullptr, nullptr};
  uint64_t bytes[2] = {0, 0};
  cudaEvent_t ready[2] = {nullptr, nullptr};  // H2D into slot k done (copy stream)
  cudaEvent_t done[2] = {nullptr, nullptr};   // kernels reading slot k done (compute stream)
  unsigned slot = 0;
};

// Per-stream scratch: calls on different streams of one context may run
// concurrently (each stream owns its staging buffers, split-K partials and
// tickets); calls on one stream are ordered by the stream.
struct Arena {
  cudaStream_t h2d = nullptr;      // copy stream for host inputs (lazily created)
  InRing in_small, in_big;         // host qu / host Q staging rings
  uint32_t* qu_dev = nullptr;      // staging for an unaligned device qu
  uint64_t qu_bytes = 0;
  uint32_t* ans_dev = nullptr;     // staging for host answers
  uint64_t ans_bytes = 0;
  uint32_t* partial = nullptr;     // [split][L] GEMV split-K partials
  uint64_t partial_bytes = 0;
  uint32_t* tickets = nullptr;     // [row blocks], zeroed once, self-resetting
  uint64_t tickets_bytes = 0;
  uint8_t* limbs = nullptr;        // Q' or A' limb planes
  uint64_t limbs_bytes = 0;
  uint32_t* big_out = nullptr;     // staging for host ANS / H
  uint64_t big_out_bytes = 0;
  unsigned long long* acc64 = nullptr;  // OUT_MODP accumulator
  uint64_t acc64_bytes = 0;
  uint32_t* kprog = nullptr;       // tcgen05 engine K-lockstep counters [kKprogCap]
  uint32_t* exc = nullptr;         // OUT_MODP2, p = 65537: [Bc] counts + [Bc][cap] columns
  uint64_t exc_bytes = 0;
  uint32_t* kb_done = nullptr;     // fused FTR limb split: per-K-block epoch flags (zeroed once)
  uint64_t kb_done_bytes = 0;
  unsigned long long* conv_ctr = nullptr;  // fused split work counter (monotonic, zeroed once)
  unsigned long long conv_base = 0;        // its value at the next launch
  uint32_t epoch = 0;                      // last epoch published into kb_done
};

struct qpir_ctx {
  Geometry geo;
  int device = 0;
  int num_sms = 148;
  uint8_t* D = nullptr;            // 128-row panels [L/128][G][128][16]
  uint8_t* rec_stage = nullptr;    // host-record staging for db_write
  uint64_t rec_stage_bytes = 0;
  uint8_t* spec_stage = nullptr;   // host spectrum staging for qpir_puzzle_bind_hct
  uint64_t spec_stage_bytes = 0;
  uint8_t* mldsa_buf = nullptr;    // ML-DSA: expanded key + 32-byte seed
  uint64_t mldsa_buf_bytes = 0;
  uint8_t* sig_stage = nullptr;    // ML-DSA signatures, 3024-byte rows
  uint64_t sig_stage_bytes = 0;
  bool bind_sig_attr = false;      // dynamic-smem attribute of the signed packing kernel set
  std::mutex mu;                   // guards `arenas`
  std::map<cudaStream_t, Arena> arenas;
  uint64_t launches = 0;
  // Tuning knobs, read once from the environment at setup (sweeps in profiles/):
  int gemv_u = 2;       // env QPIR_GEMV_U: rows per thread (1, 2, 4)
  int gemv_split = 0;   // env QPIR_GEMV_SPLIT: K splits (0 = auto)
  int gemv_chunk = 512; // env QPIR_GEMV_CHUNK: column groups staged in smem at a time
  int gemv_unroll = 4;  // env QPIR_GEMV_UNROLL: column groups in flight (4 or 8)
  int gemv_order = 0;  // env QPIR_GEMV_ORDER (1 = split-major grid)
  int gemv_pdl = 1;    // env QPIR_GEMV_PDL (programmatic dependent launch of back-to-back GEMVs)
  int gemv_pf256 = 0;  // env QPIR_GEMV_PF256: L2 256-byte prefetch hint on D loads
  int gemv_l2pf = 0;   // env QPIR_GEMV_L2PF: bulk L2 prefetch of a CTA's D slice before the PDL wait
  int flags = 0;       // qpir_params.flags (QPIR_FLAG_STABLE_INPUTS)
  std::atomic<bool> d_written{false};  // a device db_write is queued: next GEMV without PDL
  int mma_mt = 2;      // env QPIR_MMA_MT (1 or 2 row panels per CTA tile)
  int mma_l2hint = 0;  // env QPIR_MMA_L2HINT (MmaArgs::l2hint)
  int mma_split = 0;   // env QPIR_MMA_SPLIT (0 = auto)
  int mma_gpb = 8;     // env QPIR_MMA_GPB (column groups per pipeline stage: 4 or 8)
  int modp3 = 1;       // env QPIR_MODP3 (3 limbs per query for p < 2^24)
  int modp2 = 1;       // env QPIR_MODP2 (2 limbs per query for p <= 65537)
  int ftr_fuse = 1;    // env QPIR_FTR_FUSE (2-limb split inside the GEMM: 8 converter warps;
                       // ftr-c2-b128 0.262-0.264 ms vs 0.269-0.273 ms with the split kernel)
  int h2d_stream = 1;  // env QPIR_H2D_STREAM (host inputs copied on a side stream)
  int mma_ls = 16;     // env QPIR_MMA_LOCKSTEP: K-blocks per lockstep chunk (0 = off)
  int mma_drift = 1;   // env QPIR_MMA_DRIFT: chunks a CTA may run ahead of its wave
  uint64_t limb_budget = 2ull << 30;  // env QPIR_LIMB_BUDGET_MB: max bytes of Q'/A' at once
  std::string err;
};

namespace {

int fail(qpir_ctx* ctx, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx)
    ctx->err = buf;
  else
    g_setup_error = buf;
  return code;
}

#define CUDA_TRY(ctx, call)                                                              \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail((ctx), e_ == cudaErrorMemoryAllocation ? QPIR_E_OOM : QPIR_E_CUDA,     \
                  "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

#define LAUNCH_CHECK(ctx)                                                                 \
  do {                                                                                    \
    (ctx)->launches++;                                                                    \
    cudaError_t e_ = qpir_host::launch_status();                                          \
    if (e_ != cudaSuccess)                                                                \
      return fail((ctx), QPIR_E_CUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                    \
  } while (0)

int validate(const qpir_params* p, Geometry* g) {
  if (!p) return fail(nullptr, QPIR_E_PARAM, "params: NULL");
  if (p->log_q != 32) return fail(nullptr, QPIR_E_PARAM, "log_q: %u != 32", p->log_q);
  if (p->log_p != 8) return fail(nullptr, QPIR_E_PARAM, "log_p: %u != 8", p->log_p);
  if (p->reserved0 != 0) return fail(nullptr, QPIR_E_PARAM, "reserved0: must be 0");
  if (p->flags & ~QPIR_FLAG_STABLE_INPUTS)
    return fail(nullptr, QPIR_E_PARAM, "flags: unknown bits 0x%x", (unsigned)p->flags);
  if (p->lwe_n == 0 || p->lwe_n > 65536)
    return fail(nullptr, QPIR_E_PARAM, "lwe_n: %u not in [1, 65536]", p->lwe_n);
  if (p->n_cells == 0) return fail(nullptr, QPIR_E_DIMENSION, "n_cells: 0");
  if (p->n_ch == 0) return fail(nullptr, QPIR_E_DIMENSION, "n_ch: 0");
  if (p->rec_bytes == 0) return fail(nullptr, QPIR_E_DIMENSION, "rec_bytes: 0");
  if (p->device < 0) return fail(nullptr, QPIR_E_PARAM, "device: %d < 0", p->device);
  g->n_cells = p->n_cells;
  g->n_ch = p->n_ch;
  g->d = p->rec_bytes;
  g->m = p->m ? p->m : p->n_cells;
  if (g->m > (1ull << 30)) return fail(nullptr, QPIR_E_DIMENSION, "m: %llu > 2^30",
                                       (unsigned long long)g->m);
  const uint64_t n_blk = (g->n_cells + g->m - 1) / g->m;
  g->ell = n_blk * g->n_ch * g->d;
  g->row_begin = p->row_begin;
  g->row_end = p->row_end ? p->row_end : g->ell;
  if (g->row_end > g->ell)
    return fail(nullptr, QPIR_E_DIMENSION, "row_end: %llu > ell %llu",
                (unsigned long long)g->row_end, (unsigned long long)g->ell);
  if (g->row_begin >= g->row_end)
    return fail(nullptr, QPIR_E_DIMENSION, "row_begin: %llu >= row_end %llu",
                (unsigned long long)g->row_begin, (unsigned long long)g->row_end);
  g->ell_local = g->row_end - g->row_begin;
  if (g->ell_local > (1ull << 31) - 4096)
    return fail(nullptr, QPIR_E_DIMENSION, "ell_local: %llu too large",
                (unsigned long long)g->ell_local);
  g->m_pad = round_up(g->m, MMA_BK);
  g->G = g->m_pad / 16;
  g->L = round_up(g->ell_local, 2 * MMA_BM);  // whole pairs of 128-row panels
  g->lwe_n = p->lwe_n;
  g->seed_A = p->seed_A;
  return QPIR_OK;
}

int ensure(qpir_ctx* ctx, void** buf, uint64_t* have, uint64_t need) {
  if (*have >= need) return QPIR_OK;
  if (*buf) cudaFree(*buf);
  *buf = nullptr;
  *have = 0;
  CUDA_TRY(ctx, cudaMalloc(buf, need));
  *have = need;
  return QPIR_OK;
}

Arena& arena_for(qpir_ctx* ctx, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(ctx->mu);
  return ctx->arenas[st];  // std::map references stay valid across inserts
}

// Stage `bytes` of host memory for kernels on `st`: H2D on the arena's copy
// stream into the next ring slot, `st` waits on it.  Returns the slot (the
// caller records ring.done[slot] on `st` after the kernels that read it), or
// -1 after a same-stream copy (while `st` is being captured into a CUDA graph,
// or with QPIR_H2D_STREAM=0).
int stage_host(qpir_ctx* ctx, Arena& ar, InRing& ring, const void* src, uint64_t bytes,
               uint64_t alloc, cudaStream_t st, const void** dev, int* slot_out) {
  *slot_out = -1;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CUDA_TRY(ctx, cudaStreamIsCapturing(st, &cs));
  if (cs != cudaStreamCaptureStatusNone || !ctx->h2d_stream) {
    int rc = ensure(ctx, &ring.buf[0], &ring.bytes[0], alloc);
    if (rc) return rc;
    CUDA_TRY(ctx, cudaMemcpyAsync(ring.buf[0], src, bytes, cudaMemcpyHostToDevice, st));
    *dev = ring.buf[0];
    return QPIR_OK;
  }
  if (!ar.h2d) CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ar.h2d, cudaStreamNonBlocking));
  const unsigned k = ring.slot;
  ring.slot ^= 1u;
  if (!ring.ready[k]) {
    CUDA_TRY(ctx, cudaEventCreateWithFlags(&ring.ready[k], cudaEventDisableTiming));
    CUDA_TRY(ctx, cudaEventCreateWithFlags(&ring.done[k], cudaEventDisableTiming));
  }
  if (ring.bytes[k] < alloc) {
    // the slot may still be read by earlier kernels: wait before freeing it
    CUDA_TRY(ctx, cudaEventSynchronize(ring.done[k]));
    int rc = ensure(ctx, &ring.buf[k], &ring.bytes[k], alloc);
    if (rc) return rc;
  }
  CUDA_TRY(ctx, cudaStreamWaitEvent(ar.h2d, ring.done[k], 0));
  CUDA_TRY(ctx, cudaMemcpyAsync(ring.buf[k], src, bytes, cudaMemcpyHostToDevice, ar.h2d));
  CUDA_TRY(ctx, cudaEventRecord(ring.ready[k], ar.h2d));
  CUDA_TRY(ctx, cudaStreamWaitEvent(st, ring.ready[k], 0));
  *dev = ring.buf[k];
  *slot_out = (int)k;
  return QPIR_OK;
}

// NEXT-4: pack_records_kernel with the record bytes generated in place (Puzzle.Bind
// straight into the D panel layout: no record staging buffer).  Same thread map:
// one thread per (row, 16-cell column group); row b of a channel = byte b of its
// records, so all but 32 of a 3072-byte record's rows are a spectrum copy or zeros.
__global__ void pack_bind_kernel(PackArgs a, BindArgs bnd) {
  const uint32_t rl = blockIdx.y * blockDim.x + threadIdx.x;
  if (rl >= a.ell_local) return;
  const uint32_t j = a.g_lo + blockIdx.x;
  const uint64_t row = a.row_begin + rl;
  const uint64_t per_blk = (uint64_t)a.n_ch * a.d;
  const uint64_t blk = row / per_blk;
  const uint32_t rr = (uint32_t)(row % per_blk);
  const uint32_t ch = rr / a.d;
  const uint32_t b = rr % a.d;
  uint4* dst = reinterpret_cast<uint4*>(a.D + ((size_t)(rl >> 7) * a.G + j) * 2048 +
                                        (rl & 127u) * 16);
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  uint8_t* bytes = reinterpret_cast<uint8_t*>(&v);
  uint32_t touched = 0;  // columns written (a full group needs no read of the old bytes)
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t col = j * 16u + i;
    if (col >= a.m) continue;
    const uint64_t cell = blk * a.m + col;
    if (cell >= a.n_cells) continue;
    const uint64_t theta = cell * a.n_ch + ch;
    if (theta < a.theta0 || theta >= a.theta0 + a.n_rec) continue;
    bytes[i] = bound_record_byte(bnd, theta, b);
    touched |= 1u << i;
  }
  if (touched == 0xFFFFu) {
    *dst = v;
  } else if (touched) {
    uint4 o = *dst;
    const uint8_t* ob = reinterpret_cast<const uint8_t*>(&o);
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (!((touched >> i) & 1u)) bytes[i] = ob[i];
    *dst = v;
  }
}

// Register-transposed form (d and the spectrum rows 16-byte aligned): one CTA
// per (16-cell column group j, channel ch, row block blk).  Threads 0..37 each
// take 16 record-byte rows of the 608-byte data prefix (spectrum + puzzle):
// bytes 16t .. 16t + 15 of the 16 cells' records (16-byte loads, coalesced
// across the warp; nonce bytes straight from Philox), a 16 x 16 byte transpose
// in registers (4 x 4 byte transposes of words, 8 PRMT each) into shared
// memory; then all threads store the record-byte rows as 16-byte D chunks,
// consecutive threads on consecutive rows (512 contiguous bytes per warp
// store), rows past the prefix as zeros (the unsigned signature slot).
__device__ __forceinline__ void transpose4x4_bytes(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3,
                                                   uint32_t& y0, uint32_t& y1, uint32_t& y2, uint32_t& y3) {
  const uint32_t t0 = __byte_perm(x0, x1, 0x5140), t1 = __byte_perm(x0, x1, 0x7362);
  const uint32_t t2 = __byte_perm(x2, x3, 0x5140), t3 = __byte_perm(x2, x3, 0x7362);
  y0 = __byte_perm(t0, t2, 0x5410);
  y1 = __byte_perm(t0, t2, 0x7632);
  y2 = __byte_perm(t1, t3, 0x5410);
  y3 = __byte_perm(t1, t3, 0x7632);
}

constexpr uint32_t BIND_HEAD = (HCT_SPECTRUM + HCT_PUZZLE + 15) / 16 * 16;  // 608 rows with data
constexpr uint32_t BIND_HEAD_SIG = HCT_SIG_STRIDE;                              // 3024 with the signature

// SIG: the records carry ML-DSA signatures (rows [597, 3017) from bnd.sig); a
// separate instantiation keeps the unsigned kernel free of the signature branches.
template <bool SIG>
__global__ void __launch_bounds__(256, 3) pack_bind_tile_kernel(PackArgs a, BindArgs bnd) {
  // rows [0, head) of the 16 records, transposed, staged with one pad slot per 16 rows
  // (static shared memory for the 608-row unsigned prefix, dynamic for 3024 rows)
  extern __shared__ uint4 S_dyn[];
  __shared__ uint4 S_st[SIG ? 1 : BIND_HEAD + BIND_HEAD / 16];
  uint4* S = SIG ? S_dyn : S_st;
  constexpr uint32_t head = SIG ? BIND_HEAD_SIG : BIND_HEAD;
  const uint32_t j = a.g_lo + blockIdx.x, ch = blockIdx.y, blk = blockIdx.z;
  const uint32_t tid = threadIdx.x;
  const uint64_t row0 = ((uint64_t)blk * a.n_ch + ch) * a.d;  // global row of byte 0
  if (row0 + a.d <= a.row_begin || row0 >= a.row_begin + a.ell_local) return;  // outside the shard
  uint32_t valid = 0;
  uint64_t th[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t col = j * 16 + i;
    const uint64_t cell = (uint64_t)blk * a.m + col;
    th[i] = cell * a.n_ch + ch;
    if (col < a.m && cell < a.n_cells && th[i] >= a.theta0 && th[i] < a.theta0 + a.n_rec) valid |= 1u << i;
  }
  if (!valid) return;
  if (tid < head / 16) {
    const uint32_t b0 = tid * 16;
    uint32_t X[16][4];  // X[record][word]: bytes b0 .. b0 + 15 of record i
    const bool sig_chunk = SIG && b0 >= BIND_HEAD;  // whole chunk inside the signature rows
    if (b0 + 16 <= HCT_SPECTRUM || sig_chunk) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if ((valid >> i) & 1u)
          v = sig_chunk ? *reinterpret_cast<const uint4*>(bnd.sig + (th[i] - bnd.theta0) * HCT_SIG_STRIDE + b0)
                        : *reinterpret_cast<const uint4*>(bnd.spectrum + (th[i] - bnd.theta0) * bnd.spec_stride + b0);
        X[i][0] = v.x; X[i][1] = v.y; X[i][2] = v.z; X[i][3] = v.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        uint8_t by[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) by[k] = 0;
        if ((valid >> i) & 1u) {
          if (b0 + 16 <= HCT_SPECTRUM + 32) {  // one Philox block = 16 nonce bytes
            const uint2 key = make_uint2((uint32_t)bnd.seed_psd, (uint32_t)(bnd.seed_psd >> 32));
            const uint4 r = philox4x32_10(
                make_uint4((uint32_t)th[i], (uint32_t)(th[i] >> 32), (b0 - HCT_SPECTRUM) / 16, 0x48u), key);
            X[i][0] = r.x; X[i][1] = r.y; X[i][2] = r.z; X[i][3] = r.w;
            continue;
          }
          // the chunk at 592: kappa (4 B) || n_l || signature bytes 0..10 (or zeros)
          static_assert(HCT_SPECTRUM + 32 == BIND_HEAD - 16, "one straddling chunk");
#pragma unroll
          for (int k = 0; k < 4; ++k) by[k] = (uint8_t)(bnd.kappa >> (8 * k));
          by[4] = (uint8_t)bnd.n_l;
          if constexpr (SIG) {
            const uint8_t* sg = bnd.sig + (th[i] - bnd.theta0) * HCT_SIG_STRIDE;
#pragma unroll
            for (int k = 5; k < 16; ++k) by[k] = sg[b0 + k];
          }
        }
#pragma unroll
        for (int w = 0; w < 4; ++w)
          X[i][w] = by[4 * w] | (by[4 * w + 1] << 8) | (by[4 * w + 2] << 16) | ((uint32_t)by[4 * w + 3] << 24);
      }
    }
    // row b0 + 4w + k, cells 4v .. 4v + 3: byte k of X[4v .. 4v + 3][w]
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t y[4];
        transpose4x4_bytes(X[4 * v][w], X[4 * v + 1][w], X[4 * v + 2][w], X[4 * v + 3][w], y[0], y[1], y[2], y[3]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t rr = b0 + 4 * w + k;
          reinterpret_cast<uint32_t*>(&S[rr + rr / 16])[v] = y[k];
        }
      }
  }
  __syncthreads();
  // every row of the record bytes: consecutive threads, consecutive rows (16-byte chunks)
  for (uint32_t b = tid; b < a.d; b += blockDim.x) {
    const uint64_t row = row0 + b;
    if (row < a.row_begin || row >= a.row_begin + a.ell_local) continue;
    const uint64_t rl = row - a.row_begin;
    uint4* dst = reinterpret_cast<uint4*>(a.D + ((size_t)(rl >> 7) * a.G + j) * 2048 + (rl & 127u) * 16);
    uint4 v = b < head ? S[b + b / 16] : make_uint4(0u, 0u, 0u, 0u);
    if (valid != 0xFFFFu) {  // partial group: keep the other cells' bytes
      const uint4 o = *dst;
      uint8_t* vb = reinterpret_cast<uint8_t*>(&v);
      const uint8_t* ob = reinterpret_cast<const uint8_t*>(&o);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (!((valid >> i) & 1u)) vb[i] = ob[i];
    }
    *dst = v;
  }
}

int db_write_device(qpir_ctx* ctx, uint64_t theta0, uint64_t n_rec, const uint8_t* rec,
                    cudaStream_t st, const BindArgs* bind = nullptr);

int db_write_device(qpir_ctx* ctx, uint64_t theta0, uint64_t n_rec, const uint8_t* rec,
                    cudaStream_t st, const BindArgs* bind) {
  const Geometry& g = ctx->geo;
  if (n_rec == 0) return QPIR_OK;
  // column groups touched: whole range unless the chunk lies in one row block
  const uint64_t cell_lo = theta0 / g.n_ch, cell_hi = (theta0 + n_rec - 1) / g.n_ch;
  uint64_t j_lo = 0, j_hi = g.G - 1;
  if (cell_lo / g.m == cell_hi / g.m) {
    j_lo = (cell_lo % g.m) / 16;
    j_hi = (cell_hi % g.m) / 16;
  }
  PackArgs a;
  a.rec = rec;
  a.D = ctx->D;
  a.theta0 = theta0;
  a.n_rec = n_rec;
  a.row_begin = g.row_begin;
  a.ell_local = (uint32_t)g.ell_local;
  a.L = (uint32_t)g.L;
  a.n_ch = (uint32_t)g.n_ch;
  a.d = (uint32_t)g.d;
  a.m = (uint32_t)g.m;
  a.n_cells = g.n_cells;
  a.g_lo = (uint32_t)j_lo;
  a.G = (uint32_t)g.G;
  const uint32_t rb = (uint32_t)((g.ell_local + 127) / 128);
  for (uint32_t y0 = 0; y0 < rb; y0 += 65535) {
    // grid.y is limited to 65535 row blocks per launch
    PackArgs b = a;
    const uint32_t ny = std::min<uint32_t>(65535, rb - y0);
    b.D = ctx->D + (size_t)y0 * g.G * 2048;  // y0 panels of 128 rows
    b.row_begin = g.row_begin + (uint64_t)y0 * 128;
    b.ell_local = (uint32_t)std::min<uint64_t>(g.ell_local - (uint64_t)y0 * 128, (uint64_t)ny * 128);
    dim3 grid((uint32_t)(j_hi - j_lo + 1), ny);
    const bool tile = bind && g.d % 16 == 0 && g.d >= (bind->sig ? BIND_HEAD_SIG : BIND_HEAD) &&
                      bind->spec_stride % 16 == 0 &&
                      (reinterpret_cast<uintptr_t>(bind->spectrum) & 15u) == 0 &&
                      g.n_ch <= 65535 && (g.n_cells + g.m - 1) / g.m <= 65535;
    if (tile) {
      // register-transposed bind (whole shard in one launch: grid = column groups x
      // channels x row blocks; threads = 16-row chunks of a record)
      if (y0 == 0) {
        const uint32_t nblk = (uint32_t)((g.n_cells + g.m - 1) / g.m);
        dim3 tg((uint32_t)(j_hi - j_lo + 1), (uint32_t)g.n_ch, nblk);
        const size_t sm = bind->sig ? (size_t)(BIND_HEAD_SIG + BIND_HEAD_SIG / 16) * 16 : 0;
        auto kern = bind->sig ? pack_bind_tile_kernel<true> : pack_bind_tile_kernel<false>;
        // the attribute call costs host time on every launch (measured: 0.29 -> 0.46 ms
        // per unsigned C2 bind): set it once, and only for the dynamic-smem form
        if (bind->sig && !ctx->bind_sig_attr) {  // per context: attributes are per device
          CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
          ctx->bind_sig_attr = true;
        }
        kern<<<tg, 256, sm, st>>>(a, *bind);
        LAUNCH_CHECK(ctx);
      }
      continue;
    } else if (bind) {
      pack_bind_kernel<<<grid, 128, 0, st>>>(b, *bind);
    } else {
      pack_records_kernel<<<grid, 128, 0, st>>>(b);
    }
    LAUNCH_CHECK(ctx);
  }
  ctx->d_written.store(true);
  return QPIR_OK;
}

// early: qu was not written by the kernel preceding this launch on `st` (the
// library staged it from host memory with a copy, or the caller set
// QPIR_FLAG_STABLE_INPUTS), so the scan may run before griddepcontrol.wait.
template <int U, int UNR>
int launch_gemv(qpir_ctx* ctx, const uint32_t* qu, uint32_t* ans, cudaStream_t st, bool early) {
  const Geometry& g = ctx->geo;
  const uint32_t rows_per_cta = GEMV_THREADS * U;
  const uint32_t rb = (uint32_t)((g.ell_local + rows_per_cta - 1) / rows_per_cta);
  uint32_t S = ctx->gemv_split;
  if (S == 0) {
    // Many short CTAs beat one wave of long ones (measured on B200, DESIGN 6):
    // about 256 column groups (1 MB of D at U = 2) per CTA, and at least ~8
    // waves of ~6 resident CTAs per SM so the tail stays small; at least 16
    // groups per split.
    const uint32_t by_work = (uint32_t)((g.G + 255) / 256);
    const uint32_t by_waves = (uint32_t)((8u * 6u * ctx->num_sms + rb - 1) / rb);
    S = std::max(by_work, by_waves);
    S = std::min<uint32_t>(S, (uint32_t)std::max<uint64_t>(1, g.G / 16));
    // prefer a split count that divides the K range into equal pieces
    const uint32_t units = (uint32_t)(g.G / UNR);
    for (uint32_t c = S; c <= 2 * S && c <= units; ++c)
      if (units % c == 0) {
        S = c;
        break;
      }
  }
  S = std::max<uint32_t>(1, std::min<uint32_t>(S, (uint32_t)(g.G / UNR)));
  S = std::min<uint32_t>(S, 65535u);  // grid.y limit
  uint32_t gps = (uint32_t)round_up((g.G + S - 1) / S, UNR);
  S = (uint32_t)((g.G + gps - 1) / gps);
  uint32_t chunk = (uint32_t)std::max(UNR, ctx->gemv_chunk / UNR * UNR);
  chunk = std::min(chunk, gps);
  Arena& ar = arena_for(ctx, st);
  if (S > 1) {
    int rc = ensure(ctx, (void**)&ar.partial, &ar.partial_bytes, (uint64_t)S * g.L * 4);
    if (rc) return rc;
    if ((uint64_t)rb * 4 > ar.tickets_bytes) {
      rc = ensure(ctx, (void**)&ar.tickets, &ar.tickets_bytes, (uint64_t)rb * 4);
      if (rc) return rc;
      CUDA_TRY(ctx, cudaMemsetAsync(ar.tickets, 0, ar.tickets_bytes, st));
    }
  }
  GemvArgs a;
  a.D = ctx->D;
  a.qu = qu;
  a.ans = ans;
  a.partial = ar.partial;
  a.tickets = ar.tickets;
  a.ell_local = (uint32_t)g.ell_local;
  a.L = (uint32_t)g.L;
  a.m = (uint32_t)g.m;
  a.G = (uint32_t)g.G;
  a.gps = gps;
  a.chunk = chunk;
  a.split_major = (ctx->gemv_order == 1 && rb <= 65535) ? 1u : 0u;
  a.pf256 = ctx->gemv_pf256 ? 1u : 0u;
  a.l2pf = ctx->gemv_l2pf ? 1u : 0u;
  const size_t smem = (size_t)chunk * 64;
  auto kern = early ? qpir_gemv_u8_u32_kernel<U, UNR, true> : qpir_gemv_u8_u32_kernel<U, UNR, false>;
  if (smem > 48 * 1024)
    CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const dim3 grid = a.split_major ? dim3(S, rb) : dim3(rb, S);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(GEMV_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  // The GEMV reads D before griddepcontrol.wait: right after a device-side
  // db_write (pack_records_kernel writes D) it is launched without PDL.
  const bool after_write = ctx->d_written.exchange(false);
  attr[0].val.programmaticStreamSerializationAllowed = (ctx->gemv_pdl && !after_write) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, kern, a));
  LAUNCH_CHECK(ctx);
  return QPIR_OK;
}

int gemv(qpir_ctx* ctx, const uint32_t* qu, uint32_t* ans, cudaStream_t st, bool early) {
  const bool u8 = ctx->gemv_unroll == 8;
  switch (ctx->gemv_u) {
    case 1: return u8 ? launch_gemv<1, 8>(ctx, qu, ans, st, early) : launch_gemv<1, 4>(ctx, qu, ans, st, early);
    case 4: return u8 ? launch_gemv<4, 8>(ctx, qu, ans, st, early) : launch_gemv<4, 4>(ctx, qu, ans, st, early);
    default: return u8 ? launch_gemv<2, 8>(ctx, qu, ans, st, early) : launch_gemv<2, 4>(ctx, qu, ans, st, early);
  }
}

template <int MODE>
int launch_mma(qpir_ctx* ctx, uint32_t BN, const uint8_t* Bl, uint32_t Npad, uint32_t* out,
               uint32_t n_out, uint32_t out_ld, uint64_t out_elems, cudaStream_t st,
               uint32_t p = 0, unsigned long long* out64 = nullptr, bool prezeroed = false,
               const ModpExceptions& exc = ModpExceptions(), const MmaJob* conv = nullptr) {
  const Geometry& g = ctx->geo;
  MmaJob j;
  j.A = ctx->D;
  j.L = (uint32_t)g.L;
  j.G = (uint32_t)g.G;
  j.rows = (uint32_t)g.ell_local;
  j.B = Bl;
  j.Npad = Npad;
  j.BN = BN;
  j.out = out;
  j.n_out = n_out;
  j.out_ld = out_ld;
  j.out_elems = out_elems;
  j.p = p;
  j.out64 = out64;
  j.num_sms = ctx->num_sms;
  j.forced_split = ctx->mma_split;
  j.mt = ctx->mma_mt;
  j.gpb = ctx->mma_gpb;
  j.out_prezeroed = prezeroed;
  j.exc = exc;
  j.l2hint = (uint32_t)ctx->mma_l2hint;
  if (conv) {  // fused limb split (OUT_MODP2): the converter fields of the caller's job
    j.conv = true;
    j.Q = conv->Q;
    j.qB = conv->qB;
    j.qm = conv->qm;
    j.pM = conv->pM;
    j.kb_done = conv->kb_done;
    j.epoch = conv->epoch;
    j.conv_ctr = conv->conv_ctr;
    j.conv_base = conv->conv_base;
  }
  if (ctx->mma_ls > 0) {
    constexpr uint32_t kKprogCap = 4096;
    Arena& ar = arena_for(ctx, st);
    if (!ar.kprog) {
      uint64_t have = 0;
      int rc = ensure(ctx, (void**)&ar.kprog, &have, kKprogCap * 4);
      if (rc) return rc;
    }
    j.kprog = ar.kprog;
    j.kprog_cap = kKprogCap;
    j.ls_chunk = (uint32_t)ctx->mma_ls;
    j.ls_drift = (uint32_t)std::max(1, ctx->mma_drift);
  }
  const cudaError_t e = mma_launch<MODE>(j, st, &ctx->launches);
  if (e != cudaSuccess)
    return fail(ctx, e == cudaErrorMemoryAllocation ? QPIR_E_OOM : QPIR_E_CUDA,
                "tcgen05 GEMM launch: %s", cudaGetErrorString(e));
  return QPIR_OK;
}

}  // namespace

extern "C" {

int qpir_setup(const qpir_params* params, const uint8_t* records, uint64_t records_len,
               void* stream, qpir_ctx** out) {
  NvtxRange nvtx_("qpir_setup");
  g_setup_error.clear();
  if (!out) return fail(nullptr, QPIR_E_PARAM, "out: NULL");
  *out = nullptr;
  Geometry g;
  int rc = validate(params, &g);
  if (rc) return rc;
  const uint64_t n_rec = g.n_cells * g.n_ch;
  if (records && records_len != n_rec * g.d)
    return fail(nullptr, QPIR_E_DIMENSION, "records_len: %llu != %llu",
                (unsigned long long)records_len, (unsigned long long)(n_rec * g.d));
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(nullptr, QPIR_E_CUDA, "device: no CUDA device available");
  }
  if (params->device >= ndev)
    return fail(nullptr, QPIR_E_PARAM, "device: %d >= device count %d", params->device, ndev);
  DeviceGuard dg(params->device);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, params->device) != cudaSuccess)
    return fail(nullptr, QPIR_E_CUDA, "cudaGetDeviceProperties failed");
  if (prop.major != 10)
    return fail(nullptr, QPIR_E_CUDA, "device: compute capability %d.%d, need 10.x (sm_100a)",
                prop.major, prop.minor);
  qpir_ctx* ctx = new qpir_ctx();
  ctx->geo = g;
  ctx->device = params->device;
  ctx->num_sms = prop.multiProcessorCount;
  ctx->gemv_u = env_int("QPIR_GEMV_U", 2);
  ctx->gemv_split = env_int("QPIR_GEMV_SPLIT", 0);
  ctx->gemv_chunk = env_int("QPIR_GEMV_CHUNK", 512);
  ctx->gemv_unroll = env_int("QPIR_GEMV_UNROLL", 4);
  ctx->gemv_order = env_int("QPIR_GEMV_ORDER", 0);
  ctx->gemv_pdl = env_int("QPIR_GEMV_PDL", 1);
  ctx->gemv_pf256 = env_int("QPIR_GEMV_PF256", 0);
  ctx->gemv_l2pf = env_int("QPIR_GEMV_L2PF", 0);
  ctx->flags = params->flags;
  ctx->mma_mt = env_int("QPIR_MMA_MT", 2);
  ctx->mma_l2hint = env_int("QPIR_MMA_L2HINT", 0);
  ctx->mma_split = env_int("QPIR_MMA_SPLIT", 0);
  ctx->mma_gpb = env_int("QPIR_MMA_GPB", 8);
  ctx->modp3 = env_int("QPIR_MODP3", 1);
  ctx->modp2 = env_int("QPIR_MODP2", 1);
  ctx->ftr_fuse = env_int("QPIR_FTR_FUSE", 1);
  ctx->h2d_stream = env_int("QPIR_H2D_STREAM", 1);
  ctx->mma_ls = env_int("QPIR_MMA_LOCKSTEP", 16);
  ctx->mma_drift = env_int("QPIR_MMA_DRIFT", 1);
  if (env_int("QPIR_LIMB_BUDGET_MB", 0) > 0)
    ctx->limb_budget = (uint64_t)env_int("QPIR_LIMB_BUDGET_MB", 0) << 20;
  cudaStream_t st = (cudaStream_t)stream;
  auto bail = [&](int code) {
    g_setup_error = ctx->err;
    qpir_destroy(ctx);
    return code;
  };
  const size_t dbytes = (size_t)g.m_pad * g.L;
  if (cudaMalloc(&ctx->D, dbytes) != cudaSuccess) {
    cudaGetLastError();
    fail(ctx, QPIR_E_OOM, "D: cudaMalloc(%zu) failed", dbytes);
    return bail(QPIR_E_OOM);
  }
  if (cudaMemsetAsync(ctx->D, 0, dbytes, st) != cudaSuccess) {
    fail(ctx, QPIR_E_CUDA, "memset failed");
    return bail(QPIR_E_CUDA);
  }
  if (records) {
    rc = qpir_db_write(ctx, 0, n_rec, records, records_len, stream);
    if (rc) return bail(rc);
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) {
    fail(ctx, QPIR_E_CUDA, "setup: %s", cudaGetErrorString(cudaGetLastError()));
    return bail(QPIR_E_CUDA);
  }
  *out = ctx;
  return QPIR_OK;
}

int qpir_db_write(qpir_ctx* ctx, uint64_t theta_begin, uint64_t n_records,
                  const uint8_t* records, uint64_t records_len, void* stream) {
  NvtxRange nvtx_("qpir_db_write");
  if (!ctx) return fail(nullptr, QPIR_E_STATE, "ctx: NULL");
  const Geometry& g = ctx->geo;
  const uint64_t n_all = g.n_cells * g.n_ch;
  if (theta_begin > n_all || n_records > n_all - theta_begin)
    return fail(ctx, QPIR_E_DIMENSION, "theta range: [%llu, +%llu) exceeds %llu records",
                (unsigned long long)theta_begin, (unsigned long long)n_records,
                (unsigned long long)n_all);
  if (records_len != n_records * g.d)
    return fail(ctx, QPIR_E_DIMENSION, "records_len: %llu != %llu",
                (unsigned long long)records_len, (unsigned long long)(n_records * g.d));
  if (n_records == 0) return QPIR_OK;
  if (!records) return fail(ctx, QPIR_E_PARAM, "records: NULL");
  DeviceGuard dg(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int w = where(records, ctx->device);
  if (w < 0) return fail(ctx, QPIR_E_PARAM, "records: device memory of another device");
  if (w == 1) return db_write_device(ctx, theta_begin, n_records, records, st);
  // host records: stream through a device staging buffer in chunks
  const uint64_t chunk_rec = std::max<uint64_t>(1, (64ull << 20) / g.d);
  int rc = ensure(ctx, (void**)&ctx->rec_stage, &ctx->rec_stage_bytes,
                  std::min(n_records, chunk_rec) * g.d);
  if (rc) return rc;
  for (uint64_t t = 0; t < n_records; t += chunk_rec) {
    const uint64_t n = std::min(chunk_rec, n_records - t);
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->rec_stage, records + t * g.d, n * g.d,
                                  cudaMemcpyHostToDevice, st));
    rc = db_write_device(ctx, theta_begin + t, n, ctx->rec_stage, st);
    if (rc) return rc;
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return QPIR_OK;
}

int qpir_puzzle_bind_hct(qpir_ctx* ctx, uint64_t theta_begin, uint64_t n_records,
                         const uint8_t* spectrum, uint64_t spec_stride, uint64_t spectrum_len,
                         uint64_t seed_psd, uint32_t kappa, uint8_t n_l, const uint8_t* mldsa_seed,
                         uint8_t* mldsa_pk, void* stream) {
  NvtxRange nvtx_("qpir_puzzle_bind_hct");
  if (!ctx) return fail(nullptr, QPIR_E_STATE, "ctx: NULL");
  const Geometry& g = ctx->geo;
  const uint64_t n_all = g.n_cells * g.n_ch;
  if (g.d < HCT_SPECTRUM + HCT_PUZZLE)
    return fail(ctx, QPIR_E_DIMENSION, "rec_bytes: %llu < 597 (560 B spectrum + 37 B puzzle)",
                (unsigned long long)g.d);
  if (mldsa_seed && g.d < HCT_SIG_END)
    return fail(ctx, QPIR_E_DIMENSION, "rec_bytes: %llu < 3017 (spectrum + puzzle + ML-DSA signature)",
                (unsigned long long)g.d);
  if (theta_begin > n_all || n_records > n_all - theta_begin)
    return fail(ctx, QPIR_E_DIMENSION, "theta range: [%llu, +%llu) exceeds %llu records",
                (unsigned long long)theta_begin, (unsigned long long)n_records,
                (unsigned long long)n_all);
  if (spec_stride < HCT_SPECTRUM)
    return fail(ctx, QPIR_E_DIMENSION, "spec_stride: %llu < 560", (unsigned long long)spec_stride);
  if (spectrum_len != n_records * spec_stride)
    return fail(ctx, QPIR_E_DIMENSION, "spectrum_len: %llu != %llu",
                (unsigned long long)spectrum_len, (unsigned long long)(n_records * spec_stride));
  if (n_records == 0) return QPIR_OK;
  if (!spectrum) return fail(ctx, QPIR_E_PARAM, "spectrum: NULL");
  DeviceGuard dg(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int w = where(spectrum, ctx->device);
  if (w < 0) return fail(ctx, QPIR_E_PARAM, "spectrum: device memory of another device");
  // records are generated inside the pack kernel, straight into the D panels;
  // a host spectrum is staged in chunks of <= 64 MB; signatures in chunks of 64K (198 MB of staging rows)
  uint64_t chunk = w ? n_records : std::max<uint64_t>(1, (64ull << 20) / spec_stride);
  int rc = QPIR_OK;
  mldsa::MldsaKey* key = nullptr;
  uint32_t* ticket = nullptr;  // the signer's record counter (after xi in mldsa_buf)
  if (mldsa_seed) {
    chunk = std::min<uint64_t>(chunk, 65536);
    rc = ensure(ctx, (void**)&ctx->mldsa_buf, &ctx->mldsa_buf_bytes, sizeof(mldsa::MldsaKey) + 64);
    if (rc) return rc;
    key = reinterpret_cast<mldsa::MldsaKey*>(ctx->mldsa_buf);
    uint8_t* xi_dev = ctx->mldsa_buf + sizeof(mldsa::MldsaKey);
    ticket = reinterpret_cast<uint32_t*>(xi_dev + 32);
    CUDA_TRY(ctx, cudaMemcpyAsync(xi_dev, mldsa_seed, 32, cudaMemcpyDefault, st));
    CUDA_TRY(ctx, mldsa::keygen(xi_dev, key, st));
    ctx->launches++;
    if (mldsa_pk) CUDA_TRY(ctx, cudaMemcpyAsync(mldsa_pk, key->pk, mldsa::PK_BYTES, cudaMemcpyDefault, st));
    rc = ensure(ctx, (void**)&ctx->sig_stage, &ctx->sig_stage_bytes,
                std::min(n_records, chunk) * HCT_SIG_STRIDE);
    if (rc) return rc;
    // bytes outside [597, 3017) of a staging row are never written: zero once per call
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->sig_stage, 0, std::min(n_records, chunk) * HCT_SIG_STRIDE, st));
  }
  if (w == 0) {
    rc = ensure(ctx, (void**)&ctx->spec_stage, &ctx->spec_stage_bytes,
                std::min(n_records, chunk) * spec_stride);
    if (rc) return rc;
  }
  for (uint64_t t = 0; t < n_records; t += chunk) {
    const uint64_t n = std::min(chunk, n_records - t);
    const uint8_t* sp = spectrum + t * spec_stride;
    if (w == 0) {
      CUDA_TRY(ctx, cudaMemcpyAsync(ctx->spec_stage, sp, n * spec_stride, cudaMemcpyHostToDevice, st));
      sp = ctx->spec_stage;
    }
    BindArgs b;
    b.spectrum = sp;
    b.spec_stride = spec_stride;
    b.theta0 = theta_begin + t;
    b.n = n;
    b.seed_psd = seed_psd;
    b.kappa = kappa;
    b.n_l = n_l;
    b.d = (uint32_t)g.d;
    b.out = nullptr;
    b.out_stride = 0;
    if (key) {
      CUDA_TRY(ctx, mldsa::sign_records(key, theta_begin + t, n, seed_psd, kappa, n_l, ctx->sig_stage,
                                            ticket, st));
      ctx->launches++;
      b.sig = ctx->sig_stage;
    }
    rc = db_write_device(ctx, theta_begin + t, n, nullptr, st, &b);
    if (rc) return rc;
  }
  if (mldsa_pk && where(mldsa_pk, ctx->device) == 0) CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (w == 0) CUDA_TRY(ctx, cudaStreamSynchronize(st));  // the staging buffer is reused per call
  return QPIR_OK;
}

int qpir_geometry(const qpir_ctx* ctx, uint64_t* ell, uint64_t* m, uint64_t* ell_local,
                  uint64_t* row_begin) {
  if (!ctx) return QPIR_E_STATE;
  if (ell) *ell = ctx->geo.ell;
  if (m) *m = ctx->geo.m;
  if (ell_local) *ell_local = ctx->geo.ell_local;
  if (row_begin) *row_begin = ctx->geo.row_begin;
  return QPIR_OK;
}

int qpir_answer(qpir_ctx* ctx, const uint32_t* qu, uint64_t len_qu, uint32_t* ans_local,
                uint64_t len_ans, void* stream) {
  NvtxRange nvtx_("qpir_answer");
  if (!ctx) return fail(nullptr, QPIR_E_STATE, "ctx: NULL");
  const Geometry& g = ctx->geo;
  if (!qu || !ans_local) return fail(ctx, QPIR_E_PARAM, "qu/ans_local: NULL");
  if (len_qu != g.m)
    return fail(ctx, QPIR_E_DIMENSION, "m: %llu != %llu", (unsigned long long)len_qu,
                (unsigned long long)g.m);
  if (len_ans != g.ell_local)
    return fail(ctx, QPIR_E_DIMENSION, "ell_local: %llu != %llu", (unsigned long long)len_ans,
                (unsigned long long)g.ell_local);
  DeviceGuard dg(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int wq = where(qu, ctx->device), wa = where(ans_local, ctx->device);
  if (wq < 0 || wa < 0) return fail(ctx, QPIR_E_PARAM, "qu/ans_local: memory of another device");
  if ((reinterpret_cast<uintptr_t>(qu) & 3u) || (reinterpret_cast<uintptr_t>(ans_local) & 3u))
    return fail(ctx, QPIR_E_PARAM, "qu/ans_local: not 4-byte aligned");
  Arena& ar = arena_for(ctx, st);
  int rc = QPIR_OK;
  const uint32_t* qd = qu;
  int slot = -1;
  if (wq == 0) {
    const void* dv = nullptr;
    rc = stage_host(ctx, ar, ar.in_small, qu, g.m * 4, g.m_pad * 4, st, &dv, &slot);
    if (rc) return rc;
    qd = static_cast<const uint32_t*>(dv);
  } else if (!aligned16(qu)) {
    rc = ensure(ctx, (void**)&ar.qu_dev, &ar.qu_bytes, g.m_pad * 4);
    if (rc) return rc;
    CUDA_TRY(ctx, cudaMemcpyAsync(ar.qu_dev, qu, g.m * 4, cudaMemcpyDeviceToDevice, st));
    qd = ar.qu_dev;
  }
  uint32_t* ad = ans_local;
  if (!wa) {
    rc = ensure(ctx, (void**)&ar.ans_dev, &ar.ans_bytes, g.L * 4);
    if (rc) return rc;
    ad = ar.ans_dev;
  }
  // qu staged by the library (host copy / realignment copy) cannot be the
  // previous kernel's output; a caller's device buffer only with the flag
  rc = gemv(ctx, qd, ad, st, qd != qu || (ctx->flags & QPIR_FLAG_STABLE_INPUTS));
  if (rc) return rc;
  if (slot >= 0) CUDA_TRY(ctx, cudaEventRecord(ar.in_small.done[slot], st));
  if (!wa) {
    CUDA_TRY(ctx, cudaMemcpyAsync(ans_local, ad, g.ell_local * 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
  }
  return QPIR_OK;
}

static int answer_batch_impl(qpir_ctx* ctx, const uint32_t* Q, uint64_t B, uint64_t len_Q,
                             uint32_t* ans_local, uint64_t len_ans, void* stream, uint32_t p) {
  NvtxRange nvtx_(p ? "qpir_answer_batch_modp" : "qpir_answer_batch");
  if (!ctx) return fail(nullptr, QPIR_E_STATE, "ctx: NULL");
  const Geometry& g = ctx->geo;
  if (B == 0 || B > 4096) return fail(ctx, QPIR_E_PARAM, "B: %llu not in [1, 4096]",
                                      (unsigned long long)B);
  if (!Q || !ans_local) return fail(ctx, QPIR_E_PARAM, "Q/ans_local: NULL");
  if (len_Q != B * g.m)
    return fail(ctx, QPIR_E_DIMENSION, "len_Q: %llu != B*m %llu", (unsigned long long)len_Q,
                (unsigned long long)(B * g.m));
  if (len_ans != B * g.ell_local)
    return fail(ctx, QPIR_E_DIMENSION, "len_ans: %llu != B*ell_local %llu",
                (unsigned long long)len_ans, (unsigned long long)(B * g.ell_local));
  DeviceGuard dg(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int wq = where(Q, ctx->device), wa = where(ans_local, ctx->device);
  if (wq < 0 || wa < 0) return fail(ctx, QPIR_E_PARAM, "Q/ans_local: memory of another device");
  if ((reinterpret_cast<uintptr_t>(Q) & 3u) || (reinterpret_cast<uintptr_t>(ans_local) & 3u))
    return fail(ctx, QPIR_E_PARAM, "Q/ans_local: not 4-byte aligned");
  // F_p: entries reduced mod p, then 2 limbs per query for p <= 65537 (the
  // residue 65536 of p = 65537 as a listed exception), 3 for p <= 2^24
  const bool two = p != 0 && p <= 65537u && ctx->modp2;
  const bool three = !two && p != 0 && p <= (1u << 24) && ctx->modp3;
  const uint32_t LPQ = two ? 2u : three ? 3u : 4u;
  // Q' (LPQ limb columns per query) is materialised per chunk of queries so
  // that it stays within ~2 GiB whatever B and m are.
  const uint64_t budget = ctx->limb_budget;
  uint64_t Bc = B;
  if (round_up(LPQ * Bc, 256) * g.m_pad > budget)
    Bc = std::max<uint64_t>(64, (budget / g.m_pad) / LPQ / 64 * 64);
  const uint64_t ncols = LPQ * std::min<uint64_t>(Bc, B);
  const uint32_t BN = three ? mma_pick_bn3(ncols) : mma_pick_bn(ncols);
  const uint32_t Npad = (uint32_t)round_up(ncols, BN);
  Arena& ar = arena_for(ctx, st);
  int rc = ensure(ctx, (void**)&ar.limbs, &ar.limbs_bytes, (uint64_t)Npad * g.m_pad);
  if (rc) return rc;
  const uint32_t* Qd = Q;
  int slot = -1;
  if (wq == 0) {
    const void* dv = nullptr;
    rc = stage_host(ctx, ar, ar.in_big, Q, len_Q * 4, len_Q * 4, st, &dv, &slot);
    if (rc) return rc;
    Qd = static_cast<const uint32_t*>(dv);
  }
  uint32_t* out = ans_local;
  if (wa == 0) {
    rc = ensure(ctx, (void**)&ar.big_out, &ar.big_out_bytes, len_ans * 4);
    if (rc) return rc;
    out = ar.big_out;
  }
  if (p != 0) {
    rc = ensure(ctx, (void**)&ar.acc64, &ar.acc64_bytes, (uint64_t)std::min(Bc, B) * g.ell_local * 8);
    if (rc) return rc;
  }
  cudaStreamCaptureStatus cap_status = cudaStreamCaptureStatusNone;
  CUDA_TRY(ctx, cudaStreamIsCapturing(st, &cap_status));
  const bool capturing = cap_status != cudaStreamCaptureStatusNone;
  // exception lists: Poisson(m / p) entries per uniform query; cap ~ 4x the
  // mean + 64, an overflowed (adversarial) query falls back to a rescan
  const bool exc = two && p == 65537u;
  const uint32_t cap = (uint32_t)std::min<uint64_t>(g.m, 64 + 4 * ((g.m + 65536) / 65537));
  uint32_t *exc_cnt = nullptr, *exc_list = nullptr;
  if (exc) {
    const uint64_t nb = std::min(Bc, B);
    rc = ensure(ctx, (void**)&ar.exc, &ar.exc_bytes, nb * 4 * (1 + (uint64_t)cap));
    if (rc) return rc;
    exc_cnt = ar.exc;
    exc_list = ar.exc + nb;
  }
  for (uint64_t b0 = 0; b0 < B && rc == QPIR_OK; b0 += Bc) {
    const uint32_t bc = (uint32_t)std::min<uint64_t>(Bc, B - b0);
    const uint32_t* Qc = Qd + b0 * g.m;
    uint32_t* oc = out + b0 * g.ell_local;
    const uint64_t oe = (uint64_t)bc * g.ell_local;
    // 2 limbs: the split runs inside the GEMM (converter warps, mma.cuh) unless
    // QPIR_FTR_FUSE=0, the K-block is not 128 cells, or the stream is being
    // captured into a CUDA graph: the fused form's converter work counter and
    // K-block epoch advance on the host per launch, so a replayed capture would
    // wait forever on stale flags -- captures take the split-kernel form
    const bool fuse = two && ctx->ftr_fuse && ctx->mma_gpb != 4 && !capturing;
    const uint64_t pM = p >= 2 ? ~0ull / p + 1 : 0;  // fastmod_u32 constant
    if (exc) CUDA_TRY(ctx, cudaMemsetAsync(exc_cnt, 0, (uint64_t)bc * 4, st));
    MmaJob cj;
    if (fuse) {
      const uint64_t flags = (g.G / 8) * 4;
      if (ar.kb_done_bytes < flags) {
        rc = ensure(ctx, (void**)&ar.kb_done, &ar.kb_done_bytes, flags);
        if (rc) return rc;
        CUDA_TRY(ctx, cudaMemsetAsync(ar.kb_done, 0, flags, st));
        ar.epoch = 0;
      }
      if (!ar.conv_ctr) {
        uint64_t have = 0;
        rc = ensure(ctx, (void**)&ar.conv_ctr, &have, 8);
        if (rc) return rc;
        CUDA_TRY(ctx, cudaMemsetAsync(ar.conv_ctr, 0, 8, st));
        ar.conv_base = 0;
      }
      if (++ar.epoch == 0) {  // 2^32 launches: restart the flags
        CUDA_TRY(ctx, cudaMemsetAsync(ar.kb_done, 0, ar.kb_done_bytes, st));
        ar.epoch = 1;
      }
      cj.Q = Qc;
      cj.qB = bc;
      cj.qm = (uint32_t)g.m;
      cj.pM = pM;
      cj.kb_done = ar.kb_done;
      cj.epoch = ar.epoch;
      cj.conv_ctr = ar.conv_ctr;
      cj.conv_base = &ar.conv_base;
    } else {
      const uint32_t nq = Npad / LPQ;  // padded query slots
      dim3 grid((uint32_t)((g.G + 127) / 128), nq);
      if (two)
        limb_split_kernel<2><<<grid, 128, 0, st>>>(Qc, ar.limbs, bc, (uint32_t)g.m,
                                                   (uint32_t)g.G, Npad, BN, p, pM,
                                                   exc_cnt, exc_list, cap);
      else if (three)
        limb_split_kernel<3><<<grid, 128, 0, st>>>(Qc, ar.limbs, bc, (uint32_t)g.m,
                                                   (uint32_t)g.G, Npad, BN, p, pM,
                                                   nullptr, nullptr, 0u);
      else
        limb_split_kernel<4><<<grid, 128, 0, st>>>(Qc, ar.limbs, bc, (uint32_t)g.m,
                                                   (uint32_t)g.G, Npad, BN, 0u, 0ull,
                                                   nullptr, nullptr, 0u);
      LAUNCH_CHECK(ctx);
    }
    if (p == 0)
      rc = launch_mma<OUT_QUERY_MAJOR>(ctx, BN, ar.limbs, Npad, oc, bc, (uint32_t)g.ell_local, oe,
                                       st);
    else if (two) {
      ModpExceptions ex;
      if (exc) {
        ex.D = ctx->D;
        ex.G = (uint32_t)g.G;
        ex.Q = Qc;
        ex.m = (uint32_t)g.m;
        ex.cnt = exc_cnt;
        ex.list = exc_list;
        ex.cap = cap;
      }
      rc = launch_mma<OUT_MODP2>(ctx, BN, ar.limbs, Npad, oc, bc, (uint32_t)g.ell_local, oe, st,
                                 p, ar.acc64, false, ex, fuse ? &cj : nullptr);
    }
    else if (three)
      rc = launch_mma<OUT_MODP3>(ctx, BN, ar.limbs, Npad, oc, bc, (uint32_t)g.ell_local, oe, st,
                                 p, ar.acc64);
    else
      rc = launch_mma<OUT_MODP>(ctx, BN, ar.limbs, Npad, oc, bc, (uint32_t)g.ell_local, oe, st, p,
                                ar.acc64);
  }
  if (rc) return rc;
  if (slot >= 0) CUDA_TRY(ctx, cudaEventRecord(ar.in_big.done[slot], st));
  if (wa == 0) {
    CUDA_TRY(ctx, cudaMemcpyAsync(ans_local, out, len_ans * 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
  }
  return QPIR_OK;
}

int qpir_answer_batch(qpir_ctx* ctx, const uint32_t* Q, uint64_t B, uint64_t len_Q,
                      uint32_t* ans_local, uint64_t len_ans, void* stream) {
  return answer_batch_impl(ctx, Q, B, len_Q, ans_local, len_ans, stream, 0);
}

int qpir_answer_batch_modp(qpir_ctx* ctx, const uint32_t* Q, uint64_t B, uint64_t len_Q,
                           uint32_t p, uint32_t* ans_local, uint64_t len_ans, void* stream) {
  if (!ctx) return fail(nullptr, QPIR_E_STATE, "ctx: NULL");
  if (p < 2) return fail(ctx, QPIR_E_PARAM, "p: %u < 2", p);
  return answer_batch_impl(ctx, Q, B, len_Q, ans_local, len_ans, stream, p);
}

int qpir_hint(qpir_ctx* ctx, uint32_t* H_local, uint64_t len_H, void* stream) {
  NvtxRange nvtx_("qpir_hint");
  if (!ctx) return fail(nullptr, QPIR_E_STATE, "ctx: NULL");
  const Geometry& g = ctx->geo;
  if (!H_local) return fail(ctx, QPIR_E_PARAM, "H_local: NULL");
  if (len_H != g.ell_local * g.lwe_n)
    return fail(ctx, QPIR_E_DIMENSION, "len_H: %llu != ell_local*n %llu",
                (unsigned long long)len_H, (unsigned long long)(g.ell_local * g.lwe_n));
  DeviceGuard dg(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int wh = where(H_local, ctx->device);
  if (wh < 0) return fail(ctx, QPIR_E_PARAM, "H_local: memory of another device");
  if (reinterpret_cast<uintptr_t>(H_local) & 3u)
    return fail(ctx, QPIR_E_PARAM, "H_local: not 4-byte aligned");
  // A' (4 limb columns per hint column) is materialised per chunk of hint
  // columns so that it stays within ~2 GiB whatever n and m are.
  const uint64_t budget = ctx->limb_budget;
  uint64_t nc = g.lwe_n;
  if (round_up(4ull * nc, 256) * g.m_pad > budget)
    nc = std::max<uint64_t>(64, (budget / g.m_pad) / 4 / 64 * 64);
  const uint64_t ncols = 4ull * std::min<uint64_t>(nc, g.lwe_n);
  const uint32_t BN = mma_pick_bn(ncols);
  const uint32_t Npad = (uint32_t)round_up(ncols, BN);
  Arena& ar = arena_for(ctx, st);
  int rc = ensure(ctx, (void**)&ar.limbs, &ar.limbs_bytes, (uint64_t)Npad * g.m_pad);
  if (rc) return rc;
  uint32_t* out = H_local;
  if (wh == 0 || !aligned16(H_local)) {
    rc = ensure(ctx, (void**)&ar.big_out, &ar.big_out_bytes, len_H * 4);
    if (rc) return rc;
    out = ar.big_out;
  }
  const bool chunked = nc < g.lwe_n;
  if (chunked) CUDA_TRY(ctx, cudaMemsetAsync(out, 0, len_H * 4, st));  // split tiles add in
  for (uint64_t j0 = 0; j0 < g.lwe_n; j0 += nc) {
    const uint32_t w = (uint32_t)std::min<uint64_t>(nc, g.lwe_n - j0);
    {
      const uint32_t nb = Npad / 16;  // Philox blocks (4 outputs x 4 limbs), 4 lanes each
      dim3 grid((uint32_t)g.G, (nb + 63) / 64);
      expand_A_limbs_kernel<<<grid, 256, 0, st>>>(ar.limbs, g.seed_A, (uint32_t)g.m, g.lwe_n,
                                                  (uint32_t)g.G, Npad, BN, (uint32_t)j0);
      LAUNCH_CHECK(ctx);
    }
    rc = launch_mma<OUT_ROW_MAJOR>(ctx, BN, ar.limbs, Npad, out + j0, w, g.lwe_n, len_H, st, 0,
                                   nullptr, chunked);
    if (rc) return rc;
  }
  if (out != H_local) {
    CUDA_TRY(ctx, cudaMemcpyAsync(H_local, out, len_H * 4,
                                  wh ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    if (!wh) CUDA_TRY(ctx, cudaStreamSynchronize(st));
  }
  return QPIR_OK;
}

uint64_t qpir_kernel_launches(const qpir_ctx* ctx) { return ctx ? ctx->launches : 0; }

const char* qpir_last_error(const qpir_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_setup_error.c_str();
}

void qpir_destroy(qpir_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard dg(ctx->device);
  void* bufs[] = {ctx->D, ctx->rec_stage, ctx->spec_stage, ctx->mldsa_buf, ctx->sig_stage};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (auto& kv : ctx->arenas) {
    Arena& a = kv.second;
    void* ab[] = {a.qu_dev, a.ans_dev, a.partial, a.tickets, a.limbs, a.big_out, a.acc64,
                  a.exc, a.in_small.buf[0], a.in_small.buf[1], a.in_big.buf[0], a.in_big.buf[1],
                  a.kprog, a.kb_done, a.conv_ctr};
    if (a.h2d) cudaStreamSynchronize(a.h2d);
    for (void* b : ab)
      if (b) cudaFree(b);
    for (InRing* r : {&a.in_small, &a.in_big})
      for (int k = 0; k < 2; ++k) {
        if (r->ready[k]) cudaEventDestroy(r->ready[k]);
        if (r->done[k]) cudaEventDestroy(r->done[k]);
      }
    if (a.h2d) cudaStreamDestroy(a.h2d);
  }
  delete ctx;
}

}  // extern "C"
