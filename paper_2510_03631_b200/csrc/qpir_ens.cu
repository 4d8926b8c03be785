// qpir_ens.cu -- C ABI for QPADL-ENS (Chor XOR PIR; NEXT-1), include/qpir.h.
// Host side only: validation, per-stream device scratch, dispatch to the
// ens.cuh scan / CUDA-core batch kernels and the ens_mma.cuh tensor-core batch.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <string>

#include "../../include/qpir.h"
#include "ens.cuh"
#include "ens_mma.cuh"
#include "host_common.h"
#include "mma_launch.cuh"
#include "puzzle.cuh"
#include "mldsa.cuh"

using namespace qpir;
using namespace qpir_host;

namespace {
thread_local std::string g_ens_setup_error;
}

// Host-input staging ring for single answers (share, OOP q and A_i): the H2D
// copy runs on the arena's copy stream, the compute stream waits only on its
// event, so the next answer's input lands while the previous scan runs.
struct EnsRing {
  uint8_t* buf[2] = {nullptr, nullptr};
  uint64_t bytes[2] = {0, 0};
  cudaEvent_t ready[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  unsigned slot = 0;
};

// Per-stream scratch: calls on different streams of one context may run
// concurrently (each stream owns its staging rings, accumulators, scan
// partials / tickets and tensor-core operands); calls on one stream are
// ordered by the stream.
struct EnsArena {
  cudaStream_t h2d = nullptr;   // copy stream for host inputs (lazily created)
  EnsRing r_share, r_q, r_A, r_batch;
  uint32_t* acc = nullptr;      // [max_B][dp/4] response words of a batch
  uint64_t acc_B = 0;
  uint32_t* acc1 = nullptr;     // [dp/4] + 1 done ticket: single-scan accumulator, kept zero
  uint8_t* io_stage = nullptr;  // [2][d]: host answer out of a single scan
  uint64_t io_stage_bytes = 0;
  uint8_t* Q_dev = nullptr;     // OOP offline: the expanded selectors of a seed batch
  uint64_t Q_bytes = 0;
  uint32_t* Qt = nullptr;       // transposed selector bits (CUDA-core batch)
  uint64_t Qt_bytes = 0;
  uint8_t* seed_dev = nullptr;  // OOP seeds
  uint64_t seed_bytes = 0;
  uint8_t* partial = nullptr;   // scan CTA partials
  uint64_t partial_bytes = 0;
  uint32_t* tickets = nullptr;  // scan group tickets (self-resetting)
  uint64_t tickets_bytes = 0;
  uint8_t* Qb = nullptr;        // shares as 0/1 bytes (tensor-core A operand)
  uint64_t Qb_bytes = 0;
};

struct qpir_ens_ctx {
  uint64_t r = 0, d = 0, dp = 0;
  int h2d_stream = 1;           // env QPIR_H2D_STREAM
  int device = 0, num_sms = 148;
  uint8_t* R = nullptr;         // [r][dp]
  std::atomic<bool> r_written{false};  // a kernel wrote R (puzzle bind): next scan without PDL
  uint8_t* spec_stage = nullptr;       // host spectrum staging (puzzle bind)
  uint64_t spec_stage_bytes = 0;
  uint8_t* mldsa_buf = nullptr;        // ML-DSA expanded key + seed (puzzle bind)
  uint64_t mldsa_buf_bytes = 0;
  uint8_t* sig_stage = nullptr;        // ML-DSA signatures, 3024-byte rows
  uint64_t sig_stage_bytes = 0;
  std::mutex mu;                // guards `arenas`
  std::map<cudaStream_t, EnsArena> arenas;
  int group = 0;                // env QPIR_ENS_GROUP (0 = auto 32; 1 = atomics only)
  int wide = 1;                 // env QPIR_ENS_WIDE (uniform-row kernel for d > 2 KB;
                                //   2 = 32-byte chunks per thread, 256-bit loads)
  int pdl = 1;                  // env QPIR_ENS_PDL (programmatic dependent launch of scans)
  int tc = -1;                  // env QPIR_ENS_TC: -1 auto, 0 CUDA cores, 1 tensor cores
  int flags = 0;                // qpir_ens_params.flags (QPIR_FLAG_STABLE_INPUTS)
  int mma_split = 0;            // env QPIR_MMA_SPLIT (0 = auto)
  int ts = 1;                   // env QPIR_ENS_TS: bit-rows in TMEM (1) or shared memory (0)
  std::atomic<uint64_t> launches{0};
  std::atomic<int> last_path{QPIR_ENS_PATH_NONE};
  int rows_per_cta = 0;       // env QPIR_ENS_ROWS (0 = auto)
  int ur = 16;                // env QPIR_ENS_UR (rows in flight per thread: 4, 8, 16)
  std::string err;
};

#define ENS_FAIL(ctx, code, ...) set_error(&(ctx)->err, code, __VA_ARGS__)
#define ENS_CUDA(ctx, call)                                                                  \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return ENS_FAIL(ctx, e_ == cudaErrorMemoryAllocation ? QPIR_E_OOM : QPIR_E_CUDA,      \
                      "%s: %s", #call, cudaGetErrorString(e_));                              \
  } while (0)
#define ENS_LAUNCHED(ctx)                                                                    \
  do {                                                                                       \
    (ctx)->launches++;                                                                       \
    cudaError_t e_ = cudaGetLastError();                                                     \
    if (e_ != cudaSuccess)                                                                   \
      return ENS_FAIL(ctx, QPIR_E_CUDA, "kernel launch: %s", cudaGetErrorString(e_));       \
  } while (0)

namespace {

int grow(qpir_ens_ctx* ctx, void** buf, uint64_t* have, uint64_t need) {
  if (*have >= need) return QPIR_OK;
  if (*buf) cudaFree(*buf);
  *buf = nullptr;
  *have = 0;
  ENS_CUDA(ctx, cudaMalloc(buf, need));
  *have = need;
  return QPIR_OK;
}

// The arena of stream `st`, created on first use; its single-scan accumulator
// (acc1, self-resetting in the kernel) is zeroed on `st` once.
int arena_for(qpir_ens_ctx* ctx, cudaStream_t st, EnsArena** out) {
  EnsArena* ar;
  {
    std::lock_guard<std::mutex> lk(ctx->mu);
    ar = &ctx->arenas[st];  // std::map references stay valid across inserts
  }
  if (!ar->acc1) {
    ENS_CUDA(ctx, cudaMalloc(&ar->acc1, ctx->dp + 16));
    ENS_CUDA(ctx, cudaMemsetAsync(ar->acc1, 0, ctx->dp + 16, st));
  }
  *out = ar;
  return QPIR_OK;
}

// Stage a possibly-host input through `ring` for work on `st`: device inputs
// pass through (slot -1); host inputs are copied on the arena's copy stream (or
// on `st` while it is being captured into a CUDA graph).  The caller records
// ring.done[slot] on `st` after the kernels that read the slot.
int stage_ring(qpir_ens_ctx* ctx, EnsArena& ar, EnsRing& ring, const uint8_t* src,
               uint64_t bytes, cudaStream_t st, const uint8_t** dev, int* slot) {
  *slot = -1;
  const int w = where(src, ctx->device);
  if (w < 0) return ENS_FAIL(ctx, QPIR_E_PARAM, "input: memory of another device");
  if (w == 1) {
    *dev = src;
    return QPIR_OK;
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  ENS_CUDA(ctx, cudaStreamIsCapturing(st, &cs));
  const bool side = cs == cudaStreamCaptureStatusNone && ctx->h2d_stream;
  const unsigned k = side ? ring.slot : 0u;
  if (side) {
    ring.slot ^= 1u;
    if (!ar.h2d) ENS_CUDA(ctx, cudaStreamCreateWithFlags(&ar.h2d, cudaStreamNonBlocking));
    if (!ring.ready[k]) {
      ENS_CUDA(ctx, cudaEventCreateWithFlags(&ring.ready[k], cudaEventDisableTiming));
      ENS_CUDA(ctx, cudaEventCreateWithFlags(&ring.done[k], cudaEventDisableTiming));
    }
  }
  if (ring.bytes[k] < bytes) {
    if (ring.done[k]) ENS_CUDA(ctx, cudaEventSynchronize(ring.done[k]));
    int rc = grow(ctx, (void**)&ring.buf[k], &ring.bytes[k], round_up(bytes, 16));
    if (rc) return rc;
  }
  if (side) {
    ENS_CUDA(ctx, cudaStreamWaitEvent(ar.h2d, ring.done[k], 0));
    ENS_CUDA(ctx, cudaMemcpyAsync(ring.buf[k], src, bytes, cudaMemcpyHostToDevice, ar.h2d));
    ENS_CUDA(ctx, cudaEventRecord(ring.ready[k], ar.h2d));
    ENS_CUDA(ctx, cudaStreamWaitEvent(st, ring.ready[k], 0));
    *slot = (int)k;
  } else {
    ENS_CUDA(ctx, cudaMemcpyAsync(ring.buf[k], src, bytes, cudaMemcpyHostToDevice, st));
  }
  *dev = ring.buf[k];
  return QPIR_OK;
}

// Copy B rows of d bytes out of the dp-strided accumulator into `out`.
int copy_out(qpir_ens_ctx* ctx, EnsArena& ar, uint8_t* out, uint64_t B, cudaStream_t st) {
  const int w = where(out, ctx->device);
  if (w < 0) return ENS_FAIL(ctx, QPIR_E_PARAM, "out: memory of another device");
  ENS_CUDA(ctx, cudaMemcpy2DAsync(out, ctx->d, ar.acc, ctx->dp, ctx->d, B,
                                  w ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  if (!w) ENS_CUDA(ctx, cudaStreamSynchronize(st));
  return QPIR_OK;
}

}  // namespace

extern "C" {

int qpir_ens_setup(const qpir_ens_params* p, const uint8_t* records, uint64_t records_len,
                   void* stream, qpir_ens_ctx** out) {
  NvtxRange nvtx_("qpir_ens_setup");
  g_ens_setup_error.clear();
  if (!out) return set_error(&g_ens_setup_error, QPIR_E_PARAM, "out: NULL");
  *out = nullptr;
  if (!p) return set_error(&g_ens_setup_error, QPIR_E_PARAM, "params: NULL");
  if (p->flags & ~QPIR_FLAG_STABLE_INPUTS)
    return set_error(&g_ens_setup_error, QPIR_E_PARAM, "flags: unknown bits 0x%x", (unsigned)p->flags);
  if (p->n_records == 0) return set_error(&g_ens_setup_error, QPIR_E_DIMENSION, "n_records: 0");
  if (p->rec_bytes == 0 || p->rec_bytes > 16384)
    return set_error(&g_ens_setup_error, QPIR_E_DIMENSION, "rec_bytes: %llu not in [1, 16384]",
                     (unsigned long long)p->rec_bytes);
  if (records && records_len != p->n_records * p->rec_bytes)
    return set_error(&g_ens_setup_error, QPIR_E_DIMENSION, "records_len: %llu != %llu",
                     (unsigned long long)records_len,
                     (unsigned long long)(p->n_records * p->rec_bytes));
  if (p->device < 0) return set_error(&g_ens_setup_error, QPIR_E_PARAM, "device: < 0");
  int sms = 148;
  std::string e = check_device(p->device, &sms);
  if (!e.empty()) return set_error(&g_ens_setup_error, QPIR_E_CUDA, "%s", e.c_str());
  DeviceGuard dg(p->device);
  qpir_ens_ctx* ctx = new qpir_ens_ctx();
  ctx->r = p->n_records;
  ctx->d = p->rec_bytes;
  ctx->dp = round_up(p->rec_bytes, 16);
  ctx->device = p->device;
  ctx->num_sms = sms;
  ctx->rows_per_cta = env_int("QPIR_ENS_ROWS", 0);
  ctx->ur = env_int("QPIR_ENS_UR", 16);
  ctx->group = env_int("QPIR_ENS_GROUP", 0);
  ctx->wide = env_int("QPIR_ENS_WIDE", 1);
  ctx->pdl = env_int("QPIR_ENS_PDL", 1);
  ctx->h2d_stream = env_int("QPIR_H2D_STREAM", 1);
  ctx->tc = env_int("QPIR_ENS_TC", -1);
  ctx->flags = p->flags;
  ctx->mma_split = env_int("QPIR_MMA_SPLIT", 0);
  ctx->ts = env_int("QPIR_ENS_TS", 1);
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMalloc(&ctx->R, ctx->r * ctx->dp) != cudaSuccess) {
    cudaGetLastError();
    g_ens_setup_error = "records: cudaMalloc failed";
    qpir_ens_destroy(ctx);
    return QPIR_E_OOM;
  }
  int rc = QPIR_OK;
  if (cudaMemsetAsync(ctx->R, 0, ctx->r * ctx->dp, st) != cudaSuccess) rc = QPIR_E_CUDA;
  if (!rc && records) rc = qpir_ens_db_write(ctx, 0, ctx->r, records, records_len, stream);
  if (!rc && cudaStreamSynchronize(st) != cudaSuccess) rc = QPIR_E_CUDA;
  if (rc) {
    g_ens_setup_error = ctx->err.empty() ? "setup failed" : ctx->err;
    qpir_ens_destroy(ctx);
    return rc;
  }
  *out = ctx;
  return QPIR_OK;
}

int qpir_ens_db_write(qpir_ens_ctx* ctx, uint64_t theta_begin, uint64_t n_records,
                      const uint8_t* records, uint64_t records_len, void* stream) {
  NvtxRange nvtx_("qpir_ens_db_write");
  if (!ctx) return QPIR_E_STATE;
  if (theta_begin > ctx->r || n_records > ctx->r - theta_begin)
    return ENS_FAIL(ctx, QPIR_E_DIMENSION, "theta range: [%llu, +%llu) exceeds %llu records",
                    (unsigned long long)theta_begin, (unsigned long long)n_records,
                    (unsigned long long)ctx->r);
  if (records_len != n_records * ctx->d)
    return ENS_FAIL(ctx, QPIR_E_DIMENSION, "records_len: %llu != %llu",
                    (unsigned long long)records_len, (unsigned long long)(n_records * ctx->d));
  if (n_records == 0) return QPIR_OK;
  if (!records) return ENS_FAIL(ctx, QPIR_E_PARAM, "records: NULL");
  DeviceGuard dg(ctx->device);
  const int w = where(records, ctx->device);
  if (w < 0) return ENS_FAIL(ctx, QPIR_E_PARAM, "records: memory of another device");
  cudaStream_t st = (cudaStream_t)stream;
  // a copy (not a kernel): stream-ordered before any later scan, which reads R
  // only after griddepcontrol.wait
  ENS_CUDA(ctx, cudaMemcpy2DAsync(ctx->R + theta_begin * ctx->dp, ctx->dp, records, ctx->d,
                                  ctx->d, n_records,
                                  w ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  if (!w) ENS_CUDA(ctx, cudaStreamSynchronize(st));
  return QPIR_OK;
}

int qpir_ens_puzzle_bind_hct(qpir_ens_ctx* ctx, uint64_t theta_begin, uint64_t n_records,
                             const uint8_t* spectrum, uint64_t spec_stride,
                             uint64_t spectrum_len, uint64_t seed_psd, uint32_t kappa,
                             uint8_t n_l, const uint8_t* mldsa_seed, uint8_t* mldsa_pk,
                             void* stream) {
  NvtxRange nvtx_("qpir_ens_puzzle_bind_hct");
  if (!ctx) return QPIR_E_STATE;
  if (ctx->d < HCT_SPECTRUM + HCT_PUZZLE)
    return ENS_FAIL(ctx, QPIR_E_DIMENSION, "rec_bytes: %llu < 597 (560 B spectrum + 37 B puzzle)",
                    (unsigned long long)ctx->d);
  if (mldsa_seed && ctx->d < HCT_SIG_END)
    return ENS_FAIL(ctx, QPIR_E_DIMENSION, "rec_bytes: %llu < 3017 (spectrum + puzzle + ML-DSA signature)",
                    (unsigned long long)ctx->d);
  if (theta_begin > ctx->r || n_records > ctx->r - theta_begin)
    return ENS_FAIL(ctx, QPIR_E_DIMENSION, "theta range: [%llu, +%llu) exceeds %llu records",
                    (unsigned long long)theta_begin, (unsigned long long)n_records,
                    (unsigned long long)ctx->r);
  if (spec_stride < HCT_SPECTRUM)
    return ENS_FAIL(ctx, QPIR_E_DIMENSION, "spec_stride: %llu < 560", (unsigned long long)spec_stride);
  if (spectrum_len != n_records * spec_stride)
    return ENS_FAIL(ctx, QPIR_E_DIMENSION, "spectrum_len: %llu != %llu",
                    (unsigned long long)spectrum_len, (unsigned long long)(n_records * spec_stride));
  if (n_records == 0) return QPIR_OK;
  if (!spectrum) return ENS_FAIL(ctx, QPIR_E_PARAM, "spectrum: NULL");
  DeviceGuard dg(ctx->device);
  const int w = where(spectrum, ctx->device);
  if (w < 0) return ENS_FAIL(ctx, QPIR_E_PARAM, "spectrum: memory of another device");
  cudaStream_t st = (cudaStream_t)stream;
  uint64_t chunk = w ? n_records : std::max<uint64_t>(1, (64ull << 20) / spec_stride);
  qpir::mldsa::MldsaKey* key = nullptr;
  uint32_t* ticket = nullptr;  // the signer's record counter (after xi in mldsa_buf)
  if (mldsa_seed) {
    chunk = std::min<uint64_t>(chunk, 65536);
    int rc = grow(ctx, (void**)&ctx->mldsa_buf, &ctx->mldsa_buf_bytes, sizeof(qpir::mldsa::MldsaKey) + 64);
    if (rc) return rc;
    key = reinterpret_cast<qpir::mldsa::MldsaKey*>(ctx->mldsa_buf);
    uint8_t* xi_dev = ctx->mldsa_buf + sizeof(qpir::mldsa::MldsaKey);
    ticket = reinterpret_cast<uint32_t*>(xi_dev + 32);
    ENS_CUDA(ctx, cudaMemcpyAsync(xi_dev, mldsa_seed, 32, cudaMemcpyDefault, st));
    ENS_CUDA(ctx, qpir::mldsa::keygen(xi_dev, key, st));
    ctx->launches++;
    if (mldsa_pk)
      ENS_CUDA(ctx, cudaMemcpyAsync(mldsa_pk, key->pk, qpir::mldsa::PK_BYTES, cudaMemcpyDefault, st));
    rc = grow(ctx, (void**)&ctx->sig_stage, &ctx->sig_stage_bytes, std::min(n_records, chunk) * HCT_SIG_STRIDE);
    if (rc) return rc;
    ENS_CUDA(ctx, cudaMemsetAsync(ctx->sig_stage, 0, std::min(n_records, chunk) * HCT_SIG_STRIDE, st));
  }
  if (!w) {
    int rc = grow(ctx, (void**)&ctx->spec_stage, &ctx->spec_stage_bytes,
                  std::min(n_records, chunk) * spec_stride);
    if (rc) return rc;
  }
  for (uint64_t t = 0; t < n_records; t += chunk) {
    const uint64_t n = std::min(chunk, n_records - t);
    const uint8_t* sp = spectrum + t * spec_stride;
    if (!w) {
      ENS_CUDA(ctx, cudaMemcpyAsync(ctx->spec_stage, sp, n * spec_stride, cudaMemcpyHostToDevice, st));
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
    b.d = (uint32_t)ctx->d;
    b.out = ctx->R + (theta_begin + t) * ctx->dp;  // rows in place (padding bytes stay zero)
    b.out_stride = ctx->dp;
    if (key) {
      ENS_CUDA(ctx, qpir::mldsa::sign_records(key, theta_begin + t, n, seed_psd, kappa, n_l, ctx->sig_stage,
                                            ticket, st));
      ctx->launches++;
      b.sig = ctx->sig_stage;
    }
    launch_puzzle_bind(b, st);
    ENS_LAUNCHED(ctx);
    ctx->r_written.store(true);
  }
  if (mldsa_pk && where(mldsa_pk, ctx->device) == 0) ENS_CUDA(ctx, cudaStreamSynchronize(st));
  if (!w) ENS_CUDA(ctx, cudaStreamSynchronize(st));
  return QPIR_OK;
}

// One scan of rows [row_lo, row_hi) selected by share_dev, finalised in the
// kernel: out_dev (device, d bytes) = init_dev ^ XOR of the selected rows.
// early: the share was not written by the kernel preceding this launch (staged
// by the library from host memory, or QPIR_FLAG_STABLE_INPUTS): the scan may
// run before griddepcontrol.wait.
static int scan_range(qpir_ens_ctx* ctx, EnsArena& ar, const uint8_t* share_dev,
                      uint64_t row_lo, uint64_t row_hi, const uint8_t* init_dev,
                      uint8_t* out_dev, cudaStream_t st, bool early) {
  EnsArgs a;
  a.early = early ? 1u : 0u;
  a.R = ctx->R;
  a.q = share_dev;
  a.out = ar.acc1;
  a.fin_out = out_dev;
  a.init = init_dev;
  a.d = (uint32_t)ctx->d;
  a.done = ar.acc1 + ctx->dp / 4;
  a.row_lo = row_lo;
  a.row_hi = row_hi;
  a.dp = (uint32_t)ctx->dp;
  a.W = (uint32_t)(ctx->dp / 16);
  const uint32_t R = std::max<uint32_t>(1, 256 / a.W);
  uint32_t threads = a.W * R;
  const int UR = ctx->ur == 8 ? 8 : ctx->ur == 4 ? 4 : 16;
  uint64_t rows = ctx->rows_per_cta;
  if (rows == 0) {
    // ~384 KB of records per CTA (measured best on B200 at d = 3072 with the
    // 64-register wide kernel: 128 rows, profiles/r01_sweep_run40.log; 64 rows
    // before, run10), at least ~4 CTAs per SM for short ranges (OOP flip
    // chunks), and at least one full unrolled step
    const uint64_t by_bytes = (384u << 10) / ctx->dp;
    const uint64_t by_occ = (row_hi - row_lo + 4ull * ctx->num_sms - 1) / (4ull * ctx->num_sms);
    rows = std::max<uint64_t>(std::min(by_bytes, by_occ), (uint64_t)R * UR);
  }
  rows = round_up(rows, (uint64_t)R * UR);
  if (R == 1) rows = round_up(rows, 32);  // 32-row selector words (wide kernel)
  a.rows_per_cta = rows;
  const uint64_t grid = (row_hi - row_lo + rows - 1) / rows;
  a.partial = nullptr;
  a.tickets = nullptr;
  a.group = 1;
  const uint32_t group = ctx->group > 0 ? (uint32_t)ctx->group : 32;
  if (grid > 4ull * ctx->num_sms && group > 1) {
    // many small CTAs: two-level XOR reduction instead of grid x W atomics
    const uint64_t ngroups = (grid + group - 1) / group;
    int rc = grow(ctx, (void**)&ar.partial, &ar.partial_bytes, grid * a.W * 16);
    if (rc) return rc;
    if (ngroups * 4 > ar.tickets_bytes) {
      rc = grow(ctx, (void**)&ar.tickets, &ar.tickets_bytes, ngroups * 4);
      if (rc) return rc;
      ENS_CUDA(ctx, cudaMemsetAsync(ar.tickets, 0, ar.tickets_bytes, st));
    }
    a.partial = reinterpret_cast<uint4*>(ar.partial);
    a.tickets = ar.tickets;
    a.group = group;
  }
  a.leaders = (uint32_t)(a.partial ? (grid + a.group - 1) / a.group : grid);
  const size_t smem = R > 1 ? threads * 16 : 0;
  const bool wide = R == 1 && ctx->wide && (rows % 32 == 0) &&
                    ((reinterpret_cast<uintptr_t>(share_dev) & 3u) == 0);
  // 32-byte chunks per thread (256-bit loads) when the row stride allows
  const bool cw2 = wide && ctx->wide == 2 && (a.dp % 32 == 0);
  if (cw2) threads = a.W / 2;
  void (*kern)(EnsArgs);
  if (wide)
    kern = cw2 ? ens_scan_wide_kernel<16, 2>
               : UR == 8 ? ens_scan_wide_kernel<8, 1> : ens_scan_wide_kernel<16, 1>;
  else
    kern = UR == 16 ? ens_scan_kernel<16> : UR == 4 ? ens_scan_kernel<4> : ens_scan_kernel<8>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((uint32_t)grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = wide ? 0 : smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  // a scan may read R before griddepcontrol.wait: right after a kernel wrote R
  // (qpir_ens_puzzle_bind_hct) it is launched without PDL
  const bool after_write = ctx->r_written.exchange(false);
  attr[0].val.programmaticStreamSerializationAllowed = (ctx->pdl && !after_write) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ENS_CUDA(ctx, cudaLaunchKernelEx(&cfg, kern, a));
  ENS_LAUNCHED(ctx);
  ctx->last_path = QPIR_ENS_PATH_SCAN;
  return QPIR_OK;
}

int qpir_ens_answer(qpir_ens_ctx* ctx, const uint8_t* share, uint64_t len_share, uint8_t* out,
                    uint64_t len_out, void* stream) {
  NvtxRange nvtx_("qpir_ens_answer");
  if (!ctx) return QPIR_E_STATE;
  const uint64_t nb = (ctx->r + 7) / 8;
  if (!share || !out) return ENS_FAIL(ctx, QPIR_E_PARAM, "share/out: NULL");
  if (len_share != nb)
    return ENS_FAIL(ctx, QPIR_E_DIMENSION, "len_share: %llu != %llu", (unsigned long long)len_share,
                    (unsigned long long)nb);
  if (len_out != ctx->d)
    return ENS_FAIL(ctx, QPIR_E_DIMENSION, "len_out: %llu != d %llu", (unsigned long long)len_out,
                    (unsigned long long)ctx->d);
  DeviceGuard dg(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int wo = where(out, ctx->device);
  if (wo < 0) return ENS_FAIL(ctx, QPIR_E_PARAM, "out: memory of another device");
  EnsArena* ar = nullptr;
  int rc = arena_for(ctx, st, &ar);
  if (rc) return rc;
  rc = grow(ctx, (void**)&ar->io_stage, &ar->io_stage_bytes, 2 * ctx->d);
  if (rc) return rc;
  const uint8_t* qd = nullptr;
  int slot = -1;
  rc = stage_ring(ctx, *ar, ar->r_share, share, nb, st, &qd, &slot);
  if (rc) return rc;
  uint8_t* od = wo ? out : ar->io_stage + ctx->d;
  rc = scan_range(ctx, *ar, qd, 0, ctx->r, nullptr, od, st,
                  qd != share || (ctx->flags & QPIR_FLAG_STABLE_INPUTS));
  if (rc) return rc;
  if (slot >= 0) ENS_CUDA(ctx, cudaEventRecord(ar->r_share.done[slot], st));
  if (!wo) {
    ENS_CUDA(ctx, cudaMemcpyAsync(out, od, ctx->d, cudaMemcpyDeviceToHost, st));
    ENS_CUDA(ctx, cudaStreamSynchronize(st));
  }
  return QPIR_OK;
}

int qpir_oop_answer(qpir_ens_ctx* ctx, uint32_t n_chunks, uint32_t server, const uint8_t* q,
                    uint64_t len_q, const uint8_t* A, uint64_t len_A, uint8_t* out,
                    uint64_t len_out, void* stream) {
  NvtxRange nvtx_("qpir_oop_answer");
  if (!ctx) return QPIR_E_STATE;
  if (n_chunks < 2 || ctx->r % n_chunks != 0)
    return ENS_FAIL(ctx, QPIR_E_PARAM, "n_chunks: %u must be >= 2 and divide r = %llu", n_chunks,
                    (unsigned long long)ctx->r);
  if (server >= n_chunks) return ENS_FAIL(ctx, QPIR_E_PARAM, "server: %u >= n_chunks", server);
  const uint64_t k = ctx->r / n_chunks, kb = (k + 7) / 8;
  if (!q || !A || !out) return ENS_FAIL(ctx, QPIR_E_PARAM, "q/A/out: NULL");
  if (len_q != kb)
    return ENS_FAIL(ctx, QPIR_E_DIMENSION, "len_q: %llu != ceil(k/8) %llu", (unsigned long long)len_q,
                    (unsigned long long)kb);
  if (len_A != ctx->d || len_out != ctx->d)
    return ENS_FAIL(ctx, QPIR_E_DIMENSION, "len_A/len_out: must equal d %llu",
                    (unsigned long long)ctx->d);
  DeviceGuard dg(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int wo = where(out, ctx->device);
  if (wo < 0) return ENS_FAIL(ctx, QPIR_E_PARAM, "out: memory of another device");
  EnsArena* ar = nullptr;
  int rc = arena_for(ctx, st, &ar);
  if (rc) return rc;
  rc = grow(ctx, (void**)&ar->io_stage, &ar->io_stage_bytes, 2 * ctx->d);
  if (rc) return rc;
  const uint8_t* qd = nullptr;
  int sq = -1, sA = -1;
  rc = stage_ring(ctx, *ar, ar->r_q, q, kb, st, &qd, &sq);
  if (rc) return rc;
  // R_i := A_i XOR q_i . chunk_i (Lemma 2): A_i is XORed in by the finalising CTA
  const uint8_t* Ad = nullptr;
  rc = stage_ring(ctx, *ar, ar->r_A, A, ctx->d, st, &Ad, &sA);
  if (rc) return rc;
  uint8_t* od = wo ? out : ar->io_stage + ctx->d;
  rc = scan_range(ctx, *ar, qd, (uint64_t)server * k, (uint64_t)(server + 1) * k, Ad, od, st,
                  qd != q || (ctx->flags & QPIR_FLAG_STABLE_INPUTS));
  if (rc) return rc;
  if (sq >= 0) ENS_CUDA(ctx, cudaEventRecord(ar->r_q.done[sq], st));
  if (sA >= 0) ENS_CUDA(ctx, cudaEventRecord(ar->r_A.done[sA], st));
  if (!wo) {
    ENS_CUDA(ctx, cudaMemcpyAsync(out, od, ctx->d, cudaMemcpyDeviceToHost, st));
    ENS_CUDA(ctx, cudaStreamSynchronize(st));
  }
  return QPIR_OK;
}

int qpir_oop_preprocess(qpir_ens_ctx* ctx, uint32_t n_chunks, uint32_t server,
                        const uint64_t* seeds, uint64_t n_seeds, uint8_t* A_out, uint64_t len_A,
                        void* stream) {
  NvtxRange nvtx_("qpir_oop_preprocess");
  if (!ctx) return QPIR_E_STATE;
  if (n_chunks < 2 || ctx->r % n_chunks != 0)
    return ENS_FAIL(ctx, QPIR_E_PARAM, "n_chunks: %u must be >= 2 and divide r = %llu", n_chunks,
                    (unsigned long long)ctx->r);
  if (server >= n_chunks) return ENS_FAIL(ctx, QPIR_E_PARAM, "server: %u >= n_chunks", server);
  if (!seeds || !A_out) return ENS_FAIL(ctx, QPIR_E_PARAM, "seeds/A_out: NULL");
  if (n_seeds == 0 || n_seeds > 65535)
    return ENS_FAIL(ctx, QPIR_E_PARAM, "n_seeds: %llu not in [1, 65535]", (unsigned long long)n_seeds);
  if (len_A != n_seeds * ctx->d)
    return ENS_FAIL(ctx, QPIR_E_DIMENSION, "len_A: %llu != n_seeds*d %llu", (unsigned long long)len_A,
                    (unsigned long long)(n_seeds * ctx->d));
  DeviceGuard dg(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  EnsArena* ar = nullptr;
  int rc = arena_for(ctx, st, &ar);
  if (rc) return rc;
  const uint64_t nb = (ctx->r + 7) / 8;
  rc = grow(ctx, (void**)&ar->Q_dev, &ar->Q_bytes, n_seeds * nb);
  if (rc) return rc;
  rc = grow(ctx, (void**)&ar->seed_dev, &ar->seed_bytes, n_seeds * 8);
  if (rc) return rc;
  const int ws = where(seeds, ctx->device);
  if (ws < 0) return ENS_FAIL(ctx, QPIR_E_PARAM, "seeds: memory of another device");
  ENS_CUDA(ctx, cudaMemcpyAsync(ar->seed_dev, seeds, n_seeds * 8,
                                ws ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  {
    dim3 grid((uint32_t)((nb + 255) / 256), (uint32_t)n_seeds);
    oop_expand_kernel<<<grid, 256, 0, st>>>((const unsigned long long*)ar->seed_dev, ar->Q_dev,
                                            ctx->r, ctx->r / n_chunks, n_chunks, server, nb);
    ENS_LAUNCHED(ctx);
  }
  // A = q . DB for every seed: the ENS multi-request kernel on the expanded shares
  return qpir_ens_answer_batch(ctx, ar->Q_dev, n_seeds, n_seeds * nb, A_out, len_A, stream);
}

}  // extern "C"

// Multi-request GF(2) product on tensor cores (ens_mma.cuh): the records are
// read once, in place, and expanded to weighted bit-rows in shared memory;
// the shares are 0/1 bytes (B x r bytes, expanded once per call).
template <uint32_t MS, uint32_t NT, uint32_t S, uint32_t RS>
static cudaError_t ens_mma_launch(qpir_ens_ctx* ctx, EnsMmaArgs a, cudaStream_t st) {
  using C = EmCfg<MS, NT, S, RS>;
  auto kern = qpir_ens_mma_kernel<MS, NT, S, RS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::TOTAL);
  if (e != cudaSuccess) return e;
  const uint32_t units = a.s_tiles * a.w_tiles * a.splits;
  kern<<<std::min<uint32_t>(units, (uint32_t)ctx->num_sms), EM_THREADS, C::TOTAL, st>>>(a);
  return cudaGetLastError();
}

template <uint32_t S, uint32_t SA, uint32_t RS>
static cudaError_t ens_mma_ts_launch(qpir_ens_ctx* ctx, EnsMmaArgs a, cudaStream_t st) {
  using C = EtCfg<S, SA, RS>;
  auto kern = qpir_ens_mma_ts_kernel<S, SA, RS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::TOTAL);
  if (e != cudaSuccess) return e;
  const uint32_t units = a.s_tiles * a.w_tiles * a.splits;
  kern<<<std::min<uint32_t>(units, (uint32_t)ctx->num_sms), ET_THREADS, C::TOTAL, st>>>(a);
  return cudaGetLastError();
}

static int ens_batch_tc(qpir_ens_ctx* ctx, EnsArena& ar, const uint8_t* Qd, uint64_t B,
                        cudaStream_t st) {
  if (ctx->ts) {
    // shares in TMEM (ens_mma.cuh, TS form): units of 128 shares x 32 record bytes
    const uint32_t rows64 = (uint32_t)((ctx->r + 63) / 64);
    const uint32_t ld = (uint32_t)round_up(B, 128ull);
    int rc = grow(ctx, (void**)&ar.Qb, &ar.Qb_bytes, (uint64_t)rows64 * ld * 8);
    if (rc) return rc;
    unsigned long long* Qp = reinterpret_cast<unsigned long long*>(ar.Qb);
    {
      const uint32_t tiles = (rows64 + 31) / 32;  // 32 K-blocks per CTA
      const uint32_t gy = std::min<uint32_t>(tiles, 65535);
      const uint32_t gz = (tiles + gy - 1) / gy;
      dim3 grid(ld / 32, gy, gz);
      ens_share_pack_kernel<<<grid, ESP_THREADS, 0, st>>>(Qd, (uint32_t)B, ctx->r, (ctx->r + 7) / 8, Qp,
                                                          rows64, ld);
      ENS_LAUNCHED(ctx);
    }
    EnsMmaArgs a;
    a.R = ctx->R;
    a.Qb = nullptr;
    a.Qp = Qp;
    a.qp_ld = ld;
    a.qp_rows = rows64;
    a.out = ar.acc;
    a.r = ctx->r;
    a.dp = (uint32_t)ctx->dp;
    a.out_ld = (uint32_t)(ctx->dp / 4);
    a.B = (uint32_t)B;
    a.G16 = 0;
    a.s_tstride = 0;
    a.s_tiles = ld / 128;
    a.w_tiles = (uint32_t)((ctx->dp + 31) / 32);
    a.kblocks = (uint32_t)((ctx->r + ET_KB - 1) / ET_KB);
    const uint32_t tiles = a.s_tiles * a.w_tiles;
    a.splits = mma_choose_splits(tiles, a.kblocks, (uint32_t)ctx->num_sms, ctx->mma_split, 1,
                                 (double)B * ctx->dp, (double)ET_KB * 32 * ctx->num_sms, false);
    a.kbps = (a.kblocks + a.splits - 1) / a.splits;
    a.splits = (a.kblocks + a.kbps - 1) / a.kbps;
    if (a.splits > 1) ENS_CUDA(ctx, cudaMemsetAsync(ar.acc, 0, B * ctx->dp, st));
    const cudaError_t e = ens_mma_ts_launch<4, 8, 8>(ctx, a, st);
    if (e != cudaSuccess)
      return ENS_FAIL(ctx, QPIR_E_CUDA, "tcgen05 GF(2) GEMM (TS): %s", cudaGetErrorString(e));
    ctx->launches++;
    ctx->last_path = QPIR_ENS_PATH_TENSOR;
    return QPIR_OK;
  }
  // MS share tiles of 128 x NT width tiles of 256 bit-rows (32 record bytes)
  // share the 512 TMEM columns: B <= 128 -> 1 x 2 (64 record bytes per unit),
  // larger B -> 2 x 1 (the expanded record slice feeds 256 shares).
  const uint32_t MS = B <= 128 ? 1 : 2, NT = B <= 128 ? 2 : 1;
  const uint64_t m_pad = round_up(ctx->r, 128);
  const uint32_t G16 = (uint32_t)(m_pad / 16);
  const uint64_t Npad = round_up(B, 128ull * MS);
  int rc = grow(ctx, (void**)&ar.Qb, &ar.Qb_bytes, Npad * m_pad);
  if (rc) return rc;
  {
    const uint32_t gy = std::min<uint32_t>(G16, 65535);
    const uint32_t gz = (G16 + gy - 1) / gy;
    dim3 grid((uint32_t)(Npad / 128), gy, gz);
    ens_share_expand_kernel<<<grid, 128, 0, st>>>(Qd, (uint32_t)B, ctx->r, (ctx->r + 7) / 8, ar.Qb,
                                                  G16, (uint32_t)Npad, 128);
    ENS_LAUNCHED(ctx);
  }
  EnsMmaArgs a;
  a.R = ctx->R;
  a.Qb = ar.Qb;
  a.out = ar.acc;
  a.r = ctx->r;
  a.dp = (uint32_t)ctx->dp;
  a.out_ld = (uint32_t)(ctx->dp / 4);
  a.B = (uint32_t)B;
  a.G16 = G16;
  a.s_tstride = (uint64_t)G16 * 2048;
  a.s_tiles = (uint32_t)(Npad / (128ull * MS));
  a.w_tiles = (uint32_t)((ctx->dp + 32 * NT - 1) / (32 * NT));
  a.kblocks = (uint32_t)((ctx->r + EM_KB - 1) / EM_KB);
  const uint32_t tiles = a.s_tiles * a.w_tiles;
  // wave_bytes: the record bytes all CTAs expand per K-block (cost model of
  // mma_choose_splits: the split adds a memset and XOR atomics on the output)
  a.splits = mma_choose_splits(tiles, a.kblocks, (uint32_t)ctx->num_sms, ctx->mma_split, 1,
                               (double)B * ctx->dp, (double)EM_KB * 32 * NT * ctx->num_sms, false);
  a.kbps = (a.kblocks + a.splits - 1) / a.splits;
  a.splits = (a.kblocks + a.kbps - 1) / a.kbps;
  if (a.splits > 1) ENS_CUDA(ctx, cudaMemsetAsync(ar.acc, 0, B * ctx->dp, st));
  const cudaError_t e = MS == 1 ? ens_mma_launch<1, 2, 4, 8>(ctx, a, st)
                                : ens_mma_launch<2, 1, 5, 12>(ctx, a, st);
  if (e != cudaSuccess) return ENS_FAIL(ctx, QPIR_E_CUDA, "tcgen05 GF(2) GEMM: %s", cudaGetErrorString(e));
  ctx->launches++;
  ctx->last_path = QPIR_ENS_PATH_TENSOR;
  return QPIR_OK;
}

extern "C" {

int qpir_ens_answer_batch(qpir_ens_ctx* ctx, const uint8_t* shares, uint64_t B,
                          uint64_t len_shares, uint8_t* out, uint64_t len_out, void* stream) {
  NvtxRange nvtx_("qpir_ens_answer_batch");
  if (!ctx) return QPIR_E_STATE;
  const uint64_t nb = (ctx->r + 7) / 8;
  if (!shares || !out) return ENS_FAIL(ctx, QPIR_E_PARAM, "shares/out: NULL");
  if (B == 0 || B > 65536) return ENS_FAIL(ctx, QPIR_E_PARAM, "B: %llu not in [1, 65536]",
                                           (unsigned long long)B);
  if (len_shares != B * nb)
    return ENS_FAIL(ctx, QPIR_E_DIMENSION, "len_shares: %llu != B*ceil(r/8) %llu",
                    (unsigned long long)len_shares, (unsigned long long)(B * nb));
  if (len_out != B * ctx->d)
    return ENS_FAIL(ctx, QPIR_E_DIMENSION, "len_out: %llu != B*d %llu", (unsigned long long)len_out,
                    (unsigned long long)(B * ctx->d));
  DeviceGuard dg(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  EnsArena* ar = nullptr;
  int rc = arena_for(ctx, st, &ar);
  if (rc) return rc;
  rc = grow(ctx, (void**)&ar->acc, &ar->acc_B, B * ctx->dp);
  if (rc) return rc;
  const uint8_t* Qd = nullptr;
  int slot = -1;
  rc = stage_ring(ctx, *ar, ar->r_batch, shares, B * nb, st, &Qd, &slot);
  if (rc) return rc;
  // tensor cores for larger batches (the shares operand, B x r bytes, must fit)
  const bool want_tc = ctx->tc == 1 || (ctx->tc < 0 && B >= 32);
  if (want_tc) {
    rc = ens_batch_tc(ctx, *ar, Qd, B, st);
    if (rc) return rc;
  } else {
    const uint32_t QW = (uint32_t)((B + 31) / 32);
    rc = grow(ctx, (void**)&ar->Qt, &ar->Qt_bytes, ctx->r * QW * 4);
    if (rc) return rc;
    ENS_CUDA(ctx, cudaMemsetAsync(ar->acc, 0, B * ctx->dp, st));
    {
      dim3 grid((uint32_t)((ctx->r + 255) / 256), QW);
      ens_transpose_bits_kernel<<<grid, 256, 0, st>>>(Qd, ar->Qt, ctx->r, nb, (uint32_t)B, QW);
      ENS_LAUNCHED(ctx);
    }
    EnsBatchArgs a;
    a.R = ctx->R;
    a.Qt = ar->Qt;
    a.out = ar->acc;
    a.r = ctx->r;
    a.dp = (uint32_t)ctx->dp;
    a.W = (uint32_t)(ctx->dp / 16);
    a.QW = QW;
    a.B = (uint32_t)B;
    const uint32_t slices = (a.W + ENS_CW - 1) / ENS_CW;
    const uint32_t qblocks = (uint32_t)((B + ENS_QG * ENS_QB - 1) / (ENS_QG * ENS_QB));
    // enough CTAs for ~8 per SM, rows split evenly
    const uint64_t want = 8ull * ctx->num_sms;
    uint64_t splits = std::max<uint64_t>(1, (want + slices * qblocks - 1) / (slices * qblocks));
    uint64_t rows = ctx->rows_per_cta ? (uint64_t)ctx->rows_per_cta
                                      : std::min<uint64_t>(256, (ctx->r + splits - 1) / splits);
    rows = round_up(std::max<uint64_t>(rows, 4), 4);
    a.rows_per_cta = rows;
    dim3 grid((uint32_t)((ctx->r + rows - 1) / rows), slices, qblocks);
    ens_batch_kernel<<<grid, ENS_CW * ENS_QB, 0, st>>>(a);
    ENS_LAUNCHED(ctx);
    ctx->last_path = QPIR_ENS_PATH_CUDA_CORES;
  }
  if (slot >= 0) ENS_CUDA(ctx, cudaEventRecord(ar->r_batch.done[slot], st));
  return copy_out(ctx, *ar, out, B, st);
}

uint64_t qpir_ens_kernel_launches(const qpir_ens_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

int qpir_ens_last_path(const qpir_ens_ctx* ctx) {
  return ctx ? ctx->last_path.load() : QPIR_ENS_PATH_NONE;
}

const char* qpir_ens_last_error(const qpir_ens_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_ens_setup_error.c_str();
}

void qpir_ens_destroy(qpir_ens_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard dg(ctx->device);
  if (ctx->R) cudaFree(ctx->R);
  if (ctx->spec_stage) cudaFree(ctx->spec_stage);
  if (ctx->mldsa_buf) cudaFree(ctx->mldsa_buf);
  if (ctx->sig_stage) cudaFree(ctx->sig_stage);
  for (auto& kv : ctx->arenas) {
    EnsArena& a = kv.second;
    if (a.h2d) cudaStreamSynchronize(a.h2d);
    void* bufs[] = {a.acc, a.acc1, a.io_stage, a.Q_dev, a.Qt, a.seed_dev, a.partial, a.tickets, a.Qb};
    for (void* b : bufs)
      if (b) cudaFree(b);
    for (EnsRing* g : {&a.r_share, &a.r_q, &a.r_A, &a.r_batch})
      for (int k = 0; k < 2; ++k) {
        if (g->buf[k]) cudaFree(g->buf[k]);
        if (g->ready[k]) cudaEventDestroy(g->ready[k]);
        if (g->done[k]) cudaEventDestroy(g->done[k]);
      }
    if (a.h2d) cudaStreamDestroy(a.h2d);
  }
  delete ctx;
}

}  // extern "C"
