// ens.cuh -- NEXT-1: QPADL-ENS (Chor XOR PIR) server kernels on sm_100a.
//
// PIR.Query.Response for ENS (Lemma 1 proof; Alg. 3
// "Multi-request Parallel Chor-PIR"): the response to an r-bit
// share q is the XOR of the records theta with q[theta] = 1 (GF(2) product
// q . DB, DB = r rows of b = 8d bits).  HBM-bound: work W = nnz(q) * b and
// traffic ~ nnz(q) * b, so unselected rows are not read (the paper's
// conditional row fetch, Alg. 3 step 9 / P:1012-1013).
//
// Records live theta-major with a 16-byte padded row stride dp.  One thread
// owns one 16-byte chunk of the row width; a CTA walks a contiguous range of
// rows (blockDim = W * R threads, R rows per step), XOR-accumulating 128-bit
// loads of selected rows; partials fold through shared memory and land in
// the output with u32 atomicXor (XOR is associative and commutative, so the
// result is bit-identical for any grid).
//
// Multi-request form: a CTA owns a 32-chunk (512 B) column slice x 64
// queries (8 query groups of 8); every thread keeps 8 XOR accumulators and
// folds each row chunk in under an all-ones/zero mask built from the query's
// selector bit (LOP3 acc ^= chunk & mask): no divergence, one HBM read of the
// row slice per 64 queries (the other query groups of the CTA hit L1).
#pragma once
#include <cstdint>

#include "layout.cuh"
#include "philox.cuh"
#include "ptx.cuh"

namespace qpir {

struct EnsArgs {
  const uint8_t* R;     // records [r][dp]
  const uint8_t* q;     // selector bits for rows [row_lo, row_hi): bit (t - row_lo)
  uint32_t* out;        // dp / 4 words, pre-initialised (zero, or OOP's A), atomicXor target
  uint64_t row_lo, row_hi;  // scanned row range (whole DB: [0, r))
  uint32_t dp;          // row stride (multiple of 16)
  uint32_t W;           // 16-byte chunks per row
  uint64_t rows_per_cta;
  uint4* partial;       // [gridDim.x][W] CTA partials (group reduction), or nullptr
  uint32_t* tickets;    // [ceil(grid / group)] zero-initialised, self-resetting
  uint32_t group;       // CTAs per reduction group
  // In-kernel finalisation (single-share answer / OOP online): the last CTA to
  // finish its atomics writes fin_out[i] = out[i] ^ init[i] (i < d bytes) and
  // re-zeroes `out` and `done`, so a call is one kernel with no memset or
  // copies around it.  fin_out == nullptr: the result stays in `out`.
  uint8_t* fin_out;
  const uint8_t* init;  // XORed into the result (OOP's A_i), or nullptr
  uint32_t d;           // record bytes
  uint32_t* done;       // zero-initialised, self-resetting
  uint32_t leaders;     // CTAs that reach the atomics (grid, or groups)
  uint32_t early;       // 1: the share is not the previous kernel's output: scan before the PDL wait
};

// Called by every thread of a CTA that has just added its partial into a.out.
__device__ __forceinline__ void ens_finalize(const EnsArgs& a) {
  if (a.fin_out == nullptr) return;
  __shared__ uint32_t s_fin;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_fin = (atomicAdd(a.done, 1u) == a.leaders - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_fin) return;
  __threadfence();
  for (uint32_t i = threadIdx.x; i < a.dp / 4; i += blockDim.x) {
    const uint32_t v = __ldcg(a.out + i);  // every CTA's atomics, resolved at L2
    a.out[i] = 0u;
#pragma unroll
    for (uint32_t b = 0; b < 4; ++b) {
      const uint32_t k = 4 * i + b;
      if (k < a.d) {
        uint8_t x = (uint8_t)(v >> (8 * b));
        if (a.init) x ^= a.init[k];
        a.fin_out[k] = x;
      }
    }
  }
  if (threadIdx.x == 0) *a.done = 0u;
}

template <int UR>
__global__ void __launch_bounds__(1024, 1) ens_scan_kernel(EnsArgs a) {
  asm volatile("griddepcontrol.launch_dependents;");  // PDL: see ens_scan_wide_kernel
  if (!a.early) asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ uint4 s_part[];
  const uint32_t w = threadIdx.x % a.W;
  const uint32_t lr = threadIdx.x / a.W;
  const uint32_t R = blockDim.x / a.W;
  // t counts rows relative to row_lo (= the selector bit index)
  const uint64_t n_rows = a.row_hi - a.row_lo;
  const uint64_t t0 = (uint64_t)blockIdx.x * a.rows_per_cta;
  const uint64_t t1 = min(n_rows, t0 + a.rows_per_cta);
  uint4 acc = make_uint4(0, 0, 0, 0);
  const uint8_t* base = a.R + (size_t)a.row_lo * a.dp + (size_t)w * 16;
  for (uint64_t t = t0 + lr; t < t1; t += (uint64_t)R * UR) {
    // all selector bytes first (L1 hits), then all row loads, predicated
    uint32_t qb[UR];
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const uint64_t tt = t + (uint64_t)u * R;
      qb[u] = tt < t1 ? (uint32_t)__ldg(a.q + (tt >> 3)) : 0u;
    }
    uint4 v[UR];
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const uint64_t tt = t + (uint64_t)u * R;
      v[u] = ldg_stream_v4_if(base + tt * a.dp, (qb[u] >> (tt & 7)) & 1u);
    }
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      acc.x ^= v[u].x;
      acc.y ^= v[u].y;
      acc.z ^= v[u].z;
      acc.w ^= v[u].w;
    }
  }
  if (a.early) asm volatile("griddepcontrol.wait;" ::: "memory");  // before any global write
  const bool owner = lr == 0;  // one thread per 16-byte chunk keeps the CTA result
  if (R > 1) {
    s_part[threadIdx.x] = acc;
    __syncthreads();
    if (owner) {
      for (uint32_t k = 1; k < R; ++k) {
        const uint4 p = s_part[k * a.W + w];
        acc.x ^= p.x;
        acc.y ^= p.y;
        acc.z ^= p.z;
        acc.w ^= p.w;
      }
    }
  }
  if (a.partial != nullptr) {
    // two-level reduction: publish the CTA partial; the last CTA of each group
    // of `group` CTAs folds the group's partials and does the atomics.
    __shared__ uint32_t s_last;
    if (owner) a.partial[(size_t)blockIdx.x * a.W + w] = acc;
    __threadfence();
    __syncthreads();
    const uint32_t grp = blockIdx.x / a.group;
    const uint32_t g0 = grp * a.group;
    const uint32_t g1 = min(gridDim.x, g0 + a.group);
    if (threadIdx.x == 0) {
      const uint32_t t = atomicAdd(&a.tickets[grp], 1u);
      s_last = (t == g1 - g0 - 1) ? 1u : 0u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (owner) {
      acc = make_uint4(0, 0, 0, 0);
      for (uint32_t c = g0; c < g1; ++c) {
        const uint4 p = __ldcg(a.partial + (size_t)c * a.W + w);
        acc.x ^= p.x;
        acc.y ^= p.y;
        acc.z ^= p.z;
        acc.w ^= p.w;
      }
    }
    if (threadIdx.x == 0) a.tickets[grp] = 0u;
  }
  if (owner) {
    uint32_t* o = a.out + (size_t)w * 4;
    if (acc.x) atomicXor(o + 0, acc.x);
    if (acc.y) atomicXor(o + 1, acc.y);
    if (acc.z) atomicXor(o + 2, acc.z);
    if (acc.w) atomicXor(o + 3, acc.w);
  }
  ens_finalize(a);
}

// Wide-record variant (one row per CTA step: d > 2 KB, e.g. the paper's 3 KB
// records).  The row is warp-uniform, so the selector bit is tested once per
// row from a 32-row word loaded once (CTA ranges start on 32-row boundaries
// relative to row_lo, the share's bit 0), the row pointer advances by dp, and
// unselected rows issue no load at all: ~8 instructions per chunk instead of
// ~20 for the general kernel.  CW = 16-byte chunks per thread (blockDim =
// W / CW): CW = 2 uses 256-bit loads, doubling the bytes each thread has in
// flight (measured slower than CW = 1: opt-in, QPIR_ENS_WIDE=2).  The launch
// bounds (1024, 1) let ptxas spend 64 registers and keep ~11 row loads in
// flight per thread; under plain (1024) it packed into 32 registers and issued
// the loads two at a time (SASS), latency-bound at 0.61-0.90 of HBM.
// Programmatic dependent launch: the next scan's CTAs become resident while this
// grid drains.  The share decides which rows of R are read, so unless it is
// known not to be the previous kernel's output (a.early: staged by the library
// from host memory, or QPIR_FLAG_STABLE_INPUTS) every read waits at
// griddepcontrol.wait; with a.early the scan overlaps the previous grid's tail
// and only the partials / tickets / out writes wait.
template <int UR, int CW>
__global__ void __launch_bounds__(1024, 1) ens_scan_wide_kernel(EnsArgs a) {
  asm volatile("griddepcontrol.launch_dependents;");
  if (!a.early) asm volatile("griddepcontrol.wait;" ::: "memory");  // previous grid complete + visible
  const uint32_t w = threadIdx.x * CW;  // first 16-byte chunk of this thread
  const uint64_t n_rows = a.row_hi - a.row_lo;
  const uint64_t t0 = (uint64_t)blockIdx.x * a.rows_per_cta;  // multiple of 32
  const uint64_t t1 = min(n_rows, t0 + a.rows_per_cta);
  const uint32_t* q32 = reinterpret_cast<const uint32_t*>(a.q);  // 4-byte aligned
  uint4 acc[CW];
#pragma unroll
  for (int c = 0; c < CW; ++c) acc[c] = make_uint4(0, 0, 0, 0);
  for (uint64_t tb = t0; tb < t1; tb += 32) {
    uint32_t sel = __ldg(q32 + (tb >> 5));
    const uint32_t nrow = (t1 - tb) < 32 ? (uint32_t)(t1 - tb) : 32u;
    if (nrow < 32) sel &= (1u << nrow) - 1u;
    const uint8_t* p = a.R + (size_t)(a.row_lo + tb) * a.dp + (size_t)w * 16;
#pragma unroll
    for (int h = 0; h < 32; h += UR) {
      uint4 v[UR][CW];
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const bool on = (sel >> (h + u)) & 1u;
        if constexpr (CW == 2)
          ldg_stream_v8_if(p + (size_t)(h + u) * a.dp, on, v[u][0], v[u][1]);
        else
          v[u][0] = ldg_stream_v4_if(p + (size_t)(h + u) * a.dp, on);
      }
#pragma unroll
      for (int u = 0; u < UR; ++u)
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          acc[c].x ^= v[u][c].x;
          acc[c].y ^= v[u][c].y;
          acc[c].z ^= v[u][c].z;
          acc[c].w ^= v[u][c].w;
        }
    }
  }
  if (a.early) asm volatile("griddepcontrol.wait;" ::: "memory");  // before any global write
  if (a.partial != nullptr) {
    __shared__ uint32_t s_last;
#pragma unroll
    for (int c = 0; c < CW; ++c) a.partial[(size_t)blockIdx.x * a.W + w + c] = acc[c];
    __threadfence();
    __syncthreads();
    const uint32_t grp = blockIdx.x / a.group;
    const uint32_t g0 = grp * a.group;
    const uint32_t g1 = min(gridDim.x, g0 + a.group);
    if (threadIdx.x == 0) {
      const uint32_t t = atomicAdd(&a.tickets[grp], 1u);
      s_last = (t == g1 - g0 - 1) ? 1u : 0u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
#pragma unroll
    for (int c = 0; c < CW; ++c) acc[c] = make_uint4(0, 0, 0, 0);
    for (uint32_t g = g0; g < g1; ++g) {
#pragma unroll
      for (int c = 0; c < CW; ++c) {
        const uint4 v = __ldcg(a.partial + (size_t)g * a.W + w + c);
        acc[c].x ^= v.x;
        acc[c].y ^= v.y;
        acc[c].z ^= v.z;
        acc[c].w ^= v.w;
      }
    }
    if (threadIdx.x == 0) a.tickets[grp] = 0u;
  }
#pragma unroll
  for (int c = 0; c < CW; ++c) {
    uint32_t* o = a.out + (size_t)(w + c) * 4;
    if (acc[c].x) atomicXor(o + 0, acc[c].x);
    if (acc[c].y) atomicXor(o + 1, acc[c].y);
    if (acc[c].z) atomicXor(o + 2, acc[c].z);
    if (acc[c].w) atomicXor(o + 3, acc[c].w);
  }
  ens_finalize(a);
}

// Selector bits transposed for the batch: Qt[t][k] bit i = share (32k + i) bit t.
__global__ void ens_transpose_bits_kernel(const uint8_t* __restrict__ Q, uint32_t* __restrict__ Qt,
                                          uint64_t r, uint64_t nb, uint32_t B, uint32_t QW) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t k = blockIdx.y;
  if (t >= r) return;
  uint32_t word = 0;
#pragma unroll 4
  for (uint32_t i = 0; i < 32; ++i) {
    const uint32_t qi = k * 32 + i;
    if (qi < B) word |= (uint32_t)((__ldg(Q + (size_t)qi * nb + (t >> 3)) >> (t & 7)) & 1u) << i;
  }
  Qt[t * QW + k] = word;
}

constexpr uint32_t ENS_CW = 32;  // chunks (16 B) per column slice
constexpr uint32_t ENS_QG = 8;   // queries per thread
constexpr uint32_t ENS_QB = 8;   // query groups per CTA (64 queries)

struct EnsBatchArgs {
  const uint8_t* R;    // [r][dp]
  const uint32_t* Qt;  // [r][QW]
  uint32_t* out;       // [B][dp / 4], zeroed
  uint64_t r;
  uint32_t dp, W, QW, B;
  uint64_t rows_per_cta;
};

__global__ void __launch_bounds__(ENS_CW* ENS_QB) ens_batch_kernel(EnsBatchArgs a) {
  const uint32_t w = blockIdx.y * ENS_CW + threadIdx.x % ENS_CW;
  const uint32_t qg = blockIdx.z * ENS_QB + threadIdx.x / ENS_CW;  // query group
  const uint32_t q0 = qg * ENS_QG;
  const uint64_t t0 = (uint64_t)blockIdx.x * a.rows_per_cta;
  const uint64_t t1 = min(a.r, t0 + a.rows_per_cta);
  if (q0 >= a.B) return;
  const bool wok = w < a.W;
  uint4 acc[ENS_QG];
#pragma unroll
  for (int i = 0; i < (int)ENS_QG; ++i) acc[i] = make_uint4(0, 0, 0, 0);
  const uint8_t* base = a.R + (size_t)w * 16;
  const uint32_t* qt = a.Qt + (q0 >> 5);
  const uint32_t sh = q0 & 31u;
  constexpr int UR = 4;
  for (uint64_t t = t0; t < t1; t += UR) {
    uint4 v[UR];
    uint32_t bits[UR];
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const uint64_t tt = t + u;
      const bool ok = tt < t1;
      v[u] = (ok && wok) ? __ldg(reinterpret_cast<const uint4*>(base + tt * a.dp))
                         : make_uint4(0, 0, 0, 0);
      bits[u] = ok ? (__ldg(qt + tt * a.QW) >> sh) : 0u;
    }
#pragma unroll
    for (int u = 0; u < UR; ++u) {
#pragma unroll
      for (int i = 0; i < (int)ENS_QG; ++i) {
        if (bits[u] & (1u << i)) {  // predicated XOR (no mask arithmetic)
          acc[i].x ^= v[u].x;
          acc[i].y ^= v[u].y;
          acc[i].z ^= v[u].z;
          acc[i].w ^= v[u].w;
        }
      }
    }
  }
  if (!wok) return;
  const uint32_t wpr = a.dp / 4;  // words per output row
#pragma unroll
  for (int i = 0; i < (int)ENS_QG; ++i) {
    if (q0 + i >= a.B) break;
    uint32_t* o = a.out + (size_t)(q0 + i) * wpr + (size_t)w * 4;
    if (acc[i].x) atomicXor(o + 0, acc[i].x);
    if (acc[i].y) atomicXor(o + 1, acc[i].y);
    if (acc[i].z) atomicXor(o + 2, acc[i].z);
    if (acc[i].w) atomicXor(o + 3, acc[i].w);
  }
}

}  // namespace qpir

namespace qpir {
// ---------------------------------------------------------------- NEXT-3 OOP
// CIP-PIR offline expansion (P:930 steps 1-2; DESIGN R19): for each seed S,
// the full B-bit selector over the DB: 0 on server i's flip chunk, and on the
// non-flip chunks (rotated order chunk_{i+1}, ..., chunk_{i+n-1}) bit p of
// PRG(S) -- word w of PRG(S) = Philox(key = S, ctr = (w >> 2, 0, 0, 'O'))[w & 3].
// One thread per (seed, output byte).  Output: n_seeds x ceil(B/8) bytes, the
// shares of the ENS batch kernel that then computes A = q . DB.
__global__ void oop_expand_kernel(const unsigned long long* __restrict__ seeds, uint8_t* __restrict__ out,
                                  uint64_t B, uint64_t k, uint32_t n, uint32_t i, uint64_t nb) {
  const uint64_t byte = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t sidx = blockIdx.y;
  if (byte >= nb) return;
  const unsigned long long seed = seeds[sidx];
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  uint32_t v = 0;
  uint64_t cached_blk = ~0ull;
  uint4 words = make_uint4(0, 0, 0, 0);
  for (uint32_t b = 0; b < 8; ++b) {
    const uint64_t blk = byte * 8 + b;
    if (blk >= B) break;
    const uint64_t chunk = blk / k;
    if (chunk == i) continue;                        // flip chunk: online only
    const uint64_t rot = (chunk + n - i - 1) % n;    // position among non-flip chunks
    const uint64_t p = rot * k + blk % k;
    const uint64_t w = p >> 5;
    if ((w >> 2) != cached_blk) {
      cached_blk = w >> 2;
      words = philox4x32_10(make_uint4((uint32_t)cached_blk, 0u, 0u, 0x4Fu), key);
    }
    const uint32_t word = (w & 3) == 0 ? words.x : (w & 3) == 1 ? words.y : (w & 3) == 2 ? words.z : words.w;
    v |= ((word >> (p & 31)) & 1u) << b;
  }
  out[(size_t)sidx * nb + byte] = (uint8_t)v;
}
}  // namespace qpir

namespace qpir {
// ---------------------------------------------------------------- ENS on tensor cores
// Shares as a tensor-core operand (ens_mma.cuh): byte (share q, record theta) =
// bit theta of share q (0/1), in BN-row panels [Npad/BN][G16][BN][16] (K-major,
// 16 records per 16-byte row).  One thread per (q, 16-record group).
__global__ void ens_share_expand_kernel(const uint8_t* __restrict__ Q, uint32_t B, uint64_t r,
                                        uint64_t nb, uint8_t* __restrict__ Qb, uint32_t G,
                                        uint32_t Npad, uint32_t BN) {
  // Share slot fastest: consecutive threads write consecutive 16-byte columns of
  // one group (coalesced runs of BN * 16 bytes -- the 8x-expanded output is the
  // traffic that matters); their 2-byte share reads hit the L2-resident shares.
  // grid.x = blocks of share slots, grid.y / grid.z = 16-record groups
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t g = blockIdx.y + blockIdx.z * gridDim.y;
  if (q >= Npad || g >= G) return;
  uint32_t bits = 0;
  if (q < B) {
    const uint64_t b0 = (uint64_t)g * 2;
    if (b0 < nb) bits = __ldg(Q + (size_t)q * nb + b0);
    if (b0 + 1 < nb) bits |= (uint32_t)__ldg(Q + (size_t)q * nb + b0 + 1) << 8;
    const uint64_t t0 = (uint64_t)g * 16;
    if (t0 + 16 > r) bits &= (t0 >= r) ? 0u : ((1u << (r - t0)) - 1u);
  }
  uint32_t w[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const uint32_t nib = (bits >> (4 * t)) & 0xFu;
    w[t] = (nib & 1u) | ((nib >> 1) & 1u) << 8 | ((nib >> 2) & 1u) << 16 | ((nib >> 3) & 1u) << 24;
  }
  *reinterpret_cast<uint4*>(Qb + limb_off(q, g, G, BN)) = make_uint4(w[0], w[1], w[2], w[3]);
}
}  // namespace qpir
