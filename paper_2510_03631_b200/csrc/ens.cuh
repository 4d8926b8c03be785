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

#include "ptx.cuh"

namespace qpir {

struct EnsArgs {
  const uint8_t* R;     // records [r][dp]
  const uint8_t* q;     // selector bits, bit t at byte t >> 3, bit t & 7
  uint32_t* out;        // dp / 4 words, zeroed, atomicXor target
  uint64_t r;           // rows
  uint32_t dp;          // row stride (multiple of 16)
  uint32_t W;           // 16-byte chunks per row
  uint64_t rows_per_cta;
};

template <int UR>
__global__ void __launch_bounds__(1024) ens_scan_kernel(EnsArgs a) {
  extern __shared__ uint4 s_part[];
  const uint32_t w = threadIdx.x % a.W;
  const uint32_t lr = threadIdx.x / a.W;
  const uint32_t R = blockDim.x / a.W;
  const uint64_t t0 = (uint64_t)blockIdx.x * a.rows_per_cta;
  const uint64_t t1 = min(a.r, t0 + a.rows_per_cta);
  uint4 acc = make_uint4(0, 0, 0, 0);
  const uint8_t* base = a.R + (size_t)w * 16;
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
  if (R > 1) {
    s_part[threadIdx.x] = acc;
    __syncthreads();
    if (lr != 0) return;
    for (uint32_t k = 1; k < R; ++k) {
      const uint4 p = s_part[k * a.W + w];
      acc.x ^= p.x;
      acc.y ^= p.y;
      acc.z ^= p.z;
      acc.w ^= p.w;
    }
  }
  uint32_t* o = a.out + (size_t)w * 4;
  if (acc.x) atomicXor(o + 0, acc.x);
  if (acc.y) atomicXor(o + 1, acc.y);
  if (acc.z) atomicXor(o + 2, acc.z);
  if (acc.w) atomicXor(o + 3, acc.w);
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
