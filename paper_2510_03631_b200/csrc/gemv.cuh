// gemv.cuh -- K-B1: the single-query answer ans = D . qu mod 2^32 (SURVEY 8(a)
// steps a2-a4; Def. 1 "DB.Query.Response"; the "q.DB mod q"
// contraction of Alg. 4 steps 14-15, with q = 2^32).
//
// HBM-bound: every byte of the D shard is read exactly once per query.
// D layout in HBM (DESIGN "Data layout"): 128-row panels of 16-cell interleaved
// column groups,
//   D[r][c] at ((r >> 7) * G + (c >> 4)) * 2048 + (r & 127) * 16 + (c & 15),
// so one thread's 128-bit load holds 16 consecutive cells of one row, a warp's
// load covers 32 consecutive rows = 512 contiguous bytes, and each panel is one
// contiguous stream of G * 2 KB that a CTA walks front to back.
//
// Query ingest (a2) is fused: each CTA splits its slice of qu into 4 byte-limb
// planes in shared memory, laid out so that one 32-bit word holds limb k of 4
// consecutive cells:  sL[g][k] = {limb_k(qu[16g+0..3]), ..., limb_k(qu[16g+12..15])}.
// Then for one row and one group of 16 cells (4 words d0..d3 of D):
//   sum_c D[r][c] qu[c] = sum_k 2^{8k} sum_w dp4a(d_w, sL[g][k].w)       (mod 2^32)
// -- 16 IDP4A per 16 bytes of D, no byte extraction, no cross-lane reduction;
// the four limb accumulators wrap mod 2^32 and are recombined at the end
// ((x mod 2^32) << 8k == x * 2^{8k} mod 2^32).
//
// Split-K (a4): blockIdx.y selects a range of column groups; partial sums go
// to a scratch buffer and the last CTA of each row block (atomic ticket) adds
// them -- u32 addition is associative, so the result is bit-identical for any
// split factor.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace qpir {

constexpr int GEMV_THREADS = 128;

// limb word k of the four u32 values a, b, c, e: bytes k of each, packed LE.
__device__ __forceinline__ uint32_t limb_word(uint32_t a, uint32_t b, uint32_t c, uint32_t e,
                                              uint32_t k) {
  const uint32_t sel = k | ((k + 4u) << 4);  // [a.k, b.k, -, -]
  uint32_t lo = __byte_perm(a, b, sel);
  uint32_t hi = __byte_perm(c, e, sel);
  return __byte_perm(lo, hi, 0x5410);        // [lo.0, lo.1, hi.0, hi.1]
}

// Stage limb planes of groups [g0, g1) into smem (sL[(g - g0) * 4 + k]).
__device__ __forceinline__ void stage_limbs(uint4* sL, const uint32_t* __restrict__ qu,
                                            uint32_t m, uint32_t g0, uint32_t g1) {
  for (uint32_t g = g0 + threadIdx.x; g < g1; g += blockDim.x) {
    uint32_t q[16];
    const uint32_t c0 = g * 16u;
    if (c0 + 16u <= m && ((reinterpret_cast<uintptr_t>(qu) & 15u) == 0)) {
      const uint4* p = reinterpret_cast<const uint4*>(qu + c0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 v = __ldg(p + i);
        q[4 * i + 0] = v.x;
        q[4 * i + 1] = v.y;
        q[4 * i + 2] = v.z;
        q[4 * i + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) q[i] = (c0 + i < m) ? __ldg(qu + c0 + i) : 0u;
    }
    uint4* dst = sL + (size_t)(g - g0) * 4;
#pragma unroll
    for (uint32_t k = 0; k < 4; ++k) {
      uint4 w;
      w.x = limb_word(q[0], q[1], q[2], q[3], k);
      w.y = limb_word(q[4], q[5], q[6], q[7], k);
      w.z = limb_word(q[8], q[9], q[10], q[11], k);
      w.w = limb_word(q[12], q[13], q[14], q[15], k);
      dst[k] = w;
    }
  }
}

__device__ __forceinline__ void dp4a_group(const uint4& d, const uint4& l0, const uint4& l1,
                                           const uint4& l2, const uint4& l3, uint32_t (&acc)[4]) {
  acc[0] = __dp4a(d.x, l0.x, acc[0]);
  acc[1] = __dp4a(d.x, l1.x, acc[1]);
  acc[2] = __dp4a(d.x, l2.x, acc[2]);
  acc[3] = __dp4a(d.x, l3.x, acc[3]);
  acc[0] = __dp4a(d.y, l0.y, acc[0]);
  acc[1] = __dp4a(d.y, l1.y, acc[1]);
  acc[2] = __dp4a(d.y, l2.y, acc[2]);
  acc[3] = __dp4a(d.y, l3.y, acc[3]);
  acc[0] = __dp4a(d.z, l0.z, acc[0]);
  acc[1] = __dp4a(d.z, l1.z, acc[1]);
  acc[2] = __dp4a(d.z, l2.z, acc[2]);
  acc[3] = __dp4a(d.z, l3.z, acc[3]);
  acc[0] = __dp4a(d.w, l0.w, acc[0]);
  acc[1] = __dp4a(d.w, l1.w, acc[1]);
  acc[2] = __dp4a(d.w, l2.w, acc[2]);
  acc[3] = __dp4a(d.w, l3.w, acc[3]);
}

struct GemvArgs {
  const uint8_t* D;     // [L/128][G][128][16]
  const uint32_t* qu;   // m (device)
  uint32_t* ans;        // ell_local (device)
  uint32_t* partial;    // [S][L] scratch (S > 1)
  uint32_t* tickets;    // [gridDim.x] zero-initialised, self-resetting
  uint32_t ell_local;   // rows to write
  uint32_t L;           // padded rows (stride of one split's partial vector)
  uint32_t m;           // columns (cells)
  uint32_t G;           // column groups (multiple of UNR)
  uint32_t gps;         // groups per split (multiple of UNR)
  uint32_t chunk;       // groups staged in smem at a time (multiple of UNR)
  uint32_t split_major; // 1: blockIdx.x = split, blockIdx.y = row block (page-local order)
  uint32_t pf256;       // 1: L2::256B prefetch hint on the D loads
  uint32_t l2pf;        // 1: bulk L2 prefetch of the CTA's D slice before griddepcontrol.wait
};

// U rows per thread (rows r, r + 128, ...); UNR column groups per iteration.
// EARLY: qu is not the previous kernel's output (see below); a separate
// instantiation, so its loop is the plain load-then-use loop (a runtime flag
// with the D loads hoisted out of the first iteration cost 5 % on C2).
template <int U, int UNR, bool EARLY>
__global__ void __launch_bounds__(GEMV_THREADS) qpir_gemv_u8_u32_kernel(GemvArgs a) {
  extern __shared__ uint4 sL[];
  // Programmatic dependent launch: the next query's GEMV may start while this
  // grid drains; only the previous kernel's writes are visible after
  // griddepcontrol.wait.  Before the wait a CTA touches only the D shard
  // (library-owned; right after a device-side db_write the GEMV is launched
  // without PDL, qpir.cu) -- unless EARLY: then qu is known not to come from
  // the previous kernel (staged by the library from host memory, or the caller
  // set QPIR_FLAG_STABLE_INPUTS) and the whole scan runs before the wait.
  // Every global write (partials, tickets, ans) comes after the wait.
  asm volatile("griddepcontrol.launch_dependents;");
  const uint32_t tid = threadIdx.x;
  // Grid order: with split_major the CTAs that run at the same time walk
  // adjacent K ranges of the same row panels, i.e. few distinct 2 MB pages.
  const uint32_t rblk = a.split_major ? blockIdx.y : blockIdx.x;
  const uint32_t split = a.split_major ? blockIdx.x : blockIdx.y;
  const uint32_t nsplit = a.split_major ? gridDim.x : gridDim.y;
  const uint32_t row0 = rblk * (GEMV_THREADS * U) + tid;
  const uint32_t gb = split * a.gps;
  const uint32_t ge = min(a.G, gb + a.gps);

  uint32_t acc[U][4];
#pragma unroll
  for (int u = 0; u < U; ++u) acc[u][0] = acc[u][1] = acc[u][2] = acc[u][3] = 0u;

  const uint8_t* Drow[U];
  bool live[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t r = row0 + u * GEMV_THREADS;
    live[u] = r < a.ell_local;  // rows >= ell_local are zero padding: skip
    Drow[u] = a.D + (size_t)(r >> 7) * a.G * 2048 + (r & 127u) * 16;
  }
  constexpr size_t gstride = 2048;
  auto load = [&](uint32_t g, uint4 (&d)[UNR][U]) {
#pragma unroll
    for (int i = 0; i < UNR; ++i)
#pragma unroll
      for (int u = 0; u < U; ++u)
        d[i][u] = !live[u] ? make_uint4(0, 0, 0, 0)
                  : a.pf256 ? ldg_stream_v4_pf256(Drow[u] + (size_t)(g + i) * gstride)
                            : ldg_stream_v4(Drow[u] + (size_t)(g + i) * gstride);
  };

  uint4 d[UNR][U];
  if constexpr (!EARLY) {
    // ---- before the wait: D only (first UNR groups in flight; optional bulk
    // L2 prefetch of the whole slice)
    if (a.l2pf && tid < U) {
      const uint32_t r = rblk * (GEMV_THREADS * U) + tid * GEMV_THREADS;
      if (r < a.ell_local)
        l2_prefetch_bulk(a.D + (size_t)(r >> 7) * a.G * 2048 + (size_t)gb * gstride,
                         (ge - gb) * (uint32_t)gstride);
    }
    load(gb, d);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // qu may be the previous grid's output
  }

  for (uint32_t cb = gb; cb < ge; cb += a.chunk) {
    const uint32_t ce = min(ge, cb + a.chunk);
    __syncthreads();
    stage_limbs(sL, a.qu, a.m, cb, ce);
    __syncthreads();
#pragma unroll 1
    for (uint32_t g = cb; g < ce; g += UNR) {
      if (EARLY || g != gb) load(g, d);
#pragma unroll
      for (int i = 0; i < UNR; ++i) {
        const uint4* l = sL + (size_t)(g + i - cb) * 4;
        const uint4 l0 = l[0], l1 = l[1], l2 = l[2], l3 = l[3];
#pragma unroll
        for (int u = 0; u < U; ++u) dp4a_group(d[i][u], l0, l1, l2, l3, acc[u]);
      }
    }
  }
  if constexpr (EARLY) asm volatile("griddepcontrol.wait;" ::: "memory");  // before any global write

  uint32_t out[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    out[u] = acc[u][0] + (acc[u][1] << 8) + (acc[u][2] << 16) + (acc[u][3] << 24);

  if (nsplit == 1) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t r = row0 + u * GEMV_THREADS;
      if (r < a.ell_local) a.ans[r] = out[u];
    }
    return;
  }

  // split-K: publish partials, last CTA of this row block reduces.
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t r = row0 + u * GEMV_THREADS;
    if (r < a.L) a.partial[(size_t)split * a.L + r] = out[u];
  }
  __threadfence();
  __shared__ uint32_t s_last;
  __syncthreads();
  if (tid == 0) {
    const uint32_t t = atomicAdd(&a.tickets[rblk], 1u);
    s_last = (t == nsplit - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t r = row0 + u * GEMV_THREADS;
    if (r < a.ell_local) {
      uint32_t s = 0;
      for (uint32_t k = 0; k < nsplit; ++k) s += __ldcg(a.partial + (size_t)k * a.L + r);
      a.ans[r] = s;
    }
  }
  if (tid == 0) a.tickets[rblk] = 0u;
}

}  // namespace qpir
