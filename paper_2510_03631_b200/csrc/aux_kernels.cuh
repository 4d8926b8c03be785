// aux_kernels.cuh -- K-B4 helpers: DB pack (step a1), batch-query limb split
// (a6 prologue), Philox expansion of the public matrix A into limb planes (a7).
#pragma once
#include <cstdint>

#include "layout.cuh"
#include "mma.cuh"
#include "philox.cuh"

namespace qpir {

// ---------------------------------------------------------------- a1 pack
// Records theta in [theta0, theta0 + n_rec) (theta-ordered, d bytes each) are
// scattered into the D shard.  Geometry (DESIGN R9/R10; PAPER.md:515 DB matrix,
// SPEC.md:51 row-major index, PAPER.md:1107 multiple-block retrieval):
//   theta = cell * n_ch + ch,  blk = cell / m,  col = cell % m,
//   row = (blk * n_ch + ch) * d + b.
// One thread = one (local row, 16-column group): read-modify-write of 16 bytes.
// Lanes walk consecutive rows = consecutive record bytes, so the record reads
// coalesce and the 16-byte writes are contiguous.
struct PackArgs {
  const uint8_t* rec;
  uint8_t* D;          // 128-row panels: [L/128][G][128][16]
  uint64_t theta0, n_rec;
  uint64_t row_begin;  // global row of local row 0
  uint32_t ell_local, L;
  uint32_t n_ch, d, m;
  uint64_t n_cells;
  uint32_t g_lo;       // first column group of the launch (grid.x offset)
  uint32_t G;          // column groups per panel
};

__global__ void pack_records_kernel(PackArgs a) {
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
  uint4 v = *dst;
  uint8_t* bytes = reinterpret_cast<uint8_t*>(&v);
  bool touched = false;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t col = j * 16u + i;
    if (col >= a.m) continue;
    const uint64_t cell = blk * a.m + col;
    if (cell >= a.n_cells) continue;
    const uint64_t theta = cell * a.n_ch + ch;
    if (theta < a.theta0 || theta >= a.theta0 + a.n_rec) continue;
    bytes[i] = a.rec[(theta - a.theta0) * a.d + b];
    touched = true;
  }
  if (touched) *dst = v;
}

// ---------------------------------------------------------------- a6 limbs
// Q (B x m u32, query-major) -> Q' = byte-limb planes as the MMA B operand,
// K-major, 16-cell interleaved like D, in BN-column panels:
//   byte i of (limb column n, group g) at ((n / BN) * G + g) * BN * 16 + (n % BN) * 16 + i
//   = limb k of Q[j][16g + i], n = 4j + k (k = 0..3); zero for padding
// (n >= 4B or 16g + i >= m).  One MMA B tile (BN columns x 8 groups) is then
// BN * 128 contiguous bytes.  One thread per (group g, query j): 64 B in,
// 4 x 16 B out (64 B contiguous).
// LPQ limbs per query (4 for Z_{2^32}; 3 for F_p with p < 2^24 after reducing
// each entry mod p -- exact, since sum (q mod p) d = sum q d (mod p)).
// LPQ = 2 (p <= 65537): a reduced entry 65536 (only p = 65537) is written as 0
// and its column appended to the query's exception list (exc_cnt / exc_list,
// `cap` entries per query) for modp_fixup_kernel.
// fastmod_u32: mma.cuh (shared with the fused split of the tcgen05 engine).
template <int LPQ>
__global__ void limb_split_kernel(const uint32_t* __restrict__ Q, uint8_t* __restrict__ Qp,
                                  uint32_t B, uint32_t m, uint32_t G, uint32_t Npad,
                                  uint32_t BN, uint32_t p, uint64_t pM,
                                  uint32_t* __restrict__ exc_cnt,
                                  uint32_t* __restrict__ exc_list, uint32_t cap) {
  // threads walk 16-cell groups of one query row (coalesced 64 B per thread);
  // each thread writes its query's LPQ limb rows = 16 * LPQ contiguous bytes
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t jq = blockIdx.y;  // padded query index
  if (g >= G || jq * (uint32_t)LPQ >= Npad) return;
  uint32_t q[16];
  const uint32_t c0 = g * 16u;
  const uint32_t* row = Q + (size_t)jq * m;
  if (jq < B && c0 + 16u <= m && (m & 3u) == 0 &&
      (reinterpret_cast<uintptr_t>(Q) & 15u) == 0) {
    const uint4* p = reinterpret_cast<const uint4*>(row + c0);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 v = __ldg(p + i);
      q[4 * i + 0] = v.x;
      q[4 * i + 1] = v.y;
      q[4 * i + 2] = v.z;
      q[4 * i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) q[i] = (jq < B && c0 + i < m) ? __ldg(row + c0 + i) : 0u;
  }
  if (p != 0) {
#pragma unroll
    for (int i = 0; i < 16; ++i) q[i] = fastmod_u32(q[i], pM, p);
    if constexpr (LPQ == 2) {
      if (exc_cnt) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (q[i] == 65536u) {  // jq < B and c0 + i < m: padding entries are 0
            const uint32_t idx = atomicAdd(exc_cnt + jq, 1u);
            if (idx < cap) exc_list[(size_t)jq * cap + idx] = c0 + i;
            q[i] = 0u;
          }
      }
    }
  }
  uint4* dst = reinterpret_cast<uint4*>(Qp + limb_off(jq * (uint32_t)LPQ, g, G, BN));
#pragma unroll
  for (uint32_t k = 0; k < (uint32_t)LPQ; ++k) {
    const uint32_t sel = k | ((k + 4) << 4);
    uint4 w;
    w.x = __byte_perm(__byte_perm(q[0], q[1], sel), __byte_perm(q[2], q[3], sel), 0x5410);
    w.y = __byte_perm(__byte_perm(q[4], q[5], sel), __byte_perm(q[6], q[7], sel), 0x5410);
    w.z = __byte_perm(__byte_perm(q[8], q[9], sel), __byte_perm(q[10], q[11], sel), 0x5410);
    w.w = __byte_perm(__byte_perm(q[12], q[13], sel), __byte_perm(q[14], q[15], sel), 0x5410);
    dst[k] = w;
  }
}

// ---------------------------------------------------------------- a7 A'
// A' (same panel layout as Q') = limb k of A[16g + i][j], n = 4j + k.  Four
// lanes share one (group g, Philox block jb = j >> 2): lane `sub` runs the 4
// Philox calls of cells 16g + 4sub .. + 3 and writes, for each of the 16 limb
// columns of the block, its 4-byte quarter of the 16-byte chunk (the 4 lanes
// together write whole chunks).  16 registers of A per lane instead of 64 keeps
// occupancy high enough to hide the Philox latency chains.
__global__ void __launch_bounds__(256) expand_A_limbs_kernel(
    uint8_t* __restrict__ Ap, uint64_t seed, uint32_t m, uint32_t n, uint32_t G, uint32_t Npad,
    uint32_t BN, uint32_t j_off) {
  // grid.x = column groups (up to 2^31), grid.y = blocks of 64 Philox blocks;
  // this launch generates hint columns j_off .. j_off + Npad/4 - 1 (j_off % 4 == 0)
  const uint32_t sub = threadIdx.x & 3u;
  const uint32_t jb = blockIdx.y * (blockDim.x / 4) + threadIdx.x / 4;
  const uint32_t g = blockIdx.x;
  if (jb * 16u >= Npad) return;
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  const uint32_t jg = j_off + jb * 4u;  // global column of this Philox block
  uint32_t a[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t c = g * 16u + sub * 4u + i;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (c < m && jg < n) v = philox4x32_10(make_uint4(c, jg >> 2, 0u, 0x41u), key);
    a[i][0] = v.x;
    a[i][1] = (jg + 1 < n) ? v.y : 0u;
    a[i][2] = (jg + 2 < n) ? v.z : 0u;
    a[i][3] = (jg + 3 < n) ? v.w : 0u;
  }
  uint32_t* dst = reinterpret_cast<uint32_t*>(Ap + limb_off(jb * 16u, g, G, BN)) + sub;
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
#pragma unroll
    for (uint32_t k = 0; k < 4; ++k) {
      const uint32_t sel = k | ((k + 4) << 4);
      dst[(jj * 4 + k) * 4] = __byte_perm(__byte_perm(a[0][jj], a[1][jj], sel),
                                          __byte_perm(a[2][jj], a[3][jj], sel), 0x5410);
    }
  }
}

}  // namespace qpir
