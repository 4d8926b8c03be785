// mma.cuh -- K-B2/K-B3: the batched answer ANS = D . Q and the hint H = D . A,
// both mod 2^32, as a u8 x u8 -> s32 tcgen05 GEMM over byte limbs (SURVEY 8(a)
// steps a6/a7; multi-request GEMM of Alg. 4; offline
// precomputation).
//
// 32-bit right operands are split into 4 byte limbs (Q' / A', built by
// aux_kernels.cuh) so that  C = D . Q'  is an exact u8 x u8 GEMM with s32
// accumulation (no saturation: the idesc saturate bit is 0, sums wrap mod 2^32)
// and the epilogue recombines  ANS[:, j] = sum_k 2^{8k} C[:, 4j + k]  mod 2^32.
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0     : producer -- 1-D bulk async copies (TMA engine) of the A tile
//                (128 rows of D) and the B tile (BN limb columns) per K-block of
//                128 bytes into a STAGES-deep smem ring, mbarrier complete_tx.
//   warp 1     : TMEM allocator + MMA issuer -- one thread issues
//                tcgen05.mma.cta_group::1.kind::i8 (M=128, N=BN, K=32) x 4 per
//                K-block into a double-buffered TMEM accumulator, tcgen05.commit
//                frees smem stages and signals the epilogue.
//   warps 2..5 : epilogue -- tcgen05.ld 32 lanes x 16 columns, limb recombine,
//                coalesced u32 stores; then release the accumulator buffer.
// Shared-memory operand layout = the global layout (16-cell interleave):
// [8 groups][rows][16 B], i.e. the canonical no-swizzle K-major layout with
// core matrices of 8 rows x 16 B contiguous (SBO = 128 B between 8-row core
// matrices, LBO = rows * 16 B between the two 16-byte K chunks of one MMA).
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace qpir {

constexpr uint32_t MMA_BM = 128;      // rows of D per tile (UMMA M)
constexpr uint32_t MMA_BK = 128;      // K bytes (cells) per pipeline stage
constexpr uint32_t MMA_GPB = MMA_BK / 16;  // column groups per stage (8)
constexpr uint32_t MMA_THREADS = 192;

enum : int { OUT_QUERY_MAJOR = 0, OUT_ROW_MAJOR = 1 };

struct MmaArgs {
  const uint8_t* A;   // D shard [G][L][16]
  const uint8_t* B;   // limbs   [G][Npad][16]
  uint32_t* out;
  uint32_t L;         // padded rows of D (multiple of 128)
  uint32_t Npad;      // padded limb columns (multiple of BN)
  uint32_t G;         // column groups (multiple of 8)
  uint32_t rows;      // valid output rows (ell_local)
  uint32_t n_out;     // valid outputs along N (queries B, or hint width n)
  uint32_t out_ld;    // query-major: ell_local; row-major: n
  uint32_t m_tiles, n_tiles;
};

template <uint32_t BN, uint32_t STAGES>
struct MmaSmem {
  static constexpr uint32_t A_BYTES = MMA_BM * MMA_BK;  // 16 KB
  static constexpr uint32_t B_BYTES = BN * MMA_BK;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t BAR_OFF = STAGES * STAGE_BYTES;
  // full[STAGES], empty[STAGES], tfull[2], tempty[2], tmem addr
  static constexpr uint32_t TOTAL = BAR_OFF + (2 * STAGES + 4) * 8 + 16;
  static constexpr uint32_t TMEM_COLS = (2 * BN < 32) ? 32 : 2 * BN;
};

template <uint32_t BN, uint32_t STAGES, int OUT_MODE>
__global__ void __launch_bounds__(MMA_THREADS, 1) mma_u8_limb_kernel(MmaArgs a) {
  using S = MmaSmem<BN, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = threadIdx.x / 32;
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t num_tiles = a.m_tiles * a.n_tiles;
  const uint32_t kblocks = a.G / MMA_GPB;

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4 * 32);
    }
    fence_mbarrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, S::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (uint32_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const uint32_t mt = tile / a.n_tiles, nt = tile % a.n_tiles;
        const uint8_t* srcA = a.A + (size_t)mt * MMA_BM * 16;
        const uint8_t* srcB = a.B + (size_t)nt * BN * 16;
        for (uint32_t kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], S::STAGE_BYTES);
          uint8_t* dA = smem + stage * S::STAGE_BYTES;
          uint8_t* dB = dA + S::A_BYTES;
#pragma unroll
          for (uint32_t i = 0; i < MMA_GPB; ++i) {
            const size_t g = (size_t)kb * MMA_GPB + i;
            bulk_g2s(dA + i * (MMA_BM * 16), srcA + g * a.L * 16, MMA_BM * 16, &full[stage]);
            bulk_g2s(dB + i * (BN * 16), srcB + g * a.Npad * 16, BN * 16, &full[stage]);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_i8_u8u8_s32(MMA_BM, BN);
    uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
    for (uint32_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (uint32_t kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sA = smem_u32(smem + stage * S::STAGE_BYTES);
          const uint32_t sB = sA + S::A_BYTES;
#pragma unroll
          for (uint32_t k = 0; k < MMA_BK / 32; ++k) {
            const uint64_t da = smem_desc_noswizzle(sA + k * 2 * (MMA_BM * 16), MMA_BM * 16, 128);
            const uint64_t db = smem_desc_noswizzle(sB + k * 2 * (BN * 16), BN * 16, 128);
            mma_i8_ss(d_tmem, da, db, idesc, (kb | k) != 0u);
          }
          mma_commit(&empty[stage]);
          if (kb + 1 == kblocks) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
    uint32_t acc = 0, acc_phase = 0;
    for (uint32_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const uint32_t mt = tile / a.n_tiles, nt = tile % a.n_tiles;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t row = mt * MMA_BM + q * 32 + lane;
      const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * BN;
#pragma unroll 1
      for (uint32_t c0 = 0; c0 < BN; c0 += 16) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(taddr + c0, v);
        const uint32_t j0 = (nt * BN + c0) / 4;  // first output (query / hint column)
        uint32_t o[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          o[jj] = v[4 * jj] + (v[4 * jj + 1] << 8) + (v[4 * jj + 2] << 16) + (v[4 * jj + 3] << 24);
        if (row < a.rows) {
          if (OUT_MODE == OUT_QUERY_MAJOR) {
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
              if (j0 + jj < a.n_out) a.out[(size_t)(j0 + jj) * a.out_ld + row] = o[jj];
          } else {
            uint32_t* dst = a.out + (size_t)row * a.out_ld + j0;
            if (j0 + 4 <= a.n_out && (a.out_ld & 3u) == 0) {
              *reinterpret_cast<uint4*>(dst) = make_uint4(o[0], o[1], o[2], o[3]);
            } else {
#pragma unroll
              for (int jj = 0; jj < 4; ++jj)
                if (j0 + jj < a.n_out) dst[jj] = o[jj];
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, S::TMEM_COLS);
  }
}

}  // namespace qpir
