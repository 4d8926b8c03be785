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
// Structure (one CTA per SM, persistent over work units = tile x K-split,
// ordered K-split slowest so the CTAs of a wave share one K range):
//   warp 0     : producer -- per K-block of 128 cells, one 1-D bulk async copy
//                (TMA engine, SASS UBLKCP) per 128-row D panel (16 KB each) and
//                one for the B tile (BN x 128 B), into a STAGES-deep smem ring
//                (as deep as 227 KB allows); mbarrier complete_tx.  With several
//                column tiles it keeps K-lockstep with its wave (at most ls_drift
//                chunks ahead of the slowest arrived CTA) so shared D panels and
//                B tiles are read from L2, not HBM.
//   warp 1     : TMEM allocator + MMA issuer -- one thread issues
//                tcgen05.mma.cta_group::1.kind::i8 (M = 128, N = BN, K = 32),
//                MT x 4 per K-block (MT row panels share each B tile), into a
//                TMEM accumulator (double-buffered when 2 * MT * BN <= 512 cols);
//                tcgen05.commit frees smem stages and signals the epilogue.
//   warps 2..5 : epilogue -- tcgen05.ld 32 lanes x 16 columns, limb recombine,
//                coalesced u32 stores (red.add when K is split), release TMEM;
//                other modes: mod-p partials into a u64 scratch (FTR), GF(2)
//                parity packed with __ballot_sync (ENS), row-major H (hint).
// The smem operand layout equals the global layout (16-cell interleave):
// [8 groups][rows][16 B] = the canonical no-swizzle K-major layout, core
// matrices of 8 rows x 16 B contiguous (SBO = 128 B between 8-row core
// matrices, LBO = rows * 16 B between the two 16-byte K chunks of one MMA).
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace qpir {

constexpr uint32_t MMA_BM = 128;           // rows of D per UMMA (M)
constexpr uint32_t MMA_BK = 128;           // K padding unit of D (cells)
constexpr uint32_t MMA_THREADS = 192;

// OUT_MODP (NEXT-2, FTR over F_p): query-major, each K-split's exact limb sums
// (u32-exact while the split covers <= 66051 cells) are folded to
// sum_k 2^{8k} C_k mod p in 64-bit and added into a u64 scratch; a fixup
// kernel reduces mod p again.
// OUT_PARITY (NEXT-1 ENS on tensor cores): A = bit-planes of the records (rows
// 8j + k = bit k of byte j, values 0/1), B = shares as 0/1 bytes; the GF(2)
// response bit is the parity of the s32 count, 32 consecutive bit-rows (one
// warp's TMEM lanes) pack into one u32 of the response with __ballot_sync;
// K-split partials combine with atomicXor.
// OUT_MODP3: as OUT_MODP with 3 limbs per query (entries pre-reduced mod
// p < 2^24 by the limb split), BN a multiple of 48: 25 % fewer MMAs.
// OUT_MODP2: 2 limbs per query (p <= 65537; entries pre-reduced mod p, the one
// residue 65536 of p = 65537 added back by modp_fixup_kernel): half the MMAs.
enum : int {
  OUT_QUERY_MAJOR = 0, OUT_ROW_MAJOR = 1, OUT_MODP = 2, OUT_PARITY = 3, OUT_MODP3 = 4, OUT_MODP2 = 5
};

struct MmaArgs {
  const uint8_t* A;   // D shard, 128-row panels [L/128][G][128][16]
  const uint8_t* B;   // limbs, BN-column panels [Npad/BN][G][BN][16]
  uint32_t* out;
  uint32_t G;         // column groups (multiple of 8)
  uint32_t rows;      // valid output rows (ell_local)
  uint32_t n_out;     // valid outputs along N (queries B, or hint width n)
  uint32_t out_ld;    // query-major: ell_local; row-major: n
  uint32_t m_tiles, n_tiles, splits, kps;  // work units = m_tiles * n_tiles * splits
  uint32_t p;         // OUT_MODP modulus
  unsigned long long* out64;  // OUT_MODP accumulator [n_out][out_ld]
  // K-lockstep (L2 reuse): the CTAs of one wave of units issue their loads
  // chunk by chunk (ls_chunk K-blocks), at most ls_drift chunks ahead of the
  // slowest CTA of the wave, so the D panels and B tiles they share stay in L2
  // instead of being re-read from HBM by CTAs that drifted apart.
  // Only CTAs that have started a wave count (kprog[2w + 1]), so a CTA never
  // waits for one that is not resident (e.g. SMs held by a concurrent launch).
  uint32_t* kprog;    // [waves][2]: chunks issued, CTAs arrived (zeroed per launch), or nullptr
  uint32_t ls_chunk, ls_drift;
  // Byte strides of one 128-row panel of A (G * 2048) and one BN-column tile of
  // B (G * BN * 16), passed as 64-bit values: computed in-kernel from the
  // 32-bit G, ptxas (CUDA 12.9) folded "base + (u64)G << 11" into a 32-bit
  // uniform LEA with the high half zeroed (SASS "UMOV URn+1, URZ; ULEA URn"
  // feeding UBLKCP: an illegal address for the second D panel; see
  // tools/sass_counts.py, which checks every build for that pattern).
  uint64_t a_pstride, b_tstride;
  // L2 eviction hints on the bulk copies (bit 0: A = D panels evict_first,
  // bit 1: B tiles evict_last), meant to keep a split's B K range L2-resident
  // across the waves of that split.  Measured on the C5 hint with 12-24 splits:
  // DRAM reads unchanged (12.1 GB/launch) and slower than 2 splits, so off
  // (profiles/r02_c5_l2_experiments.md).
  uint32_t l2hint = 0;
  // Fused limb split (OUT_MODP2, CONV kernels): converter warps build the B
  // operand (reduced 2-limb planes) from the u32 queries while the GEMM runs.
  // Conversion chunks = K-blocks, taken from a global work counter (so every
  // chunk is converted as long as any CTA runs: no CTA waits on a non-resident
  // one) in the order the units consume them; a chunk publishes
  // kb_done[kb] = epoch (release), the producer acquires it before its bulk copy.
  const uint32_t* Q = nullptr;   // u32 queries [qB][qm]
  uint32_t qB = 0, qm = 0;
  uint64_t pM = 0;               // fastmod constant ceil(2^64 / p)
  uint8_t* Bw = nullptr;         // the B operand, written by the converters
  uint32_t* exc_cnt = nullptr;   // p = 65537: per-query exception counts / lists
  uint32_t* exc_list = nullptr;
  uint32_t exc_cap = 0;
  uint32_t* kb_done = nullptr;   // [kblocks] epoch flags
  uint32_t epoch = 0;
  unsigned long long* conv_ctr = nullptr;  // monotonic work counter
  unsigned long long conv_base = 0;        // its value at this launch
};

constexpr uint32_t MMA_CONV_THREADS = 256;  // 8 converter warps (CONV kernels; 16 measured no faster)

__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// GPB = 16-cell column groups per pipeline stage (K-block = 16 * GPB cells).
template <uint32_t BN, uint32_t MT, uint32_t GPB>
struct MmaCfg {
  static constexpr uint32_t KB_CELLS = 16 * GPB;
  static constexpr uint32_t PANEL_BYTES = MMA_BM * KB_CELLS;  // one 128-row panel x one K-block
  static constexpr uint32_t A_BYTES = MT * PANEL_BYTES;
  static constexpr uint32_t B_BYTES = BN * KB_CELLS;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  // as many stages as fit the 227 KB opt-in smem (minus barriers): deep enough
  // to cover HBM latency at the per-SM share of bandwidth
  static constexpr uint32_t STAGES_RAW = (227u * 1024u - 512u) / STAGE_BYTES;
  static constexpr uint32_t STAGES = STAGES_RAW > 16 ? 16 : STAGES_RAW;
  static constexpr uint32_t ACC_COLS = MT * BN;  // one accumulator buffer
  static constexpr uint32_t ACC_BUFS = (2 * ACC_COLS <= 512) ? 2 : 1;
  static constexpr uint32_t NEED_COLS = ACC_BUFS * ACC_COLS;
  static constexpr uint32_t TMEM_COLS =
      NEED_COLS <= 32 ? 32 : NEED_COLS <= 64 ? 64 : NEED_COLS <= 128 ? 128 : NEED_COLS <= 256 ? 256 : 512;
  static constexpr uint32_t BAR_OFF = STAGES * STAGE_BYTES;
  // full[STAGES], empty[STAGES], tfull[2], tempty[2], tmem addr
  static constexpr uint32_t TOTAL = BAR_OFF + (2 * STAGES + 4) * 8 + 16;
  static_assert(ACC_COLS <= 512, "accumulator exceeds TMEM");
};

// a mod p for any u32 a and 2 <= p < 2^32 with pM = ceil(2^64 / p) (Lemire,
// Kaser & Kurz, "Faster remainder by direct computation", 2019): exact.
__device__ __forceinline__ uint32_t fastmod_u32(uint32_t a, uint64_t pM, uint32_t p) {
  return (uint32_t)__umul64hi(pM * a, p);
}

template <uint32_t BN, uint32_t MT, uint32_t GPB, int OUT_MODE, bool CONV = false>
__global__ void __launch_bounds__(CONV ? MMA_THREADS + MMA_CONV_THREADS : MMA_THREADS, 1)
    mma_u8_limb_kernel(MmaArgs a) {
  using C = MmaCfg<BN, MT, GPB>;
  constexpr uint32_t STAGES = C::STAGES;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = threadIdx.x / 32;
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t num_units = a.m_tiles * a.n_tiles * a.splits;
  const uint32_t kblocks = a.G / GPB;

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
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // unit -> (split, m tile, n tile); the K-split slowest, n fastest: the CTAs
  // running at the same time cover the same K range of ~148 / n_tiles m tiles x
  // all n tiles, so each D panel is shared by n_tiles CTAs and each B tile by
  // the wave's m tiles through L2 (with split fastest, a wave mixed K ranges and
  // re-read every B tile once per split: hint 18.8 GB of DRAM reads -> see DESIGN).
  auto decode = [&](uint32_t u, uint32_t& mt, uint32_t& nt, uint32_t& kb0, uint32_t& kb1) {
    const uint32_t per_s = a.m_tiles * a.n_tiles;
    const uint32_t s = u / per_s;
    const uint32_t r = u % per_s;
    mt = r / a.n_tiles;
    nt = r % a.n_tiles;
    kb0 = s * a.kps;
    kb1 = min(kblocks, kb0 + a.kps);
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, wave = 0;
      const uint32_t LS = a.kprog ? a.ls_chunk : 0u;
      const uint64_t polA = (a.l2hint & 1u) ? l2_policy_evict_first() : l2_policy_evict_normal();
      const uint64_t polB = (a.l2hint & 2u) ? l2_policy_evict_last() : l2_policy_evict_normal();
      for (uint32_t u = blockIdx.x; u < num_units; u += gridDim.x, ++wave) {
        uint32_t mt, nt, kb0, kb1;
        decode(u, mt, nt, kb0, kb1);
        uint32_t* issued = LS ? a.kprog + 2 * wave : nullptr;
        if (LS) atomicAdd(issued + 1, 1u);  // arrived
        for (uint32_t kb = kb0; kb < kb1; ++kb) {
          if (LS && (kb - kb0) % LS == 0) {
            const uint32_t j = (kb - kb0) / LS;
            if (j >= a.ls_drift) {
              const uint32_t need = j - a.ls_drift + 1;  // chunks every arrived CTA issued
              while (ld_acquire_u32(issued) < ld_acquire_u32(issued + 1) * need) __nanosleep(128);
            }
          }
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          uint8_t* dst = smem + stage * C::STAGE_BYTES;
#pragma unroll
          for (uint32_t p = 0; p < MT; ++p) {
            const uint64_t panel = (uint64_t)mt * MT + p;
            const uint8_t* src = a.A + panel * a.a_pstride + (uint64_t)kb * (GPB * 2048);
            if (a.l2hint) bulk_g2s_hint(dst + p * C::PANEL_BYTES, src, C::PANEL_BYTES, &full[stage], polA);
            else bulk_g2s(dst + p * C::PANEL_BYTES, src, C::PANEL_BYTES, &full[stage]);
          }
          if constexpr (CONV) {
            // the D panels above do not depend on the conversion: only the limb
            // tile waits until the converters' generic-proxy stores of this
            // K-block are visible (acquire) to the async-proxy bulk copy
            while (ld_acquire_u32(a.kb_done + kb) != a.epoch) __nanosleep(64);
            fence_proxy_async_global();
          }
          const uint8_t* srcB = a.B + (uint64_t)nt * a.b_tstride + (uint64_t)kb * (GPB * BN * 16);
          if (a.l2hint) bulk_g2s_hint(dst + C::A_BYTES, srcB, C::B_BYTES, &full[stage], polB);
          else bulk_g2s(dst + C::A_BYTES, srcB, C::B_BYTES, &full[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          if (LS && ((kb - kb0) % LS == LS - 1 || kb + 1 == kb1))
            atomicAdd(issued, 1u);  // chunk issued
        }
        if (LS) {
          // a shorter unit (last K-split) still counts as having issued every chunk
          const uint32_t mine = (kb1 - kb0 + LS - 1) / LS, all = (a.kps + LS - 1) / LS;
          if (mine < all) atomicAdd(issued, all - mine);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_i8_u8u8_s32(MMA_BM, BN);
    uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
    for (uint32_t u = blockIdx.x; u < num_units; u += gridDim.x) {
      uint32_t mt, nt, kb0, kb1;
      decode(u, mt, nt, kb0, kb1);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * C::ACC_COLS;
      for (uint32_t kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sA = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sB = sA + C::A_BYTES;
#pragma unroll
          for (uint32_t k = 0; k < C::KB_CELLS / 32; ++k) {
            const uint64_t db = smem_desc_noswizzle(sB + k * 2 * (BN * 16), BN * 16, 128);
#pragma unroll
            for (uint32_t p = 0; p < MT; ++p) {
              const uint64_t da = smem_desc_noswizzle(
                  sA + p * C::PANEL_BYTES + k * 2 * (MMA_BM * 16), MMA_BM * 16, 128);
              mma_i8_ss(d_tmem + p * BN, da, db, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            }
          }
          mma_commit(&empty[stage]);
          if (kb + 1 == kb1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (++acc == C::ACC_BUFS) { acc = 0; acc_phase ^= 1; }
    }
  } else if (!CONV || warp < 6) {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
    const bool split = a.splits > 1;
    uint32_t acc = 0, acc_phase = 0;
    for (uint32_t u = blockIdx.x; u < num_units; u += gridDim.x) {
      uint32_t mt, nt, kb0, kb1;
      decode(u, mt, nt, kb0, kb1);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (uint32_t p = 0; p < MT; ++p) {
        const uint32_t row = (mt * MT + p) * MMA_BM + q * 32 + lane;
        const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * C::ACC_COLS + p * BN;
        // columns per TMEM wait (OUT_MODP3: 48 columns = 16 queries x 3 limbs)
        constexpr uint32_t CH = OUT_MODE == OUT_MODP3 ? 48 : (BN < 64 ? BN : 64);
        static_assert(BN % CH == 0, "BN must be a multiple of the epilogue chunk");
#pragma unroll 1
        for (uint32_t cb = 0; cb < BN; cb += CH) {
          uint32_t v[CH];
#pragma unroll
          for (uint32_t t = 0; t < CH / 16; ++t)
            tmem_ld_32x32b_x16_nowait(taddr + cb + 16 * t, *reinterpret_cast<uint32_t(*)[16]>(v + 16 * t));
          tmem_ld_wait();
          if constexpr (OUT_MODE == OUT_MODP3) {
            const uint32_t j0 = (nt * BN + cb) / 3;
            if (row < a.rows) {
#pragma unroll
              for (uint32_t jj = 0; jj < 16; ++jj) {
                const unsigned long long x = (unsigned long long)v[3 * jj] +
                                             ((unsigned long long)v[3 * jj + 1] << 8) +
                                             ((unsigned long long)v[3 * jj + 2] << 16);
                if (j0 + jj < a.n_out)
                  atomicAdd(a.out64 + (size_t)(j0 + jj) * a.out_ld + row, x % a.p);
              }
            }
          } else {
#pragma unroll
          for (uint32_t t = 0; t < CH / 16; ++t) {
            const uint32_t c0 = cb + 16 * t;
            const uint32_t j0 = (nt * BN + c0) / 4;  // first output (query / hint column)
            if constexpr (OUT_MODE == OUT_PARITY) {
              const uint32_t row0 = (mt * MT + p) * MMA_BM + q * 32;  // first bit-row of the warp
              const uint32_t widx = row0 >> 5;                       // its u32 in the response
#pragma unroll
              for (uint32_t cc = 0; cc < 16; ++cc) {
                const uint32_t word = __ballot_sync(0xffffffffu, v[16 * t + cc] & 1u);
                const uint32_t col = nt * BN + c0 + cc;  // share index
                if (lane == cc && col < a.n_out && widx < a.out_ld) {
                  uint32_t* dst = a.out + (size_t)col * a.out_ld + widx;
                  if (split) atomicXor(dst, word); else *dst = word;
                }
              }
            } else if constexpr (OUT_MODE == OUT_MODP2) {
              const uint32_t jq = (nt * BN + c0) / 2;
              if (row < a.rows) {
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                  const unsigned long long x = (unsigned long long)v[16 * t + 2 * jj] +
                                               ((unsigned long long)v[16 * t + 2 * jj + 1] << 8);
                  // x < 2^41: the u64 sum over <= 2^16 K-splits cannot wrap, so
                  // the one reduction mod p is left to modp_fixup_kernel
                  if (jq + jj < a.n_out)
                    atomicAdd(a.out64 + (size_t)(jq + jj) * a.out_ld + row, x);
                }
              }
            } else if constexpr (OUT_MODE == OUT_MODP) {
              if (row < a.rows) {
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                  const uint32_t* w = v + 16 * t + 4 * jj;
                  const unsigned long long x = (unsigned long long)w[0] +
                                               ((unsigned long long)w[1] << 8) +
                                               ((unsigned long long)w[2] << 16) +
                                               ((unsigned long long)w[3] << 24);
                  if (j0 + jj < a.n_out)
                    atomicAdd(a.out64 + (size_t)(j0 + jj) * a.out_ld + row, x % a.p);
                }
              }
            } else {
            uint32_t o[4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const uint32_t* w = v + 16 * t + 4 * jj;
              o[jj] = w[0] + (w[1] << 8) + (w[2] << 16) + (w[3] << 24);
            }
            if (row < a.rows) {
              if (OUT_MODE == OUT_QUERY_MAJOR) {
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                  if (j0 + jj < a.n_out) {
                    uint32_t* dst = a.out + (size_t)(j0 + jj) * a.out_ld + row;
                    if (split) atomicAdd(dst, o[jj]); else *dst = o[jj];
                  }
                }
              } else {
                uint32_t* dst = a.out + (size_t)row * a.out_ld + j0;
                if (!split && j0 + 4 <= a.n_out && (a.out_ld & 3u) == 0) {
                  *reinterpret_cast<uint4*>(dst) = make_uint4(o[0], o[1], o[2], o[3]);
                } else {
#pragma unroll
                  for (int jj = 0; jj < 4; ++jj)
                    if (j0 + jj < a.n_out) {
                      if (split) atomicAdd(dst + jj, o[jj]); else dst[jj] = o[jj];
                    }
                }
              }
            }
            }  // OUT_MODE not OUT_MODP / OUT_MODP2
          }
          }  // OUT_MODE != OUT_MODP3
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == C::ACC_BUFS) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    // ------------------------------------------------------------ converters
    // (CONV only) K-block kb of the B operand: limb k of (Q[j][c] mod p), c in
    // the block's 16 * GPB cells, for every padded query slot j; the residue
    // 65536 of p = 65537 (17 bits) is written as 0 and listed for the fixup.
    // Warp cw takes queries cw, cw + NCW, ...; lane l the 4 cells 4l .. 4l + 3.
    static_assert(!CONV || (OUT_MODE == OUT_MODP2 && GPB == 8), "fused split: 2 limbs, K-block 128");
    if constexpr (CONV) {
      __shared__ uint32_t s_job[2];
      const uint32_t ct = threadIdx.x - MMA_THREADS, cw = ct / 32, cl = ct % 32;
      const uint32_t total = a.splits * a.kps;
      const uint32_t nq = a.n_tiles * BN / 2;  // padded query slots
      const bool vec = (a.qm & 3u) == 0 && ((reinterpret_cast<uintptr_t>(a.Q) & 15u) == 0);
      for (uint32_t it = 0;; ++it) {
        if (ct == 0)
          s_job[it & 1] = (uint32_t)(atomicAdd(a.conv_ctr, 1ull) - a.conv_base);
        asm volatile("bar.sync 1, %0;" ::"n"(MMA_CONV_THREADS) : "memory");
        const uint32_t jb = s_job[it & 1];
        if (jb >= total) break;
        const uint32_t sp = jb % a.splits, ii = jb / a.splits;  // consumption order
        const uint32_t kb = sp * a.kps + ii;
        const bool live = kb < kblocks && ii < a.kps;
        if (live) {
          const uint32_t c0 = kb * (16 * GPB) + 4 * cl;
          const uint32_t g = c0 >> 4;
          // CU queries per batch (32: all of a warp's, nq = 128): their loads are all in flight before the
          // first is used (one load per warp at a time left the converters
          // latency-bound: 0.5 ms per FTR call instead of the GEMM's 0.2 ms)
          constexpr uint32_t NCW = MMA_CONV_THREADS / 32;
          constexpr uint32_t CU = 128 / NCW;
          for (uint32_t jb0 = cw; jb0 < nq; jb0 += NCW * CU) {
            uint4 x[CU];
#pragma unroll
            for (uint32_t u = 0; u < CU; ++u) {
              const uint32_t j = jb0 + NCW * u;
              x[u] = make_uint4(0u, 0u, 0u, 0u);
              if (j < a.qB) {
                const uint32_t* row = a.Q + (size_t)j * a.qm;
                if (vec && c0 + 4 <= a.qm) {
                  x[u] = __ldg(reinterpret_cast<const uint4*>(row + c0));
                } else {
                  x[u].x = (c0 + 0 < a.qm) ? __ldg(row + c0 + 0) : 0u;
                  x[u].y = (c0 + 1 < a.qm) ? __ldg(row + c0 + 1) : 0u;
                  x[u].z = (c0 + 2 < a.qm) ? __ldg(row + c0 + 2) : 0u;
                  x[u].w = (c0 + 3 < a.qm) ? __ldg(row + c0 + 3) : 0u;
                }
              }
            }
#pragma unroll
            for (uint32_t u = 0; u < CU; ++u) {
              const uint32_t j = jb0 + NCW * u;
              if (j >= nq) break;
              uint32_t v[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
              if (j < a.qB) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  v[e] = fastmod_u32(v[e], a.pM, a.p);
                  if (v[e] == 65536u && a.exc_cnt) {  // p = 65537 only; padding cells are 0
                    const uint32_t idx = atomicAdd(a.exc_cnt + j, 1u);
                    if (idx < a.exc_cap) a.exc_list[(size_t)j * a.exc_cap + idx] = c0 + e;
                    v[e] = 0u;
                  }
                }
              }
              const uint32_t w0 = __byte_perm(__byte_perm(v[0], v[1], 0x0040), __byte_perm(v[2], v[3], 0x0040), 0x5410);
              const uint32_t w1 = __byte_perm(__byte_perm(v[0], v[1], 0x0051), __byte_perm(v[2], v[3], 0x0051), 0x5410);
              const uint32_t n0 = 2 * j;  // limb columns 2j, 2j + 1 (same BN panel: BN even)
              uint8_t* dst = a.Bw + (((size_t)(n0 / BN) * a.G + g) * BN + (n0 % BN)) * 16 + (cl & 3) * 4;
              *reinterpret_cast<uint32_t*>(dst) = w0;
              *reinterpret_cast<uint32_t*>(dst + 16) = w1;
            }
          }
          __threadfence();
        }
        asm volatile("bar.sync 1, %0;" ::"n"(MMA_CONV_THREADS) : "memory");
        if (ct == 0 && live) st_release_u32(a.kb_done + kb, a.epoch);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace qpir

namespace qpir {
// Exception lists of OUT_MODP2 with p = 65537: the residue 65536 does not fit 2
// byte limbs; the limb split wrote it as 0 and listed its column c per query
// (up to `cap` entries; cnt[b] > cap means the list overflowed and the fixup
// rescans that query's row of Q -- adversarial input only).
struct ModpExceptions {
  const uint8_t* D = nullptr;  // 128-row panels [L/128][G][128][16]
  uint32_t G = 0;
  const uint32_t* Q = nullptr;  // the chunk's queries [B][m]
  uint32_t m = 0;
  const uint32_t* cnt = nullptr;   // [B]; nullptr = no exceptions possible
  const uint32_t* list = nullptr;  // [B][cap]
  uint32_t cap = 0;
};

// out[i] = acc[i] mod p (u64 -> u32), after the OUT_MODP* GEMM; with exception
// lists, the missing terms 65536 * D[r][c] are added first (exact in u64).
// out / acc are query-major [n][ld]: i = b * ld + r.
// v mod p by Barrett with pB = floor(2^64 / p): the quotient estimate is exact or
// one short, so one conditional subtraction (64-bit division runs as a software
// routine on the GPU).
__device__ __forceinline__ uint32_t mod_u64_barrett(unsigned long long v, uint32_t p,
                                                    unsigned long long pB) {
  const unsigned long long q = __umul64hi(v, pB);
  unsigned long long r = v - q * p;
  return (uint32_t)(r >= p ? r - p : r);
}

static __global__ void modp_fixup_kernel(const unsigned long long* __restrict__ acc,
                                         uint32_t* __restrict__ out, uint64_t n, uint32_t p,
                                         uint32_t ld, ModpExceptions ex) {
  const unsigned long long pB = ~0ull / p;  // floor(2^64 / p) for p not a power of 2
  const bool pow2 = (p & (p - 1)) == 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long v = acc[i];
    if (ex.cnt) {
      uint32_t b, r;
      if (n <= 0xFFFFFFFFull) {  // 32-bit division (64-bit runs as a software routine)
        b = (uint32_t)i / ld;
        r = (uint32_t)i - b * ld;
      } else {
        b = (uint32_t)(i / ld);
        r = (uint32_t)(i % ld);
      }
      const uint32_t k = ex.cnt[b];
      if (k) {
        const uint8_t* Dr = ex.D + (size_t)(r >> 7) * ex.G * 2048 + (r & 127u) * 16u;
        unsigned long long sum = 0;
        if (k <= ex.cap) {
          const uint32_t* lst = ex.list + (size_t)b * ex.cap;
#pragma unroll 4
          for (uint32_t e = 0; e < k; ++e) {
            const uint32_t c = lst[e];
            sum += Dr[(size_t)(c >> 4) * 2048 + (c & 15u)];
          }
        } else {
          const uint32_t* q = ex.Q + (size_t)b * ex.m;
          for (uint32_t c = 0; c < ex.m; ++c)
            if (__ldg(q + c) % p == 65536u) sum += Dr[(size_t)(c >> 4) * 2048 + (c & 15u)];
        }
        v += sum << 16;
      }
    }
    out[i] = pow2 ? (uint32_t)(v & (p - 1)) : mod_u64_barrett(v, p, pB);
  }
}
}  // namespace qpir
