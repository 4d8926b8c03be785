// ens_mma.cuh -- NEXT-1 multi-request QPADL-ENS (Alg. 3 "Multi-request Parallel
// Chor-PIR") on tcgen05 tensor cores, reading the records
// once, in their own theta-major layout (no bit-planes in HBM).
//
// Response of share q, byte j, bit i (GF(2) product q . DB):
//   out[q][j] bit i = parity( sum_theta share_q[theta] * bit_i(rec_theta[j]) ).
// As an integer GEMM: C[q][n] = sum_theta S[q][theta] * X[theta][n] with
//   S[q][theta] = share bit (0/1 byte, the A operand, K-major),
//   X[theta][n] = rec_theta[j] & (1 << i)   (the B operand, N = bit-row n = (j, i)),
// so C[q][n] = 2^i * count and the response bit is bit i of C -- exact mod 2^32
// (bits above i may wrap, bit i cannot), so no K-split limit applies.  Weighting
// each bit-row by 2^i (one power per row, the same for every record) is what lets
// the B operand be built from a record word with a single AND per 4 bytes:
//   word w = rec_theta[4t .. 4t+3]:  M_i = w & (0x01010101 << i),  i = 0..7,
// M_i holds bit-rows (4t + k, i) for k = 0..3 as 4 consecutive N elements.
// One record is one K row, its bytes run along N: the operand is N-major
// ("MN-major", idesc bit 16), built straight from theta-major record bytes with
// no transposition.
//
// CTA: persistent over units = (share tile group, width tile, K-split).
//   warp 0     : producer -- bulk copy (TMA engine) of the shares tile, MS x 128
//                shares x 64 records of 0/1 bytes (K-major, prebuilt by
//                ens_share_expand_kernel), per K-block of 64 records.
//   warp 1     : TMEM allocator + MMA issuer: tcgen05.mma.cta_group::1.kind::i8,
//                M = 128 shares, N = 256 bit-rows (32 record bytes), K = 32.
//   warps 2..5 : epilogue -- tcgen05.ld 32 lanes (shares) x 32 columns (one
//                record word), bit i of column (i, k) -> bit 8k + i of the word.
//   warps 6..9 : expanders -- cp.async (LDGSTS, zero-fill past r / dp) of the
//                raw record slice (64 records x 32*NT bytes) RS K-blocks ahead
//                into a private ring, LDS back, 8 ANDs per word, STS.128 into the
//                N-major operand stage, fence.proxy.async, mbarrier arrive.
// Smem operand layouts (no swizzle):
//   A stage: [s][4 groups of 16 records][128 shares][16 B] -- K-major,
//            LBO = 2 KB (next 16 records), SBO = 128 B (next 8 shares).
//   B stage: [ngroup (16 per 256 bit-rows)][kgroup (8 per 64 records)][8 records][16 B]
//            -- N-major, SBO = 1 KB (next 16 bit-rows), LBO = 128 B (next 8 records).
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace qpir {

constexpr uint32_t EM_KB = 64;        // records per K-block
constexpr uint32_t EM_THREADS = 320;  // 10 warps
constexpr uint32_t EM_EXP_THREADS = 128;

struct EnsMmaArgs {
  const uint8_t* R;   // records [r][dp]
  const uint8_t* Qb;  // shares as 0/1 bytes: [share tiles of 128][G16][128][16]
  uint32_t* out;      // [B][out_ld] response words (zeroed when splits > 1)
  uint64_t r;         // records
  uint32_t dp;        // record stride (multiple of 16)
  uint32_t out_ld;    // words per response row (dp / 4)
  uint32_t B;         // shares
  uint32_t G16;       // 16-record groups of Qb (>= 4 * kblocks)
  uint32_t s_tiles;   // groups of MS share tiles
  uint32_t w_tiles;   // width tiles of 32 * NT record bytes
  uint32_t splits, kbps, kblocks;
  uint64_t s_tstride;  // bytes per share tile of Qb (G16 * 2048), 64-bit: see MmaArgs::a_pstride
  const unsigned long long* Qp = nullptr;  // TS kernel: packed shares [kblocks][qp_ld]
  uint32_t qp_ld = 0;                      // shares per packed row (multiple of 128)
  uint32_t qp_rows = 0;                    // packed rows (64-record blocks)
};

template <uint32_t MS, uint32_t NT, uint32_t S, uint32_t RS>
struct EmCfg {
  static constexpr uint32_t A_TILE = 128 * EM_KB;         // 8 KB: one share tile
  static constexpr uint32_t A_BYTES = MS * A_TILE;
  static constexpr uint32_t B_TILE = 256 * EM_KB;         // 16 KB: 256 bit-rows
  static constexpr uint32_t B_BYTES = NT * B_TILE;
  static constexpr uint32_t STAGE = A_BYTES + B_BYTES;
  static constexpr uint32_t CHUNKS = EM_KB * 2 * NT;      // 16-byte raw chunks per K-block
  static constexpr uint32_t CPT = CHUNKS / EM_EXP_THREADS;  // chunks per expander thread
  static constexpr uint32_t RAW = CHUNKS * 16;
  static constexpr uint32_t RAW_OFF = S * STAGE;
  static constexpr uint32_t BAR_OFF = RAW_OFF + RS * RAW;
  static constexpr uint32_t TOTAL = BAR_OFF + (2 * S + 2) * 8 + 16;
  static constexpr uint32_t ACC_COLS = MS * NT * 256;
  static constexpr uint32_t TMEM_COLS = ACC_COLS <= 256 ? 256 : 512;
  static_assert(CHUNKS % EM_EXP_THREADS == 0, "chunks per thread");
  static_assert(ACC_COLS <= 512, "accumulator exceeds TMEM");
  static_assert(TOTAL <= 227 * 1024, "smem");
};

template <uint32_t MS, uint32_t NT, uint32_t S, uint32_t RS>
__global__ void __launch_bounds__(EM_THREADS, 1) qpir_ens_mma_kernel(EnsMmaArgs a) {
  using C = EmCfg<MS, NT, S, RS>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const uint32_t warp = threadIdx.x / 32;
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t num_units = a.s_tiles * a.w_tiles * a.splits;

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&full[s], EM_EXP_THREADS + 1);  // expanders + producer's expect_tx
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4 * 32);
    fence_mbarrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // unit -> (split slowest, share group, width tile fastest): the CTAs of a
  // wave share one K range, so each shares tile is read from L2 by every width
  // tile and the record bytes of a K range are all read at about the same time.
  auto decode = [&](uint32_t u, uint32_t& sg, uint32_t& wt, uint32_t& kb0, uint32_t& kb1) {
    const uint32_t per_s = a.s_tiles * a.w_tiles;
    const uint32_t sp = u / per_s, rem = u % per_s;
    sg = rem / a.w_tiles;
    wt = rem % a.w_tiles;
    kb0 = sp * a.kbps;
    kb1 = min(a.kblocks, kb0 + a.kbps);
  };

  if (warp == 0) {
    // ------------------------------------------------------------ shares producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (uint32_t u = blockIdx.x; u < num_units; u += gridDim.x) {
        uint32_t sg, wt, kb0, kb1;
        decode(u, sg, wt, kb0, kb1);
        for (uint32_t kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], C::A_BYTES);
          uint8_t* dst = smem + stage * C::STAGE;
#pragma unroll
          for (uint32_t s = 0; s < MS; ++s)
            bulk_g2s(dst + s * C::A_TILE,
                     a.Qb + (uint64_t)(sg * MS + s) * a.s_tstride + (uint64_t)kb * (4 * 2048), C::A_TILE,
                     &full[stage]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // M = 128 shares, N = 256 bit-rows, u8 x u8 -> s32, A K-major, B N-major
    constexpr uint32_t idesc = idesc_i8_u8u8_s32(128, 256) | (1u << 16);
    uint32_t stage = 0, phase = 0, acc_phase = 0;
    for (uint32_t u = blockIdx.x; u < num_units; u += gridDim.x) {
      uint32_t sg, wt, kb0, kb1;
      decode(u, sg, wt, kb0, kb1);
      mbar_wait(tempty, acc_phase ^ 1);  // epilogue has drained the accumulator
      tc_fence_after();
      for (uint32_t kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sA = smem_u32(smem + stage * C::STAGE);
          const uint32_t sB = sA + C::A_BYTES;
#pragma unroll
          for (uint32_t ks = 0; ks < EM_KB / 32; ++ks) {
#pragma unroll
            for (uint32_t s = 0; s < MS; ++s) {
              const uint64_t da = smem_desc_noswizzle(sA + s * C::A_TILE + ks * 2 * 2048, 2048, 128);
#pragma unroll
              for (uint32_t t = 0; t < NT; ++t) {
                const uint64_t db = smem_desc_noswizzle(sB + t * C::B_TILE + ks * 4 * 128, 128, 1024);
                mma_i8_ss(tmem_base + (s * NT + t) * 256, da, db, idesc,
                          (kb > kb0 || ks > 0) ? 1u : 0u);
              }
            }
          }
          mma_commit(&empty[stage]);
          if (kb + 1 == kb1) mma_commit(tfull);
        }
        __syncwarp();
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
      acc_phase ^= 1;
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;  // TMEM lane quarter (shares 32q .. 32q + 31 of a tile)
    const bool split = a.splits > 1;
    uint32_t acc_phase = 0;
    for (uint32_t u = blockIdx.x; u < num_units; u += gridDim.x) {
      uint32_t sg, wt, kb0, kb1;
      decode(u, sg, wt, kb0, kb1);
      mbar_wait(tfull, acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (uint32_t s = 0; s < MS; ++s) {
        const uint32_t share = (sg * MS + s) * 128 + q * 32 + lane;
#pragma unroll 1
        for (uint32_t t = 0; t < NT; ++t) {
          const uint32_t taddr = tmem_base + ((q * 32u) << 16) + (s * NT + t) * 256;
          const uint32_t w0 = (wt * NT + t) * 8;  // first response word of this N tile
#pragma unroll 1
          for (uint32_t cb = 0; cb < 8; ++cb) {
            uint32_t v[32];
            tmem_ld_32x32b_x16_nowait(taddr + cb * 32, *reinterpret_cast<uint32_t(*)[16]>(v));
            tmem_ld_32x32b_x16_nowait(taddr + cb * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
            tmem_ld_wait();
            // column 4i + k = (byte k of the word, bit i), weighted 2^i
            uint32_t word = 0;
#pragma unroll
            for (uint32_t i = 0; i < 8; ++i)
#pragma unroll
              for (uint32_t k = 0; k < 4; ++k) word |= ((v[4 * i + k] >> i) & 1u) << (8 * k + i);
            const uint32_t wi = w0 + cb;
            if (share < a.B && wi < a.out_ld) {
              uint32_t* dst = a.out + (size_t)share * a.out_ld + wi;
              if (split) {
                if (word) atomicXor(dst, word);
              } else {
                *dst = word;
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(tempty);
      acc_phase ^= 1;
    }
  } else {
    // ------------------------------------------------------------ expanders
    const uint32_t e = threadIdx.x - 6 * 32;  // 0 .. 127
    uint8_t* raw = smem + C::RAW_OFF;
    // chunk x of a K-block: bits [0,3) record & 7, then log2(2 NT) bits chunk c,
    // then record >> 3 -- lanes 8p .. 8p + 7 hold 8 consecutive records of one
    // chunk, so each STS.128 phase writes one contiguous 128-byte core matrix.
    constexpr uint32_t CB = NT == 1 ? 1 : 2;  // log2(2 * NT)
    uint32_t stage = 0, phase = 0;
    for (uint32_t u = blockIdx.x; u < num_units; u += gridDim.x) {
      uint32_t sg, wt, kb0, kb1;
      decode(u, sg, wt, kb0, kb1);
      const uint32_t byte0 = wt * NT * 32;
      auto issue = [&](uint32_t kb) {
        if (kb < kb1) {
          uint8_t* slot = raw + (kb % RS) * C::RAW;
#pragma unroll
          for (uint32_t j = 0; j < C::CPT; ++j) {
            const uint32_t x = e + j * EM_EXP_THREADS;
            const uint32_t rr = (x & 7u) | ((x >> (3 + CB)) << 3);
            const uint32_t c = (x >> 3) & (2 * NT - 1);
            const uint64_t th = (uint64_t)kb * EM_KB + rr;
            const uint32_t off = byte0 + c * 16;
            const bool ok = th < a.r && off < a.dp;
            cp_async_16(slot + x * 16, ok ? a.R + th * a.dp + off : a.R, ok);
          }
        }
        cp_async_commit();  // one group per K-block (empty past the unit's end)
      };
#pragma unroll 1
      for (uint32_t p = 0; p + 1 < RS; ++p) issue(kb0 + p);
#pragma unroll 1
      for (uint32_t kb = kb0; kb < kb1; ++kb) {
        issue(kb + RS - 1);  // into the slot consumed by the previous iteration
        cp_async_wait<RS - 1>();  // this thread's copies of K-block kb have landed
        const uint8_t* slot = raw + (kb % RS) * C::RAW;
        uint4 w[C::CPT];
#pragma unroll
        for (uint32_t j = 0; j < C::CPT; ++j)
          w[j] = *reinterpret_cast<const uint4*>(slot + (e + j * EM_EXP_THREADS) * 16);
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sB = smem + stage * C::STAGE + C::A_BYTES;
#pragma unroll
        for (uint32_t j = 0; j < C::CPT; ++j) {
          const uint32_t x = e + j * EM_EXP_THREADS;
          const uint32_t rr = (x & 7u) | ((x >> (3 + CB)) << 3);
          const uint32_t c = (x >> 3) & (2 * NT - 1);
          const uint32_t ws[4] = {w[j].x, w[j].y, w[j].z, w[j].w};
#pragma unroll
          for (uint32_t wi = 0; wi < 4; ++wi) {
            // bit-rows of record bytes 16c + 4wi .. + 3: N groups 8c + 2wi (bits 0-3)
            // and 8c + 2wi + 1 (bits 4-7); row rr & 7 of K group rr >> 3
            const uint32_t ng = 8 * c + 2 * wi;
            uint8_t* d0 = sB + ((ng * (EM_KB / 8) + (rr >> 3)) * 8 + (rr & 7)) * 16;
            const uint32_t v = ws[wi];
            *reinterpret_cast<uint4*>(d0) =
                make_uint4(v & 0x01010101u, v & 0x02020202u, v & 0x04040404u, v & 0x08080808u);
            *reinterpret_cast<uint4*>(d0 + (EM_KB / 8) * 8 * 16) =
                make_uint4(v & 0x10101010u, v & 0x20202020u, v & 0x40404040u, v & 0x80808080u);
          }
        }
        fence_proxy_async_smem();  // generic-proxy stores -> visible to tcgen05.mma
        mbar_arrive(&full[stage]);
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
      cp_async_wait<0>();
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}


// ----------------------------------------------------------------------------
// Shares in tensor memory (A operand from TMEM, "TS" form), 128-record K-blocks.
//
// The shared-memory form above is bound by per-K-block overhead, not by the
// tensor pipe: ~700 clk per 64-record K-block against 512 clk of MMAs (the
// single-thread issue loop -- barrier waits, descriptor math, commits -- and the
// expander/MMA barrier hand-offs cost a roughly fixed ~600 clk per K-block;
// tools/probes/mma_ts_probe.cu shows the MMAs themselves run at 128 clk each in
// every operand form).  Here
//   * the shares are the MMA's A operand in TMEM: share-expander warps turn
//     each share's bits into 0/1 bytes (3 ALU ops per 4 records) and write
//     them with tcgen05.st, so shared memory carries only the bit-rows and the
//     raw record slice;
//   * a K-block is 128 records: 4 MMAs (M = 128 shares, N = 256 bit-rows,
//     K = 32) = 512 clk per barrier round, descriptors advanced by constants.
// The shares come pre-packed as one u64 per (64 records, share), row-major by
// 64-record block (ens_share_pack_kernel): a warp's 32 shares are one
// 256-byte coalesced load.
//
// CTA: persistent over units = (share tile of 128, width tile of 32 record
// bytes = 256 bit-rows, K-split), split slowest.
//   warp 1      : TMEM allocator + MMA issuer
//   warps 2..5  : epilogue (tcgen05.ld, bit i of column (i, k) -> response bit)
//   warps 6..13 : bit-row expanders, two sets of 4 (set h takes the CTA's
//                 K-blocks g with g % 2 == h: two K-blocks in flight)
//   warps 14..17: share expanders (TMEM lane quarter = warp & 3)
//   warp 0      : idle
constexpr uint32_t ET_THREADS = 576;
constexpr uint32_t ET_KB = 128;  // records per K-block

// S: bit-row stages in smem, SA: share stages in TMEM, RS: raw record-slice
// ring per expander set (cp.async, RS - 1 own K-blocks ahead)
template <uint32_t S, uint32_t SA, uint32_t RS>
struct EtCfg {
  static constexpr uint32_t B_TILE = 256 * ET_KB;            // 32 KB: 256 bit-rows x 128 records
  static constexpr uint32_t RAW = ET_KB * 32;                // 4 KB: 128 records x 32 bytes
  static constexpr uint32_t RAW_OFF = S * B_TILE;
  static constexpr uint32_t BAR_OFF = RAW_OFF + 2 * RS * RAW;  // one raw ring per set
  static constexpr uint32_t TOTAL = BAR_OFF + (2 * S + 2 * SA + 2) * 8 + 16;
  static constexpr uint32_t ACC_COLS = 256;                  // 128 shares x 256 bit-rows
  static constexpr uint32_t STG_COLS = ET_KB / 4;            // 32 columns per K-block
  static constexpr uint32_t KG = ET_KB / 8;                  // 8-record K groups per K-block
  static_assert(ACC_COLS + SA * STG_COLS <= 512, "TMEM");
  static_assert(S % 2 == 0, "expander sets alternate stages");
  static_assert(TOTAL <= 227 * 1024, "smem");
};

template <uint32_t S, uint32_t SA, uint32_t RS>
__global__ void __launch_bounds__(ET_THREADS, 1) qpir_ens_mma_ts_kernel(EnsMmaArgs a) {
  using C = EtCfg<S, SA, RS>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + S;
  uint64_t* afull = empty + S;
  uint64_t* aempty = afull + SA;
  uint64_t* tfull = aempty + SA;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const uint32_t warp = threadIdx.x / 32;
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t num_units = a.s_tiles * a.w_tiles * a.splits;

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&full[s], 128);
      mbar_init(&empty[s], 1);
    }
    for (uint32_t s = 0; s < SA; ++s) {
      mbar_init(&afull[s], 128);
      mbar_init(&aempty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
    fence_mbarrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto decode = [&](uint32_t u, uint32_t& st, uint32_t& wt, uint32_t& kb0, uint32_t& kb1) {
    const uint32_t per_s = a.s_tiles * a.w_tiles;
    const uint32_t sp = u / per_s, rem = u % per_s;
    st = rem / a.w_tiles;
    wt = rem % a.w_tiles;
    kb0 = sp * a.kbps;
    kb1 = min(a.kblocks, kb0 + a.kbps);
  };

  if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // M = 128 shares (TMEM), N = 256 bit-rows (smem, N-major), u8 x u8 -> s32
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_i8_u8u8_s32(128, 256) | (1u << 16);
      // descriptor of stage 0, K step 0; stage s / step ks add (s * B_TILE + ks * 512) >> 4
      const uint64_t desc0 = smem_desc_noswizzle(smem_u32(smem), 128, C::KG * 128);
      uint32_t bs = 0, bph = 0, sa = 0, aph = 0, acc_phase = 0;
      for (uint32_t u = blockIdx.x; u < num_units; u += gridDim.x) {
        uint32_t st, wt, kb0, kb1;
        decode(u, st, wt, kb0, kb1);
        mbar_wait(tempty, acc_phase ^ 1);  // epilogue has drained the accumulator
        tc_fence_after();
        uint32_t accum = 0;
        for (uint32_t kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[bs], bph);
          mbar_wait(&afull[sa], aph);
          tc_fence_after();
          const uint64_t db = desc0 + ((bs * C::B_TILE) >> 4);
          const uint32_t aT = tmem_base + C::ACC_COLS + sa * C::STG_COLS;
#pragma unroll
          for (uint32_t ks = 0; ks < ET_KB / 32; ++ks) {
            mma_i8_ts(tmem_base, aT + ks * 8, db + ((ks * 512) >> 4), idesc, accum);
            accum = 1;
          }
          mma_commit(&empty[bs]);
          mma_commit(&aempty[sa]);
          if (++bs == S) { bs = 0; bph ^= 1; }
          if (++sa == SA) { sa = 0; aph ^= 1; }
        }
        mma_commit(tfull);
        acc_phase ^= 1;
      }
    }
    __syncwarp();
  } else if (warp >= 2 && warp < 6) {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;  // TMEM lane quarter (shares 32q .. 32q + 31 of a tile)
    const bool split = a.splits > 1;
    uint32_t acc_phase = 0;
    for (uint32_t u = blockIdx.x; u < num_units; u += gridDim.x) {
      uint32_t st, wt, kb0, kb1;
      decode(u, st, wt, kb0, kb1);
      mbar_wait(tfull, acc_phase);
      tc_fence_after();
      const uint32_t share = st * 128 + q * 32 + lane;
      const uint32_t taddr = tmem_base + ((q * 32u) << 16);
#pragma unroll 1
      for (uint32_t cb = 0; cb < 8; ++cb) {
        uint32_t v[32];
        tmem_ld_32x32b_x16_nowait(taddr + cb * 32, *reinterpret_cast<uint32_t(*)[16]>(v));
        tmem_ld_32x32b_x16_nowait(taddr + cb * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
        tmem_ld_wait();
        // column 4i + k = (byte k of the word, bit i), weighted 2^i
        uint32_t word = 0;
#pragma unroll
        for (uint32_t i = 0; i < 8; ++i)
#pragma unroll
          for (uint32_t k = 0; k < 4; ++k) word |= ((v[4 * i + k] >> i) & 1u) << (8 * k + i);
        const uint32_t wi = wt * 8 + cb;
        if (share < a.B && wi < a.out_ld) {
          uint32_t* dst = a.out + (size_t)share * a.out_ld + wi;
          if (split) {
            if (word) atomicXor(dst, word);
          } else {
            *dst = word;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(tempty);
      acc_phase ^= 1;
    }
  } else if (warp >= 6 && warp < 14) {
    // ------------------------------------------------------------ bit-row expanders
    const uint32_t e = (threadIdx.x - 6 * 32) & 127u;
    const uint32_t h = (warp - 6) >> 2;  // set
    uint8_t* raw = smem + C::RAW_OFF + h * RS * C::RAW;
    // chunk x (two per thread: e, e + 128) of a K-block: record (x & 7) |
    // ((x >> 4) << 3), half (x >> 3) & 1 -- lanes 8p .. 8p + 7 hold 8
    // consecutive records of one half, so each STS.128 phase writes one
    // contiguous 128-byte core matrix
    uint32_t g = 0;  // the CTA's K-block counter at the start of the unit
    for (uint32_t u = blockIdx.x; u < num_units; u += gridDim.x) {
      uint32_t st, wt, kb0, kb1;
      decode(u, st, wt, kb0, kb1);
      const uint32_t first = kb0 + ((g ^ h) & 1u);
      const uint32_t n = kb1 > first ? (kb1 - first + 1) / 2 : 0;
      auto issue = [&](uint32_t i) {
        if (i < n) {
#pragma unroll
          for (uint32_t j = 0; j < 2; ++j) {
            const uint32_t x = e + 128 * j;
            const uint32_t rr = (x & 7u) | ((x >> 4) << 3), c = (x >> 3) & 1u;
            const uint64_t th = (uint64_t)(first + 2 * i) * ET_KB + rr;
            const uint32_t off = wt * 32 + c * 16;
            const bool ok = th < a.r && off < a.dp;
            cp_async_16(raw + (i % RS) * C::RAW + x * 16, ok ? a.R + th * a.dp + off : a.R, ok);
          }
        }
        cp_async_commit();  // one group per own K-block (empty past the unit's end)
      };
#pragma unroll 1
      for (uint32_t p = 0; p + 1 < RS; ++p) issue(p);
#pragma unroll 1
      for (uint32_t i = 0; i < n; ++i) {
        issue(i + RS - 1);  // into the slot consumed by the previous iteration
        cp_async_wait<RS - 1>();  // this thread's chunks of its K-block i have landed
        uint4 w[2];
#pragma unroll
        for (uint32_t j = 0; j < 2; ++j)
          w[j] = *reinterpret_cast<const uint4*>(raw + (i % RS) * C::RAW + (e + 128 * j) * 16);
        const uint32_t gk = g + (first + 2 * i - kb0);  // the CTA's K-block index
        const uint32_t stage = gk % S;
        mbar_wait(&empty[stage], ((gk / S) & 1u) ^ 1u);
        uint8_t* sB = smem + stage * C::B_TILE;
#pragma unroll
        for (uint32_t j = 0; j < 2; ++j) {
          const uint32_t x = e + 128 * j;
          const uint32_t rr = (x & 7u) | ((x >> 4) << 3), c = (x >> 3) & 1u;
          const uint32_t ws[4] = {w[j].x, w[j].y, w[j].z, w[j].w};
#pragma unroll
          for (uint32_t wi = 0; wi < 4; ++wi) {
            // bit-rows of record bytes 16c + 4wi .. + 3: N groups 8c + 2wi (bits 0-3)
            // and 8c + 2wi + 1 (bits 4-7); row rr & 7 of K group rr >> 3
            const uint32_t ng = 8 * c + 2 * wi;
            uint8_t* d0 = sB + ((ng * C::KG + (rr >> 3)) * 8 + (rr & 7)) * 16;
            const uint32_t v = ws[wi];
            *reinterpret_cast<uint4*>(d0) =
                make_uint4(v & 0x01010101u, v & 0x02020202u, v & 0x04040404u, v & 0x08080808u);
            *reinterpret_cast<uint4*>(d0 + C::KG * 8 * 16) =
                make_uint4(v & 0x10101010u, v & 0x20202020u, v & 0x40404040u, v & 0x80808080u);
          }
        }
        fence_proxy_async_smem();  // generic-proxy stores -> visible to tcgen05.mma
        mbar_arrive(&full[stage]);
      }
      cp_async_wait<0>();
      g += kb1 - kb0;
    }
  } else if (warp >= 14) {
    // ------------------------------------------------------------ share expanders
    // lane = share 32q + lane of the tile; per K-block its 128 bits (two u64
    // of the packed shares) -> 32 TMEM columns of 0/1 bytes (records 4c ..
    // 4c + 3 in column c, byte k = record 4c + k).
    const uint32_t q = warp & 3;
    constexpr uint32_t PF = 4;  // K-blocks of share bits loaded ahead (registers)
    uint32_t sa = 0, aph = 0;
    for (uint32_t u = blockIdx.x; u < num_units; u += gridDim.x) {
      uint32_t st, wt, kb0, kb1;
      decode(u, st, wt, kb0, kb1);
      const unsigned long long* src = a.Qp + (size_t)st * 128 + q * 32 + lane;
      auto ld2 = [&](uint32_t kb, unsigned long long& lo, unsigned long long& hi) {
        lo = hi = 0ull;
        if (kb < kb1) {
          lo = __ldg(src + (size_t)(2 * kb) * a.qp_ld);
          if (2 * kb + 1 < a.qp_rows) hi = __ldg(src + (size_t)(2 * kb + 1) * a.qp_ld);
        }
      };
      unsigned long long nlo[PF], nhi[PF];
#pragma unroll
      for (uint32_t p = 0; p < PF; ++p) ld2(kb0 + p, nlo[p], nhi[p]);
#pragma unroll 1
      for (uint32_t base = kb0; base < kb1; base += PF) {
        unsigned long long clo[PF], chi[PF];
#pragma unroll
        for (uint32_t p = 0; p < PF; ++p) {
          clo[p] = nlo[p];
          chi[p] = nhi[p];
          ld2(base + PF + p, nlo[p], nhi[p]);
        }
#pragma unroll
        for (uint32_t p = 0; p < PF; ++p) {
          if (base + p >= kb1) break;
          uint32_t v[32];
#pragma unroll
          for (uint32_t cc = 0; cc < 16; ++cc) {
            v[cc] = (((uint32_t)(clo[p] >> (4 * cc)) & 0xFu) * 0x00204081u) & 0x01010101u;  // bit k -> byte k
            v[16 + cc] = (((uint32_t)(chi[p] >> (4 * cc)) & 0xFu) * 0x00204081u) & 0x01010101u;
          }
          mbar_wait(&aempty[sa], aph ^ 1);  // staging slot drained by its MMAs
          tc_fence_after();
          tmem_st_32x32b_x32(tmem_base + ((q * 32u) << 16) + C::ACC_COLS + sa * C::STG_COLS, v);
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&afull[sa]);
          if (++sa == SA) { sa = 0; aph ^= 1; }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// Packed shares for the TS kernel: Qp[kb][s] = bits of share s for records
// 64 kb .. 64 kb + 63 (bit t = record 64 kb + t, Def. of the share as an r-bit
// vector), zero for s >= B and past r.  CTA = 32 shares x 32 K-blocks,
// transposed through shared memory: each warp reads 256 contiguous bytes of one
// share row and writes 256 contiguous bytes of one Qp row (the thread-per-word
// form read 8 single bytes at a 5 KB stride per thread: 25 us for 5 MB).
constexpr uint32_t ESP_THREADS = 256;
__global__ void __launch_bounds__(ESP_THREADS) ens_share_pack_kernel(
    const uint8_t* __restrict__ Q, uint32_t B, uint64_t r, uint64_t nb,
    unsigned long long* __restrict__ Qp, uint32_t kblocks, uint32_t ld) {
  __shared__ unsigned long long t[32][33];
  const uint32_t s0 = blockIdx.x * 32;
  const uint32_t kb0 = (blockIdx.y + blockIdx.z * gridDim.y) * 32;
  if (kb0 >= kblocks) return;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // word loads when every row starts 8-byte aligned (nb % 8 == 0, aligned Q)
  const bool words = (nb & 7) == 0 && (reinterpret_cast<uintptr_t>(Q) & 7) == 0;
  for (uint32_t i = w; i < 32; i += ESP_THREADS / 32) {
    const uint32_t s = s0 + i, kb = kb0 + lane;
    unsigned long long x = 0;
    if (s < B && kb < kblocks) {
      const uint8_t* row = Q + (size_t)s * nb;
      const uint64_t by0 = (uint64_t)kb * 8;
      if (words && by0 + 8 <= nb) {
        x = __ldg(reinterpret_cast<const unsigned long long*>(row + by0));
      } else {
#pragma unroll
        for (uint32_t b = 0; b < 8; ++b)
          if (by0 + b < nb) x |= (unsigned long long)__ldg(row + by0 + b) << (8 * b);
      }
      const uint64_t t0 = (uint64_t)kb * 64;
      if (t0 + 64 > r) x &= (t0 >= r) ? 0ull : ((1ull << (r - t0)) - 1ull);
    }
    t[i][lane] = x;
  }
  __syncthreads();
  for (uint32_t i = w; i < 32; i += ESP_THREADS / 32) {
    const uint32_t kb = kb0 + i, s = s0 + lane;
    if (kb < kblocks && s < ld) Qp[(size_t)kb * ld + s] = t[lane][i];
  }
}

}  // namespace qpir
