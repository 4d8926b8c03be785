// mma_launch.cuh -- host-side launcher of the tcgen05 limb engine (mma.cuh),
// shared by the C-ABI translation units (LWE answer/batch/hint, FTR mod p,
// ENS GF(2) bit-plane batch).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "host_common.h"
#include "mma.cuh"

namespace qpir {

struct MmaJob {
  const uint8_t* A;  // 128-row panels [L/128][G][128][16]
  uint32_t L;        // padded rows (multiple of 256)
  uint32_t G;        // column groups (multiple of 8)
  uint32_t rows;     // valid output rows
  const uint8_t* B;  // BN-column panels [Npad/BN][G][BN][16]
  uint32_t Npad, BN;
  uint32_t* out;
  uint32_t n_out, out_ld;
  uint64_t out_elems;
  uint32_t p = 0;                       // OUT_MODP modulus
  unsigned long long* out64 = nullptr;  // OUT_MODP accumulator
  int num_sms = 148;
  int forced_split = 0;  // 0 = auto
  int mt = 2;            // row panels per CTA tile (1 or 2)
  int gpb = 8;           // column groups per pipeline stage (4 or 8)
  bool out_prezeroed = false;  // caller zeroed `out` (strided chunks): no memset here
  ModpExceptions exc;          // OUT_MODP2, p = 65537: applied by the fixup
  uint32_t* kprog = nullptr;   // K-lockstep scratch (kprog_cap u32), nullptr = off
  uint32_t kprog_cap = 0;
  uint32_t ls_chunk = 0, ls_drift = 1;  // K-blocks per lockstep chunk (0 = off)
  uint32_t l2hint = 0;                  // MmaArgs::l2hint
  // fused limb split (OUT_MODP2, gpb 8): converter warps build B from the u32
  // queries inside the GEMM (mma.cuh CONV); B is then the writable Q' buffer
  bool conv = false;
  const uint32_t* Q = nullptr;
  uint32_t qB = 0, qm = 0;
  uint64_t pM = 0;
  uint32_t* kb_done = nullptr;           // >= G / 8 flags
  uint32_t epoch = 0;
  unsigned long long* conv_ctr = nullptr;
  unsigned long long* conv_base = nullptr;  // host-side running base (advanced here)
};

// BN for 3 limbs per query (OUT_MODP3): a multiple of 48 so queries never
// straddle a tile.
inline uint32_t mma_pick_bn3(uint64_t ncols) {
  if (ncols <= 48) return 48;
  if (ncols <= 96) return 96;
  return 192;
}

inline uint32_t mma_pick_bn(uint64_t ncols) {
  if (ncols <= 16) return 16;
  if (ncols <= 32) return 32;
  if (ncols <= 64) return 64;
  if (ncols <= 128) return 128;
  return 256;
}

// Split K so that work units fill the SMs evenly without making units so
// short that their fixed cost dominates.  Cost in "wave K-blocks" (one K-block
// of every CTA): waves(s) * (K-blocks per unit + c0) for the main loop, c0 ~ 6
// K-blocks of per-unit cost (pipeline ramp, epilogue), plus the output traffic a
// split adds -- a memset and one atomic pass per split instead of plain stores
// -- converted at `wave_bytes` (the D bytes all CTAs stream per K-block).  Fitted
// to tools/batch_size_probe.py (C2, B = 4: 1-2 splits 160-165 us vs 4 splits
// 172 us; B = 64: 1 split 220 us vs 2 splits 236 us).  Split partials are
// combined with commutative atomics (exact for u32 add / XOR).
// HBM-bound tiles (hbm_bound: MT * BN <= 256, a few MMA clocks per streamed
// K-block) with enough tiles to occupy every SM take no extra split at all: a
// partial last wave costs little when the remaining CTAs share the whole HBM
// bandwidth, while every split adds per-unit cost (A/B in one process,
// tools/split_ab_probe.py: C2 B = 4..32, 1 split 159-171 us vs 2 splits 167-181).
inline uint32_t mma_choose_splits(uint32_t tiles, uint32_t kblocks, uint32_t sms, int forced,
                                  uint32_t min_splits, double out_bytes = 0.0,
                                  double wave_bytes = 1.0, bool hbm_bound = false) {
  if (forced > 0)
    return std::max<uint32_t>(min_splits,
                              std::min<uint32_t>(std::min<uint32_t>((uint32_t)forced, 65536u), kblocks));
  if (hbm_bound && tiles >= sms) return min_splits;
  constexpr double c0 = 6.0;
  auto cost = [&](uint32_t s) {
    const double waves = (double)((tiles * s + sms - 1) / sms);
    const double out_passes = s > 1 ? (double)s + 1.0 : 1.0;
    return waves * ((double)((kblocks + s - 1) / s) + c0) + out_passes * out_bytes / wave_bytes;
  };
  uint32_t best = min_splits;
  double best_cost = cost(min_splits);
  for (uint32_t s = min_splits + 1; s <= min_splits + 64; ++s) {
    if (kblocks / s < 8) break;
    const double c = cost(s);
    if (c < best_cost * 0.99) {
      best = s;
      best_cost = c;
    }
  }
  return best;
}

template <uint32_t BN, uint32_t MT, uint32_t GPB, int MODE, bool CONV = false>
cudaError_t mma_launch_cfg(const MmaJob& j, cudaStream_t st, uint64_t* launches) {
  using C = MmaCfg<BN, MT, GPB>;
  MmaArgs a;
  a.A = j.A;
  a.B = j.B;
  a.out = j.out;
  a.G = j.G;
  a.rows = j.rows;
  a.n_out = j.n_out;
  a.out_ld = j.out_ld;
  a.m_tiles = j.L / (MMA_BM * MT);
  a.n_tiles = j.Npad / BN;
  const uint32_t kblocks = j.G / GPB;
  // OUT_MODP(3): each split's limb sums must stay exact in u32 (<= 66051 cells)
  constexpr bool modp = MODE == OUT_MODP || MODE == OUT_MODP3 || MODE == OUT_MODP2;
  const uint32_t max_kps = modp ? 66048u / (16u * GPB) : kblocks;
  const uint32_t min_splits = (kblocks + max_kps - 1) / max_kps;
  a.splits = mma_choose_splits(a.m_tiles * a.n_tiles, kblocks, (uint32_t)j.num_sms,
                               j.forced_split, min_splits,
                               (double)j.out_elems * (modp ? 8.0 : 4.0),
                               (double)C::A_BYTES * (double)j.num_sms, MT * BN <= 256);
  a.kps = std::min((kblocks + a.splits - 1) / a.splits, max_kps);
  a.splits = (kblocks + a.kps - 1) / a.kps;  // no empty split
  a.p = j.p;
  a.out64 = j.out64;
  const uint32_t units = a.m_tiles * a.n_tiles * a.splits;
  const uint32_t grid = std::min<uint32_t>(units, (uint32_t)j.num_sms);
  const uint32_t waves = (units + grid - 1) / grid;
  // lockstep only pays when CTAs share D panels (several N tiles) over long K
  // ranges (C5 hint: 42.5 -> 18.8 GB of DRAM reads per launch; FTR and C4 B = 64
  // have one N tile)
  const bool ls = j.kprog && j.ls_chunk && a.n_tiles >= 2 && 2 * waves <= j.kprog_cap &&
                  a.kps >= 4 * j.ls_chunk;
  a.kprog = ls ? j.kprog : nullptr;
  a.ls_chunk = j.ls_chunk;
  a.ls_drift = std::max<uint32_t>(1, j.ls_drift);
  a.l2hint = j.l2hint;
  cudaError_t e = cudaSuccess;
  if (ls) e = cudaMemsetAsync(j.kprog, 0, waves * 8, st);
  if (e != cudaSuccess) return e;
  if (modp)
    e = cudaMemsetAsync(j.out64, 0, j.out_elems * 8, st);
  else if (a.splits > 1 && !j.out_prezeroed)
    e = cudaMemsetAsync(j.out, 0, j.out_elems * 4, st);
  if (e != cudaSuccess) return e;
  if constexpr (CONV) {
    a.Q = j.Q;
    a.qB = j.qB;
    a.qm = j.qm;
    a.pM = j.pM;
    a.Bw = const_cast<uint8_t*>(j.B);
    a.exc_cnt = const_cast<uint32_t*>(j.exc.cnt);
    a.exc_list = const_cast<uint32_t*>(j.exc.list);
    a.exc_cap = j.exc.cap;
    a.kb_done = j.kb_done;
    a.epoch = j.epoch;
    a.conv_ctr = j.conv_ctr;
    a.conv_base = *j.conv_base;
    // every converter group takes one index past the end before it stops
    *j.conv_base += (unsigned long long)a.splits * a.kps + grid;
  }
  a.a_pstride = (uint64_t)j.G * 2048;
  a.b_tstride = (uint64_t)j.G * BN * 16;
  auto kern = mma_u8_limb_kernel<BN, MT, GPB, MODE, CONV>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::TOTAL);
  if (e != cudaSuccess) return e;
  kern<<<grid, CONV ? MMA_THREADS + MMA_CONV_THREADS : MMA_THREADS, C::TOTAL, st>>>(a);
  ++*launches;
  e = qpir_host::launch_status();
  if (e != cudaSuccess) return e;
  if (modp) {
    const uint32_t blocks = (uint32_t)std::min<uint64_t>((j.out_elems + 255) / 256, 4096);
    modp_fixup_kernel<<<blocks, 256, 0, st>>>(j.out64, j.out, j.out_elems, j.p, j.out_ld, j.exc);
    ++*launches;
    e = qpir_host::launch_status();
  }
  return e;
}

template <int MODE>
cudaError_t mma_launch(const MmaJob& j, cudaStream_t st, uint64_t* launches) {
  if constexpr (MODE == OUT_MODP2) {
    if (j.conv) {  // fused limb split: K-block of 128 cells, BN = 2 x queries per tile
      const bool m2 = j.mt != 1;
      switch (j.BN) {
        case 16: return m2 ? mma_launch_cfg<16, 2, 8, MODE, true>(j, st, launches)
                           : mma_launch_cfg<16, 1, 8, MODE, true>(j, st, launches);
        case 32: return m2 ? mma_launch_cfg<32, 2, 8, MODE, true>(j, st, launches)
                           : mma_launch_cfg<32, 1, 8, MODE, true>(j, st, launches);
        case 64: return m2 ? mma_launch_cfg<64, 2, 8, MODE, true>(j, st, launches)
                           : mma_launch_cfg<64, 1, 8, MODE, true>(j, st, launches);
        case 128: return m2 ? mma_launch_cfg<128, 2, 8, MODE, true>(j, st, launches)
                            : mma_launch_cfg<128, 1, 8, MODE, true>(j, st, launches);
        default: return m2 ? mma_launch_cfg<256, 2, 8, MODE, true>(j, st, launches)
                           : mma_launch_cfg<256, 1, 8, MODE, true>(j, st, launches);
      }
    }
  }
  const bool mt2 = j.mt != 1;
  const bool g4 = j.gpb == 4;
#define QPIR_MMA_CASE(BNV)                                                           \
  case BNV:                                                                          \
    if (g4)                                                                          \
      return mt2 ? mma_launch_cfg<BNV, 2, 4, MODE>(j, st, launches)                  \
                 : mma_launch_cfg<BNV, 1, 4, MODE>(j, st, launches);                 \
    return mt2 ? mma_launch_cfg<BNV, 2, 8, MODE>(j, st, launches)                    \
               : mma_launch_cfg<BNV, 1, 8, MODE>(j, st, launches);
  if constexpr (MODE == OUT_MODP3) {
    switch (j.BN) {
      QPIR_MMA_CASE(48)
      QPIR_MMA_CASE(96)
      default:
        QPIR_MMA_CASE(192)
    }
  } else {
    switch (j.BN) {
      QPIR_MMA_CASE(16)
      QPIR_MMA_CASE(32)
      QPIR_MMA_CASE(64)
      QPIR_MMA_CASE(128)
      default:
        QPIR_MMA_CASE(256)
    }
  }
#undef QPIR_MMA_CASE
}

}  // namespace qpir
