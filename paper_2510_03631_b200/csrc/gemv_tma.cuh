// gemv_tma.cuh -- K-B1, persistent TMA-fed variant of the single-query answer
// ans = D . qu mod 2^32 (same math and layout as gemv.cuh).
//
// One CTA per SM, warp-specialised:
//   warp 0     : producer -- for each (panel pair, K-block of 8 groups) of the
//                CTA's stream-K range: builds the 512 B of query limb words of
//                the K-block into the stage (LDG qu + PRMT, whole warp), then
//                one lane issues two 16 KB 1-D bulk copies (TMA engine) of the
//                two 128-row panels' K-block; mbarrier complete_tx.
//   warps 1..8 : consumers -- thread (row, half) folds 2 rows (one per panel)
//                x 4 column groups per stage with IDP4A, limb words read as
//                warp-broadcast LDS.128; at a panel-pair change the two halves
//                are combined in smem and added into ans with RED.ADD.u32.
// The grid covers the flattened iteration space [0, pairs * kblocks) in equal
// contiguous ranges (stream-K), so every SM streams the same number of bytes
// and there is no wave tail; ans must be zeroed before the launch (partial
// panel pairs at range boundaries are shared by two CTAs).
#pragma once
#include <cstdint>

#include "gemv.cuh"
#include "ptx.cuh"

namespace qpir {

constexpr uint32_t GT_CONSUMERS = 512;                 // 16 consumer warps
constexpr uint32_t GT_PARTS = GT_CONSUMERS / 128;      // threads per row (split over groups)
constexpr uint32_t GT_THREADS = GT_CONSUMERS + 32;     // + producer warp
constexpr uint32_t GT_GROUPS = 8;                      // column groups per stage (128 cells)
constexpr uint32_t GT_PANEL_BYTES = GT_GROUPS * 2048;  // 16 KB: one panel x one K-block
constexpr uint32_t GT_STAGE_BYTES = 2 * GT_PANEL_BYTES + GT_GROUPS * 64;  // + limb words
constexpr uint32_t GT_STAGES = 6;
constexpr uint32_t GT_SMEM =
    GT_STAGES * GT_STAGE_BYTES + 2 * GT_STAGES * 8 + (GT_PARTS - 1) * 2 * 128 * 16;

struct GemvTmaArgs {
  const uint8_t* D;    // [L/128][G][128][16]
  const uint32_t* qu;  // m
  uint32_t* ans;       // ell_local, zeroed before the launch
  uint32_t ell_local, m, G;
  uint32_t pairs;      // panel pairs covering ell_local
  uint64_t iters;      // pairs * (G / GT_GROUPS)
};

__global__ void __launch_bounds__(GT_THREADS, 1) gemv_tma_kernel(GemvTmaArgs a) {
  extern __shared__ __align__(1024) uint8_t gt_smem[];
  uint8_t* smem = gt_smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GT_STAGES * GT_STAGE_BYTES);
  uint64_t* empty = full + GT_STAGES;
  uint4* xchg = reinterpret_cast<uint4*>(empty + GT_STAGES);  // [parts-1][2 panels][128 rows]

  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t kblocks = a.G / GT_GROUPS;
  const uint64_t it0 = a.iters * blockIdx.x / gridDim.x;
  const uint64_t it1 = a.iters * (blockIdx.x + 1) / gridDim.x;

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < GT_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], GT_CONSUMERS / 32);
    }
    fence_mbarrier_init();
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;");

  if (warp == 0) {
    // ---------------------------------------------------------- producer
    uint32_t stage = 0, phase = 0;
    for (uint64_t it = it0; it < it1; ++it) {
      const uint32_t pair = (uint32_t)(it / kblocks), kb = (uint32_t)(it % kblocks);
      mbar_wait(&empty[stage], phase ^ 1);
      uint8_t* st = smem + stage * GT_STAGE_BYTES;
      // limb words of this K-block: lane -> (group lane & 7, limb lane >> 3)
      {
        const uint32_t g = kb * GT_GROUPS + (lane & 7u), k = lane >> 3;
        const uint32_t c0 = g * 16u;
        uint32_t q[16];
        if (c0 + 16u <= a.m && ((reinterpret_cast<uintptr_t>(a.qu) & 15u) == 0)) {
          const uint4* p = reinterpret_cast<const uint4*>(a.qu + c0);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint4 v = __ldg(p + i);
            q[4 * i] = v.x;
            q[4 * i + 1] = v.y;
            q[4 * i + 2] = v.z;
            q[4 * i + 3] = v.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) q[i] = (c0 + i < a.m) ? __ldg(a.qu + c0 + i) : 0u;
        }
        uint4 w;
        w.x = limb_word(q[0], q[1], q[2], q[3], k);
        w.y = limb_word(q[4], q[5], q[6], q[7], k);
        w.z = limb_word(q[8], q[9], q[10], q[11], k);
        w.w = limb_word(q[12], q[13], q[14], q[15], k);
        reinterpret_cast<uint4*>(st + 2 * GT_PANEL_BYTES)[(lane & 7u) * 4 + k] = w;
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_expect_tx(&full[stage], 2 * GT_PANEL_BYTES);  // releases the limb stores
        const uint8_t* src = a.D + ((size_t)(2 * pair) * a.G + (size_t)kb * GT_GROUPS) * 2048;
        bulk_g2s(st, src, GT_PANEL_BYTES, &full[stage]);
        bulk_g2s(st + GT_PANEL_BYTES, src + (size_t)a.G * 2048, GT_PANEL_BYTES, &full[stage]);
      }
      __syncwarp();
      if (++stage == GT_STAGES) { stage = 0; phase ^= 1; }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const uint32_t ct = threadIdx.x - 32;     // 0 .. GT_CONSUMERS-1
  const uint32_t row = ct & 127u;           // row within each panel
  const uint32_t part = ct >> 7;            // groups part*GPP .. (warp-uniform)
  constexpr uint32_t GPP = GT_GROUPS / GT_PARTS;
  uint32_t acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
  uint32_t stage = 0, phase = 0;
  uint32_t cur = 0xFFFFFFFFu;

  auto flush = [&](uint32_t pair) {
    // combine the parts of every row, then add into ans
    if (part) {
      xchg[((part - 1) * 2 + 0) * 128 + row] = make_uint4(acc[0][0], acc[0][1], acc[0][2], acc[0][3]);
      xchg[((part - 1) * 2 + 1) * 128 + row] = make_uint4(acc[1][0], acc[1][1], acc[1][2], acc[1][3]);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(GT_CONSUMERS));
    if (!part) {
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        uint32_t s0 = acc[p][0], s1 = acc[p][1], s2 = acc[p][2], s3 = acc[p][3];
#pragma unroll
        for (uint32_t o_ = 1; o_ < GT_PARTS; ++o_) {
          const uint4 o = xchg[((o_ - 1) * 2 + p) * 128 + row];
          s0 += o.x;
          s1 += o.y;
          s2 += o.z;
          s3 += o.w;
        }
        const uint32_t v = s0 + (s1 << 8) + (s2 << 16) + (s3 << 24);
        const uint32_t r = (2 * pair + p) * 128u + row;
        if (r < a.ell_local) atomicAdd(a.ans + r, v);
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(GT_CONSUMERS));
  };

  asm volatile("griddepcontrol.wait;" ::: "memory");  // ans zeroed, previous grid done
  for (uint64_t it = it0; it < it1; ++it) {
    const uint32_t pair = (uint32_t)(it / kblocks);
    if (pair != cur) {
      if (cur != 0xFFFFFFFFu) flush(cur);
      cur = pair;
#pragma unroll
      for (int p = 0; p < 2; ++p) acc[p][0] = acc[p][1] = acc[p][2] = acc[p][3] = 0u;
    }
    mbar_wait(&full[stage], phase);
    const uint8_t* st = smem + stage * GT_STAGE_BYTES;
    const uint4* lw = reinterpret_cast<const uint4*>(st + 2 * GT_PANEL_BYTES);
#pragma unroll
    for (uint32_t gi = 0; gi < GPP; ++gi) {
      const uint32_t g = part * GPP + gi;
      const uint4 l0 = lw[g * 4 + 0], l1 = lw[g * 4 + 1], l2 = lw[g * 4 + 2], l3 = lw[g * 4 + 3];
      const uint4 d0 = *reinterpret_cast<const uint4*>(st + g * 2048 + row * 16);
      const uint4 d1 = *reinterpret_cast<const uint4*>(st + GT_PANEL_BYTES + g * 2048 + row * 16);
      dp4a_group(d0, l0, l1, l2, l3, acc[0]);
      dp4a_group(d1, l0, l1, l2, l3, acc[1]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == GT_STAGES) { stage = 0; phase ^= 1; }
  }
  if (cur != 0xFFFFFFFFu) flush(cur);
}

}  // namespace qpir
