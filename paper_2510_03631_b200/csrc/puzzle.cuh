// puzzle.cuh -- NEXT-4: PSD.Puzzle.Bind with HCT puzzles on the GPU (Alg. 1
// step 1; HCT.Puzzle.Gen PAPER.md:855; record layout
// PAPER.md:1686, DESIGN R11 / R21).
//
// For every record theta of [theta0, theta0 + n): pi_theta = n_s || kappa ||
// n_l with n_s the 256-bit nonce drawn from Philox4x32-10(key = seed_psd,
// ctr = (theta_lo, theta_hi, w >> 2, 0x48)) (DESIGN R21), and the record
// written as spectrum data (560 B, the caller's) || pi_theta (37 B) || zero
// (the ML-DSA signature slot, left unsigned: DESIGN R21) || zero padding.
// One thread per 16-byte chunk of a record; the chunk's bytes are assembled in
// registers and stored with one 16-byte store when the destination row is
// 16-byte aligned.
#pragma once
#include <cstdint>

#include "philox.cuh"

namespace qpir {

constexpr uint32_t HCT_SPECTRUM = 560;
constexpr uint32_t HCT_PUZZLE = 37;     // 32 B nonce + 4 B kappa + 1 B n_l

struct BindArgs {
  const uint8_t* spectrum;  // n x spec_stride (device)
  uint64_t spec_stride;     // >= 560
  uint64_t theta0, n;
  uint64_t seed_psd;
  uint32_t kappa;
  uint32_t n_l;
  uint32_t d;               // record bytes (>= 597)
  uint8_t* out;             // records, row stride out_stride
  uint64_t out_stride;
  // ML-DSA signatures (mldsa.cuh): n rows of 3024 bytes, the signature of
  // record i at bytes [597, 3017) of row i (16-byte aligned with the record);
  // nullptr = unsigned (zero slot)
  const uint8_t* sig = nullptr;
};

constexpr uint32_t HCT_SIG_END = 3017;   // 597 + 2420
constexpr uint32_t HCT_SIG_STRIDE = 3024;

static __global__ void puzzle_bind_hct_kernel(BindArgs a) {
  const uint32_t chunks = (a.d + 15) / 16;
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t i = gid / chunks;
  const uint32_t c = (uint32_t)(gid % chunks);
  if (i >= a.n) return;
  const uint64_t theta = a.theta0 + i;
  const uint32_t b0 = c * 16;
  uint8_t v[16];
  // nonce words are needed only by the chunks overlapping [560, 592)
  uint32_t nw[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
  if (b0 < HCT_SPECTRUM + 32 && b0 + 16 > HCT_SPECTRUM) {
    const uint2 key = make_uint2((uint32_t)a.seed_psd, (uint32_t)(a.seed_psd >> 32));
#pragma unroll
    for (uint32_t blk = 0; blk < 2; ++blk) {
      const uint4 r = philox4x32_10(make_uint4((uint32_t)theta, (uint32_t)(theta >> 32), blk, 0x48u), key);
      nw[4 * blk + 0] = r.x;
      nw[4 * blk + 1] = r.y;
      nw[4 * blk + 2] = r.z;
      nw[4 * blk + 3] = r.w;
    }
  }
  const uint8_t* sp = a.spectrum + i * a.spec_stride;
#pragma unroll
  for (uint32_t k = 0; k < 16; ++k) {
    const uint32_t b = b0 + k;
    uint8_t x = 0;
    if (b < HCT_SPECTRUM) {
      x = sp[b];
    } else if (b < HCT_SPECTRUM + 32) {
      const uint32_t o = b - HCT_SPECTRUM;
      x = (uint8_t)(nw[o >> 2] >> (8 * (o & 3)));
    } else if (b < HCT_SPECTRUM + 36) {
      x = (uint8_t)(a.kappa >> (8 * (b - HCT_SPECTRUM - 32)));
    } else if (b == HCT_SPECTRUM + 36) {
      x = (uint8_t)a.n_l;
    } else if (a.sig && b < HCT_SIG_END) {
      x = a.sig[i * HCT_SIG_STRIDE + b];
    }
    v[k] = x;  // unsigned signature slot and padding stay zero
  }
  uint8_t* dst = a.out + i * a.out_stride + b0;
  if (b0 + 16 <= a.d && ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0)) {
    uint4 w;
    w.x = v[0] | (v[1] << 8) | (v[2] << 16) | ((uint32_t)v[3] << 24);
    w.y = v[4] | (v[5] << 8) | (v[6] << 16) | ((uint32_t)v[7] << 24);
    w.z = v[8] | (v[9] << 8) | (v[10] << 16) | ((uint32_t)v[11] << 24);
    w.w = v[12] | (v[13] << 8) | (v[14] << 16) | ((uint32_t)v[15] << 24);
    *reinterpret_cast<uint4*>(dst) = w;
  } else {
    for (uint32_t k = 0; k < 16 && b0 + k < a.d; ++k) dst[k] = v[k];
  }
}

// Byte b of the bound record theta (b < d): the same record as
// puzzle_bind_hct_kernel writes, one byte at a time (for the fused pack below).
__device__ __forceinline__ uint8_t bound_record_byte(const BindArgs& a, uint64_t theta, uint32_t b) {
  if (b < HCT_SPECTRUM) return a.spectrum[(theta - a.theta0) * a.spec_stride + b];
  if (b < HCT_SPECTRUM + 32) {
    const uint32_t o = b - HCT_SPECTRUM, w = o >> 2;
    const uint2 key = make_uint2((uint32_t)a.seed_psd, (uint32_t)(a.seed_psd >> 32));
    const uint4 r = philox4x32_10(make_uint4((uint32_t)theta, (uint32_t)(theta >> 32), w >> 2, 0x48u), key);
    const uint32_t x = (w & 3) == 0 ? r.x : (w & 3) == 1 ? r.y : (w & 3) == 2 ? r.z : r.w;
    return (uint8_t)(x >> (8 * (o & 3)));
  }
  if (b < HCT_SPECTRUM + 36) return (uint8_t)(a.kappa >> (8 * (b - HCT_SPECTRUM - 32)));
  if (b == HCT_SPECTRUM + 36) return (uint8_t)a.n_l;
  if (a.sig && b < HCT_SIG_END) return a.sig[(theta - a.theta0) * HCT_SIG_STRIDE + b];
  return 0;  // unsigned signature slot and the padding
}

static inline void launch_puzzle_bind(const BindArgs& a, cudaStream_t st) {
  const uint64_t threads = a.n * ((a.d + 15) / 16);
  const uint32_t blocks = (uint32_t)((threads + 255) / 256);
  puzzle_bind_hct_kernel<<<blocks, 256, 0, st>>>(a);
}

}  // namespace qpir
