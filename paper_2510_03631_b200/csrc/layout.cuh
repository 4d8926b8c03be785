// layout.cuh -- address helpers of the HBM operand layouts (DESIGN 5).
#pragma once
#include <cstddef>
#include <cstdint>

namespace qpir {

// Byte offset of the 16-byte chunk (column n, 16-cell group g) of a right-hand
// operand in BN-column panels: [Npad / BN][G][BN][16].
__host__ __device__ __forceinline__ size_t limb_off(uint32_t n, uint32_t g, uint32_t G,
                                                    uint32_t BN) {
  return (((size_t)(n / BN) * G + g) * BN + (n % BN)) * 16;
}

}  // namespace qpir
