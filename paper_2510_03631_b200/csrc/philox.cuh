// philox.cuh -- device Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11),
// the counter-based generator behind the LWE public matrix A (DESIGN R7) and
// the OOP PRG (DESIGN R19).  Independent of the oracle's C implementation.
#pragma once
#include <cstdint>

namespace qpir {

// Philox4x32-10 (Salmon et al., SC'11), device implementation of the public
// matrix generator (DESIGN R7): A[c][j] = Philox(key = seed_A,
// ctr = (c, j >> 2, 0, 0x41))[j & 3].
__device__ __forceinline__ uint4 philox4x32_10(uint4 ctr, uint2 key) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * ctr.x, hi0 = __umulhi(0xD2511F53u, ctr.x);
    const uint32_t lo1 = 0xCD9E8D57u * ctr.z, hi1 = __umulhi(0xCD9E8D57u, ctr.z);
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += 0x9E3779B9u;
    key.y += 0xBB67AE85u;
  }
  return ctr;
}

}  // namespace qpir
