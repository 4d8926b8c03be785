// qpir_combine.cu -- C ABI (include/qpir.h) of the cross-rank combine steps of
// the record-sharded NEXT rows: after the NCCL all-gather of every rank's
// partial response (dist.py), one kernel folds the parts on the device.
//   ENS / OOP (GF(2), Lemma 1 proof P:1227, Alg. 3): response = XOR of
//     the per-shard partial responses (the XOR over all selected records splits
//     over any partition of the records).
//   FTR (F_p, Lemma 1 proof "R_j := rho_j . DB", Alg. 4):
//     response = sum of the per-shard partial products mod p.
#include <cuda_runtime.h>

#include <string>

#include "../../include/qpir.h"
#include "host_common.h"

using namespace qpir_host;

namespace {

thread_local std::string g_combine_error;

// out[i] = parts[0][i] ^ ... ^ parts[n-1][i]; 16 bytes per thread when aligned.
__global__ void qpir_xor_fold_kernel(const uint8_t* __restrict__ parts, uint64_t n, uint64_t len,
                                     uint8_t* __restrict__ out, bool vec) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  if (vec) {
    const uint64_t nv = len / 16;
    const uint4* P = reinterpret_cast<const uint4*>(parts);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
      uint4 a = P[i];
      for (uint64_t r = 1; r < n; ++r) {
        const uint4 b = P[r * nv + i];
        a.x ^= b.x;
        a.y ^= b.y;
        a.z ^= b.z;
        a.w ^= b.w;
      }
      reinterpret_cast<uint4*>(out)[i] = a;
    }
    return;
  }
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += stride) {
    uint8_t a = parts[i];
    for (uint64_t r = 1; r < n; ++r) a ^= parts[r * len + i];
    out[i] = a;
  }
}

// out[i] = (parts[0][i] + ... + parts[n-1][i]) mod p, summed exactly in 64 bits.
__global__ void qpir_sum_mod_p_kernel(const uint32_t* __restrict__ parts, uint64_t n,
                                      uint64_t len, uint32_t p, uint32_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += stride) {
    unsigned long long s = 0;
    for (uint64_t r = 0; r < n; ++r) s += parts[r * len + i];
    out[i] = (uint32_t)(s % p);
  }
}

int check_dev(const void* a, const void* b, int* dev) {
  cudaPointerAttributes x, y;
  if (cudaPointerGetAttributes(&x, a) != cudaSuccess || cudaPointerGetAttributes(&y, b) != cudaSuccess) {
    cudaGetLastError();
    return set_error(&g_combine_error, QPIR_E_PARAM, "parts/out: not device memory");
  }
  if (x.type != cudaMemoryTypeDevice || y.type != cudaMemoryTypeDevice || x.device != y.device)
    return set_error(&g_combine_error, QPIR_E_PARAM,
                     "parts/out: must be device memory of one device (no host fallback)");
  *dev = x.device;
  return QPIR_OK;
}

uint32_t grid_for(uint64_t work) {
  const uint64_t b = (work + 255) / 256;
  return (uint32_t)(b < 4096 ? (b ? b : 1) : 4096);
}

}  // namespace

extern "C" {

int qpir_xor_fold(const uint8_t* parts, uint64_t n_parts, uint64_t len, uint8_t* out,
                  void* stream) {
  NvtxRange nvtx_("qpir_xor_fold");
  g_combine_error.clear();
  if (!parts || !out) return set_error(&g_combine_error, QPIR_E_PARAM, "parts/out: NULL");
  if (n_parts == 0) return set_error(&g_combine_error, QPIR_E_PARAM, "n_parts: 0");
  if (len == 0) return QPIR_OK;
  int dev = 0;
  int rc = check_dev(parts, out, &dev);
  if (rc) return rc;
  DeviceGuard dg(dev);
  const bool vec = len % 16 == 0 && aligned16(parts) && aligned16(out);
  qpir_xor_fold_kernel<<<grid_for(vec ? len / 16 : len), 256, 0, (cudaStream_t)stream>>>(
      parts, n_parts, len, out, vec);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_error(&g_combine_error, QPIR_E_CUDA, "xor fold: %s", cudaGetErrorString(e));
  return QPIR_OK;
}

int qpir_sum_mod_p(const uint32_t* parts, uint64_t n_parts, uint64_t len, uint32_t p,
                   uint32_t* out, void* stream) {
  NvtxRange nvtx_("qpir_sum_mod_p");
  g_combine_error.clear();
  if (!parts || !out) return set_error(&g_combine_error, QPIR_E_PARAM, "parts/out: NULL");
  if (n_parts == 0 || n_parts > (1ull << 32))
    return set_error(&g_combine_error, QPIR_E_PARAM, "n_parts: %llu not in [1, 2^32]",
                     (unsigned long long)n_parts);
  if (p < 2) return set_error(&g_combine_error, QPIR_E_PARAM, "p: %u < 2", p);
  if (len == 0) return QPIR_OK;
  int dev = 0;
  int rc = check_dev(parts, out, &dev);
  if (rc) return rc;
  DeviceGuard dg(dev);
  qpir_sum_mod_p_kernel<<<grid_for(len), 256, 0, (cudaStream_t)stream>>>(parts, n_parts, len, p, out);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_error(&g_combine_error, QPIR_E_CUDA, "sum mod p: %s", cudaGetErrorString(e));
  return QPIR_OK;
}

const char* qpir_combine_last_error(void) { return g_combine_error.c_str(); }

}  // extern "C"
