// Throughput probe: back-to-back tcgen05.mma kind::i8, M = 128, N = 256, K = 32,
// A from shared memory (SS) vs from tensor memory (TS); optionally with
// concurrent tcgen05.st traffic into other TMEM columns.  One CTA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I ../../paper_2510_03631_b200/csrc mma_ts_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace qpir;

template <int MODE>  // 0 = SS, 1 = TS, 2 = TS + STTM traffic, 3 = SS / 4 = TS with B N-major (no swizzle)
__global__ void __launch_bounds__(256, 1) probe(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2[16];
  __shared__ __align__(8) uint64_t bar3;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 24 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 16; ++i) mbar_init(&bar2[i], 1); mbar_init(&bar3, 1); mbar_arrive(&bar3); fence_mbarrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  constexpr uint32_t idesc = idesc_i8_u8u8_s32(128, 256) | ((MODE == 3 || MODE == 4 || MODE >= 10) ? (1u << 16) : 0u);
  unsigned long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    const uint32_t sA = smem_u32(smem), sB = sA + 8192;
    const uint64_t da = smem_desc_noswizzle(sA, 2048, 128);
    const uint64_t db = (MODE == 3 || MODE == 4 || MODE >= 10) ? smem_desc_noswizzle(sB, 128, 1024) : smem_desc_noswizzle(sB, 4096, 128);
    for (int i = 0; i < iters; ++i) {
      if (MODE == 8 && (i & 1) == 0) tc_fence_after();
      if (MODE == 9 && (i & 1) == 0) { mbar_wait(&bar3, 0); tc_fence_after(); }
      if (MODE == 0 || MODE == 3 || (MODE >= 5 && MODE != 11)) mma_i8_ss(tb, da, db, idesc, i > 0);
      else mma_i8_ts(tb, tb + 256 + (i & 7) * 8, db, idesc, i > 0);
      if (MODE == 5 && (i & 1)) mma_commit(&bar2[(i >> 1) & 7]);
      if (MODE == 6 && (i & 3) == 3) mma_commit(&bar2[(i >> 2) & 7]);
      if (MODE == 7 && (i & 1)) { mma_commit(&bar2[(i >> 1) & 7]); mma_commit(&bar2[8 + ((i >> 1) & 7)]); }
    }
    mma_commit(&bar);
  }
  if ((MODE == 10 || MODE == 11) && warp >= 4) {
    // concurrent STS.128 into smem [32 KB, 96 KB): 16 KB per 2 MMAs' worth
    uint4* dst = reinterpret_cast<uint4*>(smem + 32 * 1024);
    const uint32_t t = threadIdx.x - 128;
    for (int i = 0; i < iters / 2; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k) dst[((i & 3) * 1024 + k * 128 + t) & 4095] = make_uint4(i, k, t, 0);
    }
  }
  if (MODE == 2 && warp >= 4) {
    const uint32_t q = warp & 3;
    uint32_t v[16];
    for (int k = 0; k < 16; ++k) v[k] = k * lane;
    for (int i = 0; i < iters / 4; ++i) {
      tmem_st_32x32b_x16(tb + ((q * 32u) << 16) + 384 + (i & 7) * 16, v);
      tmem_st_wait();
    }
  }
  if (threadIdx.x == 0) mbar_wait(&bar, 0);
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tb, 512); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  unsigned long long h[148];
  const int iters = 20000;
  for (int mode = 0; mode < 12; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      auto k = mode == 0 ? probe<0> : mode == 1 ? probe<1> : mode == 2 ? probe<2> : mode == 3 ? probe<3> : mode == 4 ? probe<4> : mode == 5 ? probe<5> : mode == 6 ? probe<6> : mode == 7 ? probe<7> : mode == 8 ? probe<8> : mode == 9 ? probe<9> : mode == 10 ? probe<10> : probe<11>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
      cudaEventRecord(e0);
      k<<<148, 256, 100 * 1024>>>(iters, d);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double macs = 148.0 * iters * 128 * 256 * 32;
      printf("mode %d (%s): %s  %.3f ms  %.1f TOPS  cyc/mma %.1f\n", mode,
             mode == 0 ? "SS" : mode == 1 ? "TS" : mode == 2 ? "TS+STTM" : mode == 3 ? "SS Bmn" : mode == 4 ? "TS Bmn" : mode == 5 ? "SS commit/2" : mode == 6 ? "SS commit/4" : mode == 7 ? "SS 2commits/2" : mode == 8 ? "SS fence/2" : mode == 9 ? "SS wait+fence/2" : mode == 10 ? "SS Bmn + STS" : "TS Bmn + STS", cudaGetErrorString(err), ms,
             2 * macs / ms / 1e9, (double)h[0] / iters);
    }
  }
  return 0;
}
