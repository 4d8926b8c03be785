// Load-path probe for the ENS multi-request kernel: 148 persistent CTAs stream
// [64 records x W bytes] slices of a 1 GB record array (records of 3072 B),
// units = (w-tile fastest, K-split slowest) as in qpir_ens_mma_ts_kernel.
// (a) cp.async 16 B per thread into an RS-deep ring; (b) TMA 2D box (W x 64)
// into an RS-deep ring (one elected thread, mbarrier complete_tx).
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace qpir;

constexpr uint32_t R = 327680, DP = 3072, KB = 64;

template <uint32_t W, uint32_t RS>
__global__ void __launch_bounds__(256, 1) cpasync_probe(const uint8_t* rec, uint32_t splits, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t wt_n = DP / W, kblocks = R / KB, kbps = (kblocks + splits - 1) / splits;
  const uint32_t units = wt_n * splits;
  const uint32_t t = threadIdx.x;
  constexpr uint32_t CH = KB * W / 16;  // chunks per slice
  unsigned long long acc = 0;
  for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
    const uint32_t sp = u / wt_n, wt = u % wt_n;
    const uint32_t kb0 = sp * kbps, kb1 = min(kblocks, kb0 + kbps);
    auto issue = [&](uint32_t kb) {
      if (kb < kb1)
        for (uint32_t c = t; c < CH; c += blockDim.x) {
          const uint32_t rr = c / (W / 16), part = c % (W / 16);
          cp_async_16(smem + (kb % RS) * KB * W + c * 16, rec + ((size_t)kb * KB + rr) * DP + wt * W + part * 16, true);
        }
      cp_async_commit();
    };
    for (uint32_t p = 0; p + 1 < RS; ++p) issue(kb0 + p);
    for (uint32_t kb = kb0; kb < kb1; ++kb) {
      issue(kb + RS - 1);
      cp_async_wait<RS - 1>();
      __syncthreads();
      acc += reinterpret_cast<const uint32_t*>(smem + (kb % RS) * KB * W)[t % (KB * W / 4)];
      __syncthreads();
    }
    cp_async_wait<0>();
  }
  if (acc == 0x1234567) sink[0] = acc;
}

// cp.async probe with K-lockstep among the CTAs of one split: every LS K-blocks a
// CTA publishes progress and waits until all CTAs that arrived in its split have
// issued the chunk before the previous one (drift <= 1 chunk).
template <uint32_t W, uint32_t RS, uint32_t LS>
__global__ void __launch_bounds__(256, 1) cpasync_ls_probe(const uint8_t* rec, uint32_t splits, unsigned int* prog,
                                                           unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t wt_n = DP / W, kblocks = R / KB, kbps = (kblocks + splits - 1) / splits;
  const uint32_t units = wt_n * splits;
  const uint32_t t = threadIdx.x;
  constexpr uint32_t CH = KB * W / 16;
  unsigned long long acc = 0;
  for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
    const uint32_t sp = u / wt_n, wt = u % wt_n;
    const uint32_t kb0 = sp * kbps, kb1 = min(kblocks, kb0 + kbps);
    unsigned int* issued = prog + 2 * sp;
    if (t == 0) atomicAdd(issued + 1, 1u);
    auto issue = [&](uint32_t kb) {
      if (kb < kb1) {
        const uint32_t j = (kb - kb0);
        if (j % LS == 0 && j >= LS) {
          if (t == 0) {
            const uint32_t need = j / LS - 1;
            while (true) {
              uint32_t a, b;
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(a) : "l"(issued) : "memory");
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(b) : "l"(issued + 1) : "memory");
              if (a >= b * need) break;
              __nanosleep(100);
            }
          }
          __syncthreads();
        }
        for (uint32_t c = t; c < CH; c += blockDim.x) {
          const uint32_t rr = c / (W / 16), part = c % (W / 16);
          cp_async_16(smem + (kb % RS) * KB * W + c * 16, rec + ((size_t)kb * KB + rr) * DP + wt * W + part * 16, true);
        }
        if (t == 0 && (j % LS == LS - 1)) atomicAdd(issued, 1u);
      }
      cp_async_commit();
    };
    for (uint32_t p = 0; p + 1 < RS; ++p) issue(kb0 + p);
    for (uint32_t kb = kb0; kb < kb1; ++kb) {
      issue(kb + RS - 1);
      cp_async_wait<RS - 1>();
      __syncthreads();
      acc += reinterpret_cast<const uint32_t*>(smem + (kb % RS) * KB * W)[t % (KB * W / 4)];
      __syncthreads();
    }
    cp_async_wait<0>();
    if (t == 0) atomicAdd(issued, 100000u);  // done: never block the others
  }
  if (acc == 0x1234567) sink[0] = acc;
}

template <uint32_t W, uint32_t RS>
__global__ void __launch_bounds__(160, 1) tma_probe(const __grid_constant__ CUtensorMap map, uint32_t splits, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RS * KB * W);
  uint64_t* empty = full + RS;
  const uint32_t wt_n = DP / W, kblocks = R / KB, kbps = (kblocks + splits - 1) / splits;
  const uint32_t units = wt_n * splits;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < RS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 4); }
    fence_mbarrier_init();
  }
  __syncthreads();
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  unsigned long long acc = 0;
  uint32_t n = 0;
  if (warp == 4) {
    if (lane == 0)
    for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
      const uint32_t sp = u / wt_n, wt = u % wt_n;
      const uint32_t kb0 = sp * kbps, kb1 = min(kblocks, kb0 + kbps);
      for (uint32_t kb = kb0; kb < kb1; ++kb, ++n) {
        const uint32_t s = n % RS;
        mbar_wait(&empty[s], ((n / RS) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], KB * W);
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     :: "r"(smem_u32(smem + s * KB * W)), "l"(&map), "r"(wt * W), "r"(kb * KB), "r"(smem_u32(&full[s])) : "memory");
      }
    }
  }
  n = 0;
  if (warp < 4)
  for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
    const uint32_t sp = u / wt_n;
    const uint32_t kb0 = sp * kbps, kb1 = min(kblocks, kb0 + kbps);
    for (uint32_t kb = kb0; kb < kb1; ++kb, ++n) {
      const uint32_t s = n % RS;
      mbar_wait(&full[s], (n / RS) & 1);
      acc += reinterpret_cast<const uint32_t*>(smem + s * KB * W)[threadIdx.x % (KB * W / 4)];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  if (acc == 0x1234567) sink[0] = acc;
}

int main() {
  uint8_t* rec; cudaMalloc(&rec, (size_t)R * DP);
  cudaMemset(rec, 1, (size_t)R * DP);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("%-28s %s %.3f ms %.0f GB/s\n", name, cudaGetErrorString(err), ms, (double)R * DP / ms / 1e6); fflush(stdout);
    }
  };
#define CPA(W, RS, SPL) { auto k = cpasync_probe<W, RS>; size_t sm = RS * KB * W; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    run("cp.async W=" #W " RS=" #RS " sp=" #SPL, [&] { k<<<148, 256, sm>>>(rec, SPL, sink); }); }
#define TMA(W, RS, SPL) { CUtensorMap map; cuuint64_t dims[2] = {DP, R}; cuuint64_t str[1] = {DP}; cuuint32_t box[2] = {W, KB}; cuuint32_t es[2] = {1, 1}; \
    CUresult cr = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, rec, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); \
    if (cr) printf("encode %d\n", (int)cr); \
    auto k = tma_probe<W, RS>; size_t sm = RS * KB * W + 2 * RS * 8; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    run("TMA W=" #W " RS=" #RS " sp=" #SPL, [&] { k<<<148, 160, sm>>>(map, SPL, sink); }); }
  unsigned int* prog; cudaMalloc(&prog, 4096);
#define CPL(W, RS, LS, SPL) { auto k = cpasync_ls_probe<W, RS, LS>; size_t sm = RS * KB * W; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    run("cp.async+LS W=" #W " RS=" #RS " LS=" #LS " sp=" #SPL, [&] { cudaMemsetAsync(prog, 0, 4096); k<<<148, 256, sm>>>(rec, SPL, prog, sink); }); }
  CPA(32, 12, 3) CPA(48, 12, 3) CPA(64, 12, 3) CPA(32, 12, 2) CPA(48, 12, 2)
  TMA(32, 12, 3) TMA(48, 12, 3) TMA(64, 12, 3)
  return 0;
}
