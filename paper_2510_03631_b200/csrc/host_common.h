// host_common.h -- host-side helpers shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

#include <nvtx3/nvToolsExt.h>

namespace qpir_host {

// NVTX range for the duration of a C-ABI call (visible in Nsight Systems /
// Compute timelines; header-only nvtx3, no-op without a profiler attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

inline uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// QPIR_DEBUG_SYNC=1: synchronise after every launch so that an execution error
// is reported by the launch that caused it (debugging aid; off by default).
inline bool debug_sync_enabled() {
  static const bool on = getenv("QPIR_DEBUG_SYNC") && atoi(getenv("QPIR_DEBUG_SYNC")) != 0;
  return on;
}
inline cudaError_t launch_status() {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && debug_sync_enabled()) e = cudaDeviceSynchronize();
  return e;
}

inline int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// Formats an error message into *dst and returns code.
inline int set_error(std::string* dst, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  *dst = buf;
  return code;
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// 1 = device memory of `dev`, 0 = host memory, -1 = device memory of another device.
inline int where(const void* p, int dev) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged)
    return at.device == dev ? 1 : -1;
  return 0;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Checks for an sm_100 device; returns an error message or "".
inline std::string check_device(int device, int* num_sms) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return "device: no CUDA device available";
  }
  if (device >= ndev) return "device: ordinal out of range";
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return "cudaGetDeviceProperties failed";
  if (prop.major != 10) {
    char b[128];
    snprintf(b, sizeof b, "device: compute capability %d.%d, need 10.x (sm_100a)", prop.major,
             prop.minor);
    return b;
  }
  *num_sms = prop.multiProcessorCount;
  return "";
}

}  // namespace qpir_host
