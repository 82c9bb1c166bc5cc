// Shared definitions for the specpart-b200 CUDA library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/specpart_b200.h"

namespace spb {

// Per-thread last error message (spb_last_error()).
void set_error(const char* fmt, ...);

struct CudaFail {};

#define SPB_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t _e = (call);                                                        \
    if (_e != cudaSuccess) {                                                        \
      ::spb::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__, \
                       __LINE__, cudaGetErrorString(_e));                           \
      return SPB_ERR_CUDA;                                                          \
    }                                                                               \
  } while (0)

#define SPB_TRY(call)                 \
  do {                                \
    int _s = (call);                  \
    if (_s != SPB_OK) return _s;      \
  } while (0)

#define SPB_LAUNCH_CHECK() SPB_CUDA(cudaGetLastError())

constexpr int kWarp = 32;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Bump allocator over a caller-provided workspace (torch owns the memory).
struct Arena {
  char* base = nullptr;
  size_t cap = 0;
  size_t used = 0;
  bool dry = false;  // size query mode
  template <typename T>
  T* take(size_t count) {
    size_t off = round_up((int64_t)used, 256);
    used = off + count * sizeof(T);
    if (dry) return nullptr;
    if (used > cap) return nullptr;
    return reinterpret_cast<T*>(base + off);
  }
};

inline int num_sms() {
  static int sms = -1;
  if (sms < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
  }
  return sms;
}

// Kernel attributes (dynamic shared memory, cluster sizes) belong to a device
// context: remember per device ordinal that they were set. Setting them twice is
// harmless, so two threads racing here both set them before launching.
inline uint64_t device_bit() {
  int dev = 0;
  cudaGetDevice(&dev);
  return 1ull << (dev & 63);
}
inline bool done_on_device(const std::atomic<uint64_t>& mask) {
  return (mask.load(std::memory_order_acquire) & device_bit()) != 0;
}
inline void mark_on_device(std::atomic<uint64_t>& mask) {
  mask.fetch_or(device_bit(), std::memory_order_release);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace spb
