// Shared helpers of the femmin_b200 CUDA library (sm_100a, fp64).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "femmin_b200.h"

namespace fm {

// thread-local last error (fm_last_error)
void set_error(const std::string &msg);

#define FM_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t _e = (call);                                                 \
    if (_e != cudaSuccess) {                                                 \
      ::fm::set_error(std::string(#call) + ": " + cudaGetErrorString(_e));   \
      return FM_CUDA_ERROR;                                                  \
    }                                                                        \
  } while (0)

#define FM_CHECK_LAUNCH() FM_CUDA(cudaGetLastError())

#define FM_ARG(cond, msg)                                                    \
  do {                                                                       \
    if (!(cond)) {                                                           \
      ::fm::set_error(msg);                                                  \
      return FM_INVALID_ARG;                                                 \
    }                                                                        \
  } while (0)

// NVTX range around a C-ABI entry point (header-only NVTX v3: a no-op unless
// a profiler is attached), so nsys / ncu timelines show the femmin calls
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};
#define FM_NVTX(name) ::fm::NvtxRange _fm_nvtx_range(name)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// SM count of the current device (queried once per device; 148 on B200)
inline int sm_count() {
  static thread_local int cached_dev = -1, cached_n = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached_dev = dev;
    cached_n = n > 0 ? n : 1;
  }
  return cached_n;
}

// grid-stride launches: at most 64 blocks per SM
inline unsigned grid_for(int64_t n, int block, int64_t cap = 0) {
  if (cap <= 0) cap = (int64_t)sm_count() * 64;
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

// stream-ordered scratch allocation, freed at scope exit
struct Scratch {
  void *p = nullptr;
  cudaStream_t s = nullptr;
  Scratch() = default;
  Scratch(const Scratch &) = delete;
  Scratch &operator=(const Scratch &) = delete;
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
  cudaError_t alloc(size_t bytes, cudaStream_t st) {
    s = st;
    if (bytes == 0) bytes = 16;
    return cudaMallocAsync(&p, bytes, st);
  }
  template <class T> T *as() const { return reinterpret_cast<T *>(p); }
  void reset() {  // stream-ordered free now (lowers the build's peak)
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
  }
};

// counter-based splitmix64 (same constants as the CPU checker used by the tests)
__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ inline double uniform01(uint64_t base, uint64_t idx) {
  uint64_t z = splitmix64(base + idx);
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

}  // namespace fm
