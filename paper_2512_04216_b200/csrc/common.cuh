// Shared device/host helpers for libsvb (B200, sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>

#include "../../include/svb.h"
#include "device_core.cuh"

namespace svb {

// ---- error plumbing -------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SVB_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      int code_ = (e_ == cudaErrorMemoryAllocation) ? SVB_E_OOM : SVB_E_CUDA;       \
      throw ::svb::Error(code_, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    }                                                                               \
  } while (0)

#define SVB_CHECK_LAUNCH() SVB_CUDA(cudaGetLastError())

void set_last_error(const char* msg);  // api.cu (thread-local, svb_last_error)

inline void require(bool ok, int code, const std::string& msg) {
  if (!ok) throw Error(code, msg);
}

// cudaMalloc for state-sized buffers: the stream-ordered pool keeps up to
// 1 GiB of freed scratch mapped (svb_create) and the batch executor keeps its
// worker buffers, so on failure both are released and the allocation retried once.
void release_batch_arenas();  // batch.cu: the batch executor's cached buffers
inline cudaError_t state_malloc(void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaErrorMemoryAllocation) return e;
  cudaGetLastError();
  release_batch_arenas();
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(pool, 0);
  }
  cudaGetLastError();
  return cudaMalloc(p, bytes);
}

// Function attributes (max dynamic shared memory, carveout) are per device:
// run `f` once for each device this process launches on.
template <class F> inline void once_per_device(std::atomic<uint64_t>& done, F&& f) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (done.load(std::memory_order_relaxed) & bit) return;
  f();
  done.fetch_or(bit, std::memory_order_release);
}

// Keep up to 1 GiB of freed stream-ordered scratch mapped in the device's
// default pool (per-call scratch: program uploads, sampler leaves, workspaces);
// with the default threshold of 0 every free unmaps at the next sync.
inline void keep_pool_mapped(int device) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = 1ull << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
}

inline int grid_for(uint64_t work, int block, int max_blocks = 148 * 16) {
  uint64_t g = (work + block - 1) / block;
  if (g > (uint64_t)max_blocks) g = max_blocks;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace svb
