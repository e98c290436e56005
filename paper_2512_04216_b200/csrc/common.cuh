// Shared device/host helpers for libsvb (B200, sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/svb.h"

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

inline void require(bool ok, int code, const std::string& msg) {
  if (!ok) throw Error(code, msg);
}

// ---- complex arithmetic on float2 / double2 --------------------------------
template <typename R> struct CT;
template <> struct CT<float> { using T = float2; };
template <> struct CT<double> { using T = double2; };
template <typename R> using cplx = typename CT<R>::T;

template <typename R> __host__ __device__ __forceinline__ cplx<R> mk(R x, R y) {
  cplx<R> r; r.x = x; r.y = y; return r;
}
template <typename R>
__host__ __device__ __forceinline__ cplx<R> cmul(cplx<R> a, cplx<R> b) {
  return mk<R>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// acc + a*b
template <typename R>
__host__ __device__ __forceinline__ cplx<R> cfma(cplx<R> a, cplx<R> b, cplx<R> acc) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
template <typename R> __host__ __device__ __forceinline__ R norm2(cplx<R> a) {
  return a.x * a.x + a.y * a.y;
}

// insert a zero bit at position q
__host__ __device__ __forceinline__ uint64_t insert0(uint64_t i, int q) {
  uint64_t lo = i & ((1ull << q) - 1ull);
  return ((i >> q) << (q + 1)) | lo;
}

inline int grid_for(uint64_t work, int block, int max_blocks = 148 * 16) {
  uint64_t g = (work + block - 1) / block;
  if (g > (uint64_t)max_blocks) g = max_blocks;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace svb
