// Write-only HBM bandwidth on one B200 (16 GiB): streaming 16-byte stores
// (st.global.cs, as the pass kernels' last round), plain stores, and
// cudaMemsetAsync; copy (read + write) for reference.  Best of 5, CUDA events.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o writebench tools/writebench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(256) k_write_cs(double2* __restrict__ out, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const double2 v = make_double2(1.0, 0.0);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) __stcs(out + i, v);
}
__global__ void __launch_bounds__(256) k_write(double2* __restrict__ out, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const double2 v = make_double2(1.0, 0.0);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = v;
}
__global__ void __launch_bounds__(256) k_copy(const double2* __restrict__ in, double2* __restrict__ out, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) __stcs(out + i, __ldcs(in + i));
}

template <class F> float best(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  float bt = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t;
    cudaEventElapsedTime(&t, a, b);
    if (t < bt) bt = t;
  }
  return bt;
}

int main() {
  const uint64_t bytes = 16ull << 30, n = bytes / 16;
  double2 *x, *y;
  if (cudaMalloc(&x, bytes) != cudaSuccess || cudaMalloc(&y, bytes) != cudaSuccess) return 1;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int per : {4, 8, 16}) {
    const int g = nsm * per;
    const float tcs = best([&] { k_write_cs<<<g, 256>>>(x, n); });
    const float tw = best([&] { k_write<<<g, 256>>>(x, n); });
    const float tc = best([&] { k_copy<<<g, 256>>>(y, x, n); });
    std::printf("{\"ctas_per_sm\": %d, \"write_cs_gbs\": %.1f, \"write_gbs\": %.1f, \"copy_rw_gbs\": %.1f}\n", per,
                bytes / tcs / 1e6, bytes / tw / 1e6, 2.0 * bytes / tc / 1e6);
  }
  const float tm = best([&] { cudaMemsetAsync(x, 0, bytes); });
  std::printf("{\"memset_gbs\": %.1f}\n", bytes / tm / 1e6);
  return 0;
}
