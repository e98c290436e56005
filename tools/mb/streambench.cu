// Streaming microbenchmark: read+write a large buffer on B200 with
//   (a) LDG.128 -> registers -> STG.128 (grid-stride, 16 loads in flight/thread)
//   (b) TMA bulk copies (cp.async.bulk) of CHUNK bytes into a 3-stage smem ring,
//       then LDS -> STG, persistent one CTA per SM.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/streambench.cu -o build/streambench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void __launch_bounds__(256) k_ldg(const double2* __restrict__ in, double2* __restrict__ out, uint64_t n) {
  const uint64_t per = 16;
  uint64_t tiles = n / (256 * per);
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    double2 v[16];
    uint64_t base = t * 256 * per + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = __ldcs(in + base + k * 256);
#pragma unroll
    for (int k = 0; k < 16; ++k) { v[k].x *= 0.5; __stcs(out + base + k * 256, v[k]); }
  }
}

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES>
__global__ void __launch_bounds__(256, 1) k_tma(const double2* __restrict__ in, double2* __restrict__ out, uint64_t n,
                                                 uint32_t chunk_bytes, uint32_t tile_bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[STAGES];
  if (threadIdx.x == 0) {
    for (int b = 0; b < STAGES; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t tiles = n * 16 / tile_bytes;
  const uint32_t nch = tile_bytes / chunk_bytes;
  auto issue = [&](uint64_t t, int b) {
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[b])), "r"(tile_bytes) : "memory");
      __syncwarp();
      for (uint32_t c = threadIdx.x; c < nch; c += 32) {
        const char* src = reinterpret_cast<const char*>(in) + t * tile_bytes + (uint64_t)c * chunk_bytes;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su(sm + (size_t)b * tile_bytes + c * chunk_bytes)), "l"(src), "r"(chunk_bytes), "r"(su(&full[b])) : "memory");
      }
    }
  };
  uint64_t t0 = blockIdx.x;
  for (int s = 0; s < STAGES - 1; ++s)
    if (t0 + s * gridDim.x < tiles) issue(t0 + s * gridDim.x, s);
  int it = 0;
  for (uint64_t t = t0; t < tiles; t += gridDim.x, ++it) {
    int b = it % STAGES;
    uint64_t tn = t + (STAGES - 1) * (uint64_t)gridDim.x;
    if (tn < tiles) issue(tn, (it + STAGES - 1) % STAGES);
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                 ::"r"(su(&full[b])), "r"((uint32_t)((it / STAGES) & 1)) : "memory");
    const double2* cur = reinterpret_cast<const double2*>(sm + (size_t)b * tile_bytes);
    double2* o = out + t * (tile_bytes / 16);
    for (uint32_t i = threadIdx.x; i < tile_bytes / 16; i += blockDim.x) {
      double2 v = cur[i];
      v.x *= 0.5;
      __stcs(o + i, v);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
}

// (c) cp.async 16B per thread into a STAGES ring, persistent
template <int STAGES>
__global__ void __launch_bounds__(256, 1) k_ldgsts(const double2* __restrict__ in, double2* __restrict__ out, uint64_t n,
                                                    uint32_t tile_elems) {
  extern __shared__ __align__(128) double2 smd[];
  const uint64_t tiles = n / tile_elems;
  auto issue = [&](uint64_t t, int b) {
    for (uint32_t i = threadIdx.x; i < tile_elems; i += blockDim.x)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(smd + (size_t)b * tile_elems + i)),
                   "l"(in + t * tile_elems + i) : "memory");
  };
  uint64_t t0 = blockIdx.x;
  for (int s = 0; s < STAGES - 1; ++s) {
    if (t0 + s * gridDim.x < tiles) issue(t0 + s * gridDim.x, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  int it = 0;
  for (uint64_t t = t0; t < tiles; t += gridDim.x, ++it) {
    int b = it % STAGES;
    uint64_t tn = t + (STAGES - 1) * (uint64_t)gridDim.x;
    if (tn < tiles) issue(tn, (it + STAGES - 1) % STAGES);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1) : "memory");
    __syncthreads();
    const double2* cur = smd + (size_t)b * tile_elems;
    double2* o = out + t * tile_elems;
    for (uint32_t i = threadIdx.x; i < tile_elems; i += blockDim.x) {
      double2 v = cur[i];
      v.x *= 0.5;
      __stcs(o + i, v);
    }
    __syncthreads();
  }
}

// (d) persistent LDG with a register double buffer (prefetch next tile)
__global__ void __launch_bounds__(256, 1) k_ldg_pf(const double2* __restrict__ in, double2* __restrict__ out, uint64_t n) {
  const uint64_t tiles = n / 4096;
  double2 cur[16], nxt[16];
  uint64_t t = blockIdx.x;
  if (t < tiles)
#pragma unroll
    for (int k = 0; k < 16; ++k) cur[k] = __ldcs(in + t * 4096 + threadIdx.x + k * 256);
  for (; t < tiles; t += gridDim.x) {
    uint64_t tn = t + gridDim.x;
    if (tn < tiles)
#pragma unroll
      for (int k = 0; k < 16; ++k) nxt[k] = __ldcs(in + tn * 4096 + threadIdx.x + k * 256);
#pragma unroll
    for (int k = 0; k < 16; ++k) { cur[k].x *= 0.5; __stcs(out + t * 4096 + threadIdx.x + k * 256, cur[k]); }
#pragma unroll
    for (int k = 0; k < 16; ++k) cur[k] = nxt[k];
  }
}

int main() {
  const uint64_t n = 1ull << 30;  // double2 elements = 16 GiB
  double2 *a, *b;
  CK(cudaMalloc(&a, n * 16));
  CK(cudaMalloc(&b, n * 16));
  CK(cudaMemset(a, 0, n * 16));
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto report = [&](const char* name, float ms) { printf("%-40s %8.3f ms  %8.1f GB/s\n", name, ms, 2.0 * n * 16 / (ms / 1e3) / 1e9); };
  for (int grid : {nsm * 2, nsm * 4, nsm * 8}) {
    k_ldg<<<grid, 256>>>(a, b, n);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_ldg<<<grid, 256>>>(a, b, n);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    char nm[64];
    snprintf(nm, 64, "ldg16 grid=%d", grid);
    report(nm, ms);
  }
  const uint32_t tile = 64 * 1024;
  CK(cudaFuncSetAttribute(k_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * tile));
  CK(cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * tile));
  for (uint32_t chunk : {256u, 512u, 2048u, 8192u, 65536u}) {
    for (int st : {2, 3}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (st == 3) k_tma<3><<<nsm, 256, 3 * tile>>>(a, b, n, chunk, tile);
        else k_tma<2><<<nsm, 256, 2 * tile>>>(a, b, n, chunk, tile);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) {
          char nm[64];
          snprintf(nm, 64, "tma chunk=%u stages=%d", chunk, st);
          report(nm, ms);
        }
      }
    }
  }
  for (int st : {2, 3}) {
    const uint32_t te = 4096;
    if (st == 3) CK(cudaFuncSetAttribute(k_ldgsts<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * te * 16));
    else CK(cudaFuncSetAttribute(k_ldgsts<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * te * 16));
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (st == 3) k_ldgsts<3><<<nsm, 256, 3 * te * 16>>>(a, b, n, te);
      else k_ldgsts<2><<<nsm, 256, 2 * te * 16>>>(a, b, n, te);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) { char nm[64]; snprintf(nm, 64, "ldgsts16 stages=%d (64KB tiles)", st); report(nm, ms); }
    }
  }
  for (int g : {nsm, 2 * nsm}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_ldg_pf<<<g, 256>>>(a, b, n);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) { char nm[64]; snprintf(nm, 64, "ldg register-prefetch grid=%d", g); report(nm, ms); }
    }
  }
  return 0;
}
