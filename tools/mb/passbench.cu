// Store-pattern microbenchmark for the QFT-30 dominant pass (c128, one round,
// direct loads): 2^30 amplitudes, tiles of 256 threads x 16 registers, the 16
// registers of a thread 1 GiB apart (register bits = the top 4 qubits), one
// 16-byte load per thread per tile from the support, K dependent-free FP64
// FMAs per register, 16 streaming stores.  Separates the store pattern's own
// ceiling from the compute/store overlap.  Best of 5, CUDA events.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o passbench tools/mb/passbench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

template <int LV>
__device__ __forceinline__ double2 ldv(const double2* p) {
  if (LV == 0) return __ldcs(p);
  if (LV == 3) return __ldg(p);
  double2 v;
  if (LV == 1)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  else
    asm volatile("ld.global.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

template <int K, bool STRIDED, bool LOAD, int AHEAD, int PF, int LV = 0>
__global__ void __launch_bounds__(256) k_pass(const double2* __restrict__ in, double2* __restrict__ out,
                                              uint32_t ntiles, double c0, uint32_t t0 = 0) {
  // AHEAD > 0: the loads of the next AHEAD tiles are in flight in registers
  double2 q[AHEAD > 0 ? AHEAD : 1];
  const uint64_t lmask = (1ull << 26) - 1;
#pragma unroll
  for (int j = 0; j < AHEAD; ++j) {
    const uint32_t tj = t0 + blockIdx.x + j * gridDim.x;
    q[j] = tj < ntiles ? ldv<LV>(in + ((((uint64_t)tj << 8) | threadIdx.x) & lmask)) : make_double2(0, 0);
  }
  uint32_t it = 0;
  for (uint32_t t = t0 + blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const uint64_t base = ((uint64_t)t << 8) | threadIdx.x;  // bits 0..25
    if (PF > 0 && LOAD && (it % PF) == 0 && threadIdx.x < PF) {
      // this CTA's next PF tiles: all CTAs together prefetch one contiguous
      // PF * grid * 4 KB burst of the input into L2
      const uint32_t tj = t + threadIdx.x * gridDim.x;
      if (tj < ntiles) {
        const double2* src = in + (((uint64_t)tj << 8) & lmask);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], 4096;\n" ::"l"(src) : "memory");
      }
    }
    double2 a[16];
    double2 x = make_double2(c0, 0.5);
    if (LOAD) {
      if (AHEAD == 0) {
        x = ldv<LV>(in + (base & lmask));
      } else {
        x = q[0];
#pragma unroll
        for (int j = 0; j + 1 < AHEAD; ++j) q[j] = q[j + 1];
        const uint32_t tn = t + AHEAD * gridDim.x;
        q[AHEAD - 1] = tn < ntiles ? ldv<LV>(in + ((((uint64_t)tn << 8) | threadIdx.x) & lmask)) : make_double2(0, 0);
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) a[r] = make_double2(x.x + r, x.y - r);
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        a[r].x = fma(a[r].x, c0, a[r].y);
        a[r].y = fma(a[r].y, c0, -a[r].x);
      }
    if (STRIDED) {
#pragma unroll
      for (int r = 0; r < 16; ++r) __stcs(out + (base | ((uint64_t)r << 26)), a[r]);
    } else {
      const uint64_t b2 = ((uint64_t)t << 12) | threadIdx.x;
#pragma unroll
      for (int r = 0; r < 16; ++r) __stcs(out + (b2 | ((uint64_t)r << 8)), a[r]);
    }
  }
}

// pull one segment of the input into L2 (one 4 KB bulk prefetch per tile)
__global__ void k_l2_segment(const double2* __restrict__ in, uint32_t t0, uint32_t t1) {
  const uint32_t t = t0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (t < t1) {
    const double2* src = in + (((uint64_t)t << 8) & ((1ull << 26) - 1));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], 4096;\n" ::"l"(src) : "memory");
  }
}

template <int K>
void run_segmented(const double2* x, double2* y, int per, int nsm, int nseg) {
  const uint32_t ntiles = 1u << 18, seg = ntiles / nseg;
  const int g = nsm * per;
  const float t = best([&] {
    for (int s = 0; s < nseg; ++s) {
      k_l2_segment<<<(seg + 255) / 256, 256>>>(x, s * seg, (s + 1) * seg);
      k_pass<K, true, true, 1, 0><<<g, 256>>>(x, y, (s + 1) * seg, 0.999, s * seg);
    }
  });
  std::printf("{\"K\": %d, \"segments\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f}\n", K, nseg, per, t);
}

template <class F> float best(F f);

// Stores staged through shared memory and written by bulk copies: the 16
// register rows of a tile are 16 contiguous 4 KB runs; one thread issues one
// cp.async.bulk per run once the CTA's rows are in shared memory.
template <int K, int AHEAD, int NT = 256>
__global__ void __launch_bounds__(NT) k_pass_bulk(const double2* __restrict__ in, double2* __restrict__ out,
                                                  uint32_t ntiles, double c0) {
  extern __shared__ __align__(128) double2 stile[];  // 16 rows x NT
  const uint64_t lmask = (1ull << 26) - 1;
  double2 q[AHEAD > 0 ? AHEAD : 1];
#pragma unroll
  for (int j = 0; j < AHEAD; ++j) {
    const uint32_t tj = blockIdx.x + j * gridDim.x;
    q[j] = tj < ntiles ? __ldcs(in + ((((uint64_t)tj * NT) | threadIdx.x) & lmask)) : make_double2(0, 0);
  }
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    double2 x = q[0];
#pragma unroll
    for (int j = 0; j + 1 < AHEAD; ++j) q[j] = q[j + 1];
    const uint32_t tn = t + AHEAD * gridDim.x;
    q[AHEAD - 1] = tn < ntiles ? __ldcs(in + ((((uint64_t)tn * NT) | threadIdx.x) & lmask)) : make_double2(0, 0);
    double2 a[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) a[r] = make_double2(x.x + r, x.y - r);
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        a[r].x = fma(a[r].x, c0, a[r].y);
        a[r].y = fma(a[r].y, c0, -a[r].x);
      }
    // the previous tile's bulk stores must have read shared memory
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) stile[r * NT + threadIdx.x] = a[r];
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 16) {
      const int r = threadIdx.x;
      double2* dst = out + (((uint64_t)t * NT) | ((uint64_t)r << 26));
      const uint32_t src = (uint32_t)__cvta_generic_to_shared(stile + r * NT);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(src), "r"((uint32_t)(NT * 16)) : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  }
  if (threadIdx.x < 16) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// Per-warp variant: each warp stages its 32 lanes x 16 rows and its lanes
// 0..15 issue one 512 B bulk copy per row: no CTA barrier, only __syncwarp.
template <int K, int AHEAD>
__global__ void __launch_bounds__(256) k_pass_bulkw(const double2* __restrict__ in, double2* __restrict__ out,
                                                    uint32_t ntiles, double c0) {
  extern __shared__ __align__(128) double2 stile[];  // 8 warps x 16 rows x 32
  const uint64_t lmask = (1ull << 26) - 1;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  double2* ws = stile + warp * 16 * 32;
  double2 q[AHEAD > 0 ? AHEAD : 1];
#pragma unroll
  for (int j = 0; j < AHEAD; ++j) {
    const uint32_t tj = blockIdx.x + j * gridDim.x;
    q[j] = tj < ntiles ? __ldcs(in + ((((uint64_t)tj << 8) | threadIdx.x) & lmask)) : make_double2(0, 0);
  }
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    double2 x = q[0];
#pragma unroll
    for (int j = 0; j + 1 < AHEAD; ++j) q[j] = q[j + 1];
    const uint32_t tn = t + AHEAD * gridDim.x;
    q[AHEAD - 1] = tn < ntiles ? __ldcs(in + ((((uint64_t)tn << 8) | threadIdx.x) & lmask)) : make_double2(0, 0);
    double2 a[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) a[r] = make_double2(x.x + r, x.y - r);
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        a[r].x = fma(a[r].x, c0, a[r].y);
        a[r].y = fma(a[r].y, c0, -a[r].x);
      }
    if (lane < 16) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 16; ++r) ws[r * 32 + lane] = a[r];
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane < 16) {
      const int r = lane;
      double2* dst = out + ((((uint64_t)t << 8) | (warp << 5)) | ((uint64_t)r << 26));
      const uint32_t src = (uint32_t)__cvta_generic_to_shared(ws + r * 32);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;\n" ::"l"(dst), "r"(src) : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  }
  if (lane < 16) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

template <int K, int AH>
void run_bulkw(const double2* x, double2* y, int per, int nsm) {
  const uint32_t ntiles = 1u << 18;
  const int g = nsm * per;
  cudaFuncSetAttribute(k_pass_bulkw<K, AH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const float t = best([&] { k_pass_bulkw<K, AH><<<g, 256, 65536>>>(x, y, ntiles, 0.999); });
  std::printf("{\"K\": %d, \"bulk_stores_per_warp_512B\": 1, \"ctas_per_sm\": %d, \"ahead\": %d, \"ms\": %.3f, \"err\": \"%s\"}\n",
              K, per, AH, t, cudaGetErrorString(cudaGetLastError()));
}

template <int K, int AH, int NT = 256>
void run_bulk(const double2* x, double2* y, int per, int nsm) {
  const uint32_t ntiles = (1u << 26) / NT;
  const int g = nsm * per;
  const int sm = 16 * NT * 16;
  cudaFuncSetAttribute(k_pass_bulk<K, AH, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  const float t = best([&] { k_pass_bulk<K, AH, NT><<<g, NT, sm>>>(x, y, ntiles, 0.999); });
  std::printf("{\"K\": %d, \"bulk_stores\": 1, \"row_bytes\": %d, \"ctas_per_sm\": %d, \"ahead\": %d, \"ms\": %.3f, \"err\": \"%s\"}\n", K,
              NT * 16, per, AH, t, cudaGetErrorString(cudaGetLastError()));
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

template <int K, bool S, bool L, int AH = 0, int PF = 0, int LV = 0>
void run(const double2* x, double2* y, int per, int nsm) {
  const uint32_t ntiles = 1u << 18;
  const int g = nsm * per;
  const float t = best([&] { k_pass<K, S, L, AH, PF, LV><<<g, 256>>>(x, y, ntiles, 0.999); });
  const double wbytes = 16.0 * (1ull << 30);
  const double rbytes = L ? 16.0 * (1ull << 26) : 0.0;
  std::printf("{\"K\": %d, \"fp64_per_amp\": %d, \"strided\": %d, \"load\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, "
              "\"gbs\": %.1f, \"ahead\": %d, \"l2_prefetch_tiles\": %d, \"load_variant\": %d}\n",
              K, 2 * K, (int)S, (int)L, per, t, (wbytes + rbytes) / t / 1e6, AH, PF, LV);
}

int main() {
  const uint64_t bytes = 16ull << 30;
  double2 *x, *y;
  if (cudaMalloc(&x, bytes) != cudaSuccess || cudaMalloc(&y, bytes) != cudaSuccess) return 1;
  cudaMemset(x, 0, bytes);
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  run_bulk<14, 1, 256>(x, y, 2, nsm);
  run_bulk<14, 1, 512>(x, y, 1, nsm);
  run_bulk<14, 2, 512>(x, y, 1, nsm);
  run_bulk<0, 1, 512>(x, y, 1, nsm);
  run_bulk<14, 1, 256>(x, y, 1, nsm);
  return 0;
}
