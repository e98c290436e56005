// FP32 pipe throughput on this GPU: FFMA (3-register) vs FFMA2 (packed f32x2).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITER = 4096;
__global__ void k_ffma(float* out, float s, float t) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  float b = s + threadIdx.x, c = t;
#pragma unroll 4
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b, c);
    b += 1e-7f;  // keep operands in registers
  }
  float r = 0; for (int i = 0; i < 16; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_ffma2(float* out, float s, float t) {
  float2 a[8];
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  float2 b = make_float2(s + threadIdx.x, s), c = make_float2(t, t + 1);
#pragma unroll 4
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], b, c);
    b.x += 1e-7f;
  }
  float r = 0; for (int i = 0; i < 8; ++i) r += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
// complex MAC forms: acc += u * x (scalar 4 FFMA vs packed 2 FFMA2)
__global__ void k_cmac(float2* out, float2 u) {
  float2 x[8], acc[8];
  for (int i = 0; i < 8; ++i) { x[i] = make_float2(threadIdx.x + i, i); acc[i] = make_float2(0, 0); }
#pragma unroll 2
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      acc[i].x = fmaf(u.x, x[i].x, acc[i].x); acc[i].x = fmaf(-u.y, x[i].y, acc[i].x);
      acc[i].y = fmaf(u.x, x[i].y, acc[i].y); acc[i].y = fmaf(u.y, x[i].x, acc[i].y);
    }
    u.x += 1e-7f;
  }
  float2 r = make_float2(0, 0); for (int i = 0; i < 8; ++i) { r.x += acc[i].x; r.y += acc[i].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_cmac2(float2* out, float2 u) {
  float2 x[8], acc[8];
  for (int i = 0; i < 8; ++i) { x[i] = make_float2(threadIdx.x + i, i); acc[i] = make_float2(0, 0); }
#pragma unroll 2
  for (int it = 0; it < ITER; ++it) {
    const float2 urr = make_float2(u.x, u.x), uii = make_float2(-u.y, u.y);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      acc[i] = __ffma2_rn(x[i], urr, acc[i]);
      acc[i] = __ffma2_rn(make_float2(x[i].y, x[i].x), uii, acc[i]);
    }
    u.x += 1e-7f;
  }
  float2 r = make_float2(0, 0); for (int i = 0; i < 8; ++i) { r.x += acc[i].x; r.y += acc[i].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, 64 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * 4, thr = 512;
  auto run = [&](const char* name, auto launch, double fma_per_thread) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    double fma = fma_per_thread * blocks * thr;
    double per_sm_clk = fma / (ms * 1e-3) / sms / (clk * 1e3);
    printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"tflops\": %.1f, \"fma_per_sm_per_clk_at_max\": %.1f}\n", name, ms, 2 * fma / ms / 1e9, per_sm_clk);
  };
  run("ffma_3reg", [&] { k_ffma<<<blocks, thr>>>(out, 1.f, 2.f); }, 16.0 * ITER);
  run("ffma2_3reg", [&] { k_ffma2<<<blocks, thr>>>(out, 1.f, 2.f); }, 16.0 * ITER);
  run("cmac_scalar", [&] { k_cmac<<<blocks, thr>>>((float2*)out, make_float2(0.5f, 0.25f)); }, 32.0 * ITER);
  run("cmac_packed", [&] { k_cmac2<<<blocks, thr>>>((float2*)out, make_float2(0.5f, 0.25f)); }, 32.0 * ITER);
  printf("{\"sms\": %d, \"clock_khz\": %d, \"err\": \"%s\"}\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
}
