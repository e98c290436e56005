// Device->host bandwidth for a 16 GiB state into pinned memory: one copy vs
// chunks over several streams (copy engines), and H2D for reference.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
int main() {
  const size_t bytes = 16ull << 30;
  void *d = nullptr, *h = nullptr;
  if (cudaMalloc(&d, bytes) != cudaSuccess || cudaHostAlloc(&h, bytes, cudaHostAllocPortable) != cudaSuccess) {
    printf("{\"error\": \"alloc\"}\n");
    return 1;
  }
  cudaMemset(d, 1, bytes);
  std::vector<cudaStream_t> st(8);
  for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](int ns, size_t chunk, bool d2h) {
    cudaDeviceSynchronize();
    cudaEventRecord(e0, st[0]);
    for (int i = 1; i < ns; ++i) cudaStreamWaitEvent(st[i], e0);
    size_t off = 0; int k = 0;
    while (off < bytes) {
      size_t c = std::min(chunk, bytes - off);
      if (d2h) cudaMemcpyAsync((char*)h + off, (char*)d + off, c, cudaMemcpyDeviceToHost, st[k % ns]);
      else cudaMemcpyAsync((char*)d + off, (char*)h + off, c, cudaMemcpyHostToDevice, st[k % ns]);
      off += c; ++k;
    }
    for (int i = 1; i < ns; ++i) { cudaEvent_t ev; cudaEventCreate(&ev); cudaEventRecord(ev, st[i]); cudaStreamWaitEvent(st[0], ev); }
    cudaEventRecord(e1, st[0]);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"dir\": \"%s\", \"streams\": %d, \"chunk_mb\": %zu, \"ms\": %.1f, \"gbs\": %.1f}\n", d2h ? "d2h" : "h2d", ns,
           chunk >> 20, ms, bytes / (ms * 1e-3) / 1e9);
  };
  run(1, bytes, true);
  run(1, bytes, true);
  run(2, 256ull << 20, true);
  run(4, 256ull << 20, true);
  run(2, 1ull << 30, true);
  run(8, 64ull << 20, true);
  run(1, bytes, false);
  run(2, 256ull << 20, false);
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
}
