// pinned H2D bandwidth vs transfer size (cudaHostAlloc source, cudaMemcpyAsync, best of 20, CUDA events)
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t maxb = size_t(256) << 20;
  void *h, *d;
  cudaHostAlloc(&h, maxb, cudaHostAllocDefault);
  cudaMalloc(&d, maxb);
  memset(h, 1, maxb);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (size_t sz = 64 << 10; sz <= maxb; sz *= 2) {
    float best = 1e9f;
    for (int r = 0; r < 20; r++) {
      cudaEventRecord(a, s);
      cudaMemcpyAsync(d, h, sz, cudaMemcpyHostToDevice, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    // 4 back-to-back copies of sz/4 (pipelined small copies)
    float best4 = 1e9f;
    for (int r = 0; r < 20; r++) {
      cudaEventRecord(a, s);
      for (int k = 0; k < 4; k++) cudaMemcpyAsync((char*)d + k * (sz / 4), (char*)h + k * (sz / 4), sz / 4, cudaMemcpyHostToDevice, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best4) best4 = ms;
    }
    printf("{\"bytes\": %zu, \"h2d_gbs\": %.1f, \"us\": %.1f, \"as_4_copies_gbs\": %.1f}\n", sz, sz / best / 1e6, best * 1e3, sz / best4 / 1e6);
  }
  return 0;
}
