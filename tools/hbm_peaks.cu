// hbm_peaks.cu -- store-only / load-only / copy HBM bandwidth on this B200 (16-byte vector accesses,
// grid = SMs x 8 CTAs x 256 threads, grid-stride), 1 GiB buffers, best of 10 (CUDA events).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_store(uint4* p, size_t n) {
  const uint4 v = make_uint4(threadIdx.x, blockIdx.x, 1, 2);
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) p[i] = v;
}
__global__ void k_store_unroll4(uint4* p, size_t n) {
  const uint4 v = make_uint4(threadIdx.x, blockIdx.x, 1, 2);
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) { p[i] = v; p[i + stride] = v; p[i + 2 * stride] = v; p[i + 3 * stride] = v; }
  for (; i < n; i += stride) p[i] = v;
}
__global__ void k_load(const uint4* p, size_t n, unsigned* sink) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    uint4 v = __ldcs(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}
__global__ void k_copy(const uint4* a, uint4* b, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) b[i] = __ldcs(a + i);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = size_t(1) << 30, n = bytes / 16;
  uint4 *a, *b;
  unsigned* sink;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMalloc(&sink, 4);
  cudaMemset(a, 1, bytes); cudaMemset(b, 2, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int occ : {4, 8, 16}) {
    const int grid = sms * occ;
    float best[4] = {1e9f, 1e9f, 1e9f, 1e9f};
    for (int rep = 0; rep < 10; rep++) {
      float ms;
      cudaEventRecord(e0); k_store<<<grid, 256>>>(b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (ms < best[0]) best[0] = ms;
      cudaEventRecord(e0); k_store_unroll4<<<grid, 256>>>(b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (ms < best[1]) best[1] = ms;
      cudaEventRecord(e0); k_load<<<grid, 256>>>(a, n, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (ms < best[2]) best[2] = ms;
      cudaEventRecord(e0); k_copy<<<grid, 256>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (ms < best[3]) best[3] = ms;
    }
    printf("{\"ctas_per_sm\": %d, \"store_gbs\": %.1f, \"store_unroll4_gbs\": %.1f, \"load_gbs\": %.1f, \"copy_rw_gbs\": %.1f}\n",
           occ, bytes / best[0] / 1e6, bytes / best[1] / 1e6, bytes / best[2] / 1e6, 2 * bytes / best[3] / 1e6);
  }
  // small outputs (a config-2 sized decode writes ~48 MB per chunk): store of 48 MB, L2-flushed first
  for (size_t mb : {16, 48, 144}) {
    const size_t nn = (mb << 20) / 16;
    float best = 1e9f;
    for (int rep = 0; rep < 10; rep++) {
      cudaMemset(a, rep, bytes);  // evict
      float ms;
      cudaEventRecord(e0); k_store_unroll4<<<sms * 8, 256>>>(b, nn); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("{\"store_mb\": %zu, \"after_flush_gbs\": %.1f, \"us\": %.2f}\n", mb, (mb << 20) / best / 1e6, best * 1e3);
  }
  return 0;
}
