// kernels_util.cu -- the engine's per-group bookkeeping as two tiny kernels instead of memset / D2H copy
// operations (those queue behind the H2D copy engine while a pipeline is streaming; kernels do not).
#include "kernels.h"

namespace cdm {
namespace {

// One-warp CTAs: they must find room on SMs fully occupied by a long RLE grid (a few hundred registers).
constexpr int kUtilThreads = 32;

__global__ void __launch_bounds__(kUtilThreads) zero_kernel(uint4* p, uint32_t n16) {
  for (uint32_t i = blockIdx.x * kUtilThreads + threadIdx.x; i < n16; i += gridDim.x * kUtilThreads)
    p[i] = make_uint4(0u, 0u, 0u, 0u);
}

__global__ void __launch_bounds__(kUtilThreads) harvest_kernel(uint32_t* err, uint32_t* host, uint32_t n) {
  // plain stores to mapped pinned memory: the kernel's completion (the group's done event) makes them
  // visible to the host thread that synchronised on it.  The words are zeroed for the next use.
  for (uint32_t i = threadIdx.x; i < n; i += kUtilThreads) {
    host[i] = err[i];
    err[i] = 0u;
  }
}

// H9 positional checksum: h = sum_i splitmix64(chunk_id ^ i ^ w_i) mod 2^64 over the
// little-endian 8-byte words of a decoded buffer, the last one zero padded.  Grid-stride 16-byte loads,
// warp sums, one 64-bit atomicAdd per warp (addition mod 2^64 is order-free).
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

constexpr int kSumThreads = 256;

__global__ void __launch_bounds__(kSumThreads) checksum_kernel(const uint8_t* p, uint64_t bytes, uint64_t cid,
                                                               unsigned long long* out) {
  const uint64_t nw = bytes / 8;  // full words
  const uint64_t stride = uint64_t(gridDim.x) * kSumThreads;
  const uint64_t t = uint64_t(blockIdx.x) * kSumThreads + threadIdx.x;
  uint64_t h = 0;
  if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {
    const ulonglong2* v = reinterpret_cast<const ulonglong2*>(p);
    for (uint64_t i = t; i < nw / 2; i += stride) {
      const ulonglong2 w = __ldcs(v + i);
      h += splitmix64(cid ^ (2 * i) ^ w.x) + splitmix64(cid ^ (2 * i + 1) ^ w.y);
    }
    if (t == 0 && (nw & 1)) h += splitmix64(cid ^ (nw - 1) ^ reinterpret_cast<const unsigned long long*>(p)[nw - 1]);
  } else {  // 8-byte aligned
    const unsigned long long* v = reinterpret_cast<const unsigned long long*>(p);
    for (uint64_t i = t; i < nw; i += stride) h += splitmix64(cid ^ i ^ v[i]);
  }
  if (t == 0 && (bytes & 7)) {  // the zero-padded tail word
    uint64_t w = 0;
    for (uint64_t k = 0; k < (bytes & 7); k++) w |= uint64_t(p[nw * 8 + k]) << (8 * k);
    h += splitmix64(cid ^ nw ^ w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xFFFFFFFFu, h, o);
  if ((threadIdx.x & 31) == 0 && h) atomicAdd(out, (unsigned long long)h);
}

}  // namespace

cudaError_t launch_checksum(const void* p, uint64_t bytes, uint64_t chunk_id, uint64_t* dev_out, cudaStream_t s) {
  if (!bytes) return cudaSuccess;
  const uint64_t blocks = std::min<uint64_t>((bytes / 16 + kSumThreads - 1) / kSumThreads + 1, uint64_t(device_sms()) * 8);
  checksum_kernel<<<uint32_t(blocks), kSumThreads, 0, s>>>(static_cast<const uint8_t*>(p), bytes, chunk_id,
                                                            reinterpret_cast<unsigned long long*>(dev_out));
  return cudaGetLastError();
}

cudaError_t launch_zero(void* p, size_t bytes, cudaStream_t s) {
  const size_t n16 = (bytes + 15) / 16;
  if (!n16) return cudaSuccess;
  const uint32_t grid = uint32_t(std::min<size_t>((n16 + kUtilThreads - 1) / kUtilThreads, 148));
  zero_kernel<<<grid, kUtilThreads, 0, s>>>(static_cast<uint4*>(p), uint32_t(n16));
  return cudaGetLastError();
}

cudaError_t launch_harvest(uint32_t* err, uint32_t* host_mapped, uint32_t n, cudaStream_t s) {
  if (!n) return cudaSuccess;
  harvest_kernel<<<1, kUtilThreads, 0, s>>>(err, host_mapped, n);
  return cudaGetLastError();
}

}  // namespace cdm
