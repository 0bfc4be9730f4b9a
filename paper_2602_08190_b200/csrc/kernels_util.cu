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

}  // namespace

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
