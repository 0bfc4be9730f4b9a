// kernels_lz4.cu -- H8: chunk-sequential ("Non-Parallel") LZ4 block decode.
//
// The payload of a VARCHAR row group is cut into independent sub-chunks (64 KiB decompressed by
// default), each an LZ4 block (PAPER.md:179 names LZ4 among the LZ77 family; the paper leaves the format
// open -> DESIGN.md reading R16).  The paper's schedule gives ONE THREAD per chunk in SIMT lockstep
// (PAPER.md:329).  On B200 that leaves 31 lanes idle while one lane copies bytes, so this kernel gives one
// WARP per sub-chunk: every lane parses the same token (broadcast loads), literal runs are copied by the
// 32 lanes together, and a match of length L at offset o is copied in parallel with
// out[p + k] = out[p - o + (k mod o)], which is exact even when the match overlaps its own output.
// Every length and offset is bounds-checked; a malformed block sets CDM_ERR_LZ4 and stops that warp.
#include "device_util.cuh"
#include "kernels.h"

namespace cdm {
namespace {

using namespace dev;

constexpr int kWarpsPerCta = 8;

__device__ __forceinline__ int find_desc_lz4(const Lz4Batch& B, uint32_t sub) {
  int lo = 0, hi = int(B.n) - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (B.d[mid].sub0 <= sub) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kWarpsPerCta * 32) lz4_kernel(const __grid_constant__ Lz4Batch B) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gs = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (gs >= B.total_subs) return;
  const Lz4Desc& D = B.d[find_desc_lz4(B, gs)];
  const uint32_t s = gs - D.sub0;
  const uint32_t* tab = reinterpret_cast<const uint32_t*>(D.table);

  // output offset = sum of the preceding sub-chunks' decompressed lengths (warp-parallel)
  uint64_t off = 0;
  for (uint32_t k = lane; k < s; k += 32) off += __ldg(tab + 3 * k + 2);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) off += __shfl_xor_sync(FULL, off, o);
  const uint32_t co = __ldg(tab + 3 * s), cl = __ldg(tab + 3 * s + 1), dl = __ldg(tab + 3 * s + 2);
  bool bad = uint64_t(co) + cl > D.payload_bytes || off + dl > D.n;
  if (s + 1 == D.n_sub && off + dl != D.n) bad = true;
  if (bad) {
    if (lane == 0) atomicOr(B.err + D.err_idx, 0x4u);
    return;
  }
  const uint8_t* __restrict__ in = D.payload + co;
  uint8_t* out = D.out + off;
  uint32_t ip = 0, op = 0;
  for (;;) {
    if (ip >= cl) { bad = true; break; }
    const uint32_t token = __ldg(in + ip++);
    uint32_t lit = token >> 4;
    if (lit == 15) {
      uint32_t b;
      do {
        if (ip >= cl) { bad = true; break; }
        b = __ldg(in + ip++);
        lit += b;
      } while (b == 255);
      if (bad) break;
    }
    if (lit > cl - ip || lit > dl - op) { bad = true; break; }
    for (uint32_t k = lane; k < lit; k += 32) out[op + k] = __ldg(in + ip + k);
    ip += lit;
    op += lit;
    if (ip == cl) break;  // the last sequence carries literals only
    if (cl - ip < 2) { bad = true; break; }
    const uint32_t moff = uint32_t(__ldg(in + ip)) | (uint32_t(__ldg(in + ip + 1)) << 8);
    ip += 2;
    if (moff == 0 || moff > op) { bad = true; break; }
    uint32_t ml = token & 15;
    if (ml == 15) {
      uint32_t b;
      do {
        if (ip >= cl) { bad = true; break; }
        b = __ldg(in + ip++);
        ml += b;
      } while (b == 255);
      if (bad) break;
    }
    ml += 4;
    if (ml > dl - op) { bad = true; break; }
    __syncwarp();  // literal bytes written by other lanes are visible to the match copy
    if (moff >= 32 || moff >= ml) {
      // sources of a 32-byte batch lie before the batch (moff >= 32) -> batches in order
      for (uint32_t base = 0; base < ml; base += 32) {
        const uint32_t k = base + lane;
        if (k < ml) out[op + k] = out[op - moff + k];
        __syncwarp();
      }
    } else {
      // overlapping short period: every lane reads the period window once, then replicates it
      for (uint32_t k = lane; k < ml; k += 32) out[op + k] = out[op - moff + (k % moff)];
    }
    __syncwarp();
    op += ml;
  }
  if (!bad && op != dl) bad = true;
  if (bad && lane == 0) atomicOr(B.err + D.err_idx, 0x4u);
}

}  // namespace

cudaError_t launch_lz4(const Lz4Batch& b, cudaStream_t s) {
  if (!b.total_subs) return cudaSuccess;
  const uint32_t grid = (b.total_subs + kWarpsPerCta - 1) / kWarpsPerCta;
  lz4_kernel<<<grid, kWarpsPerCta * 32, 0, s>>>(b);
  return cudaGetLastError();
}

}  // namespace cdm
