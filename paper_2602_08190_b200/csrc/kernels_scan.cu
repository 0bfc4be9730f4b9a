// kernels_scan.cu -- H6: scan-dependent delta decode / VARCHAR offsets in ONE pass.
//
//   DELTA   out[i]   = base + sum_{k<=i} (FOR + bits_k)         (mod 2^bits)
//   OFFSETS out[0] = 0, out[i+1] = sum_{k<=i} (FOR + bits_k)    (lengths -> int32 offsets, reading R17)
//
// The paper decodes delta with PyTorch's cumsum as a separate pass.  Here the
// unpack is fused into a single-pass decoupled look-back scan: one 4096-element tile
// per CTA, tile order from an epoch|ticket counter (predecessors are always resident), the tile's
// packed bytes staged by one TMA bulk copy, a blocked thread-local scan of 16 values, a CTA scan of
// the thread totals, a warp-wide look-back over 32 predecessors at a time, then the results are
// transposed through shared memory so every warp store is a contiguous 16-byte-per-lane write.
#include "device_util.cuh"
#include "kernels.h"

namespace cdm {
namespace {

using namespace dev;

__device__ __forceinline__ int find_desc_scan(const ScanBatch& B, uint32_t tile) {
  int lo = 0, hi = int(B.n) - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (B.d[mid].tile0 <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

constexpr int kPer = kScanTile / kThreads;  // 16 values per thread

__global__ void __launch_bounds__(kThreads) scan_kernel(const __grid_constant__ ScanBatch B) {
  // one buffer: the staged packed tile, then (after the CTA scan) the transposed results
  __shared__ __align__(128) uint64_t buf_s[(kScanTile * 8 + 32) / 8];
  uint8_t* packed_s = reinterpret_cast<uint8_t*>(buf_s);
  uint64_t* res_s = buf_s;
  __shared__ uint64_t warp_s[kThreads / 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tile_s, epoch_s;
  __shared__ uint64_t prefix_s;
  const uint32_t tid = threadIdx.x;

  if (tid == 0) {
    uint32_t t, e;
    take_ticket(B.ticket, B.total_tiles - 1, &t, &e);
    tile_s = t;
    epoch_s = e;
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t gt = tile_s, epoch = epoch_s;
  if (gt >= B.total_tiles) return;
  trace_stamp(B.trace, gt, 0);
  trace_stamp(B.trace, gt, 7);
  const ScanDesc& D = B.d[find_desc_scan(B, gt)];
  const uint32_t lt = gt - D.tile0;
  const uint32_t w = D.w;
  const uint64_t tile_start = uint64_t(lt) * kScanTile;
  const uint32_t valid = uint32_t(min(uint64_t(kScanTile), uint64_t(D.n) - tile_start));

  if (tid == 0) {
    const uint64_t stream_bytes = ((uint64_t(D.n) * w + 7) / 8 + 15) & ~15ull;
    const uint64_t start = tile_start / 8 * w;
    const uint64_t want = uint64_t(kScanTile / 8) * w;
    const uint64_t have = stream_bytes > start ? stream_bytes - start : 0ull;
    const uint32_t nb = uint32_t(want < have ? want : have);
    mbar_arrive_expect_tx(&bar, nb);
    if (nb) tma_load_1d(packed_s, D.packed + start, nb, &bar);
  }
  mbar_wait(&bar, 0);

  // blocked: thread t owns values [16t, 16t+16)
  const uint32_t* wd = reinterpret_cast<const uint32_t*>(packed_s);
  uint64_t v[kPer];
  uint64_t run = 0;
#pragma unroll
  for (int j = 0; j < kPer; j++) {
    const uint32_t i = tid * kPer + j;
    const uint64_t x = (i < valid) ? D.for_base + (w ? extract_bits(wd, uint64_t(i) * w, w) : 0ull) : 0ull;
    run += x;
    v[j] = run;  // inclusive within the thread
  }
  trace_stamp(B.trace, gt, 1);
  uint64_t tile_total;
  const uint64_t texcl = block_excl_scan_u64<kThreads>(run, warp_s, &tile_total);
  trace_stamp(B.trace, gt, 2);

  // decoupled look-back (warp 0)
  if (tid < 32) {
    uint64_t pc, p0;
    lb_tile(B.lb, gt, D.tile0, epoch, 0, tile_total, &pc, &p0);
    trace_stamp(B.trace, gt, 3);
    if (tid == 0) {
      prefix_s = p0;
      if (D.mode == SCAN_OFFSETS && lt + 1 == D.ntiles && p0 + tile_total != D.base)
        atomicOr(B.err + D.err_idx, 0x8u);  // lengths do not sum to the payload (CDM_ERR_LENGTHS)
    }
  }
  __syncthreads();
  const uint64_t add = (D.mode == SCAN_DELTA ? D.base : 0ull) + prefix_s + texcl;
#pragma unroll
  for (int j = 0; j < kPer; j++) res_s[tid * kPer + j] = add + v[j];
  __syncthreads();

  if (D.mode == SCAN_DELTA) {
    // striped: thread t stores values k*1024 + 4t .. +3 (16 or 32 contiguous bytes per lane)
#pragma unroll
    for (uint32_t k = 0; k < 4; k++) {
      const uint32_t i0 = k * 1024 + tid * 4;
      if (i0 >= valid) break;
      const uint64_t gi = tile_start + i0;
      if (D.out_bytes == 8) {
        uint64_t* o = reinterpret_cast<uint64_t*>(D.out) + gi;
        if (i0 + 4 <= valid) {
          st_v2_u64(o, res_s[i0], res_s[i0 + 1]);
          st_v2_u64(o + 2, res_s[i0 + 2], res_s[i0 + 3]);
        } else {
#pragma unroll
          for (uint32_t j = 0; j < 4; j++) if (i0 + j < valid) o[j] = res_s[i0 + j];
        }
      } else {
        uint32_t* o = reinterpret_cast<uint32_t*>(D.out) + gi;
        if (i0 + 4 <= valid) {
          st_v4_u32(o, uint32_t(res_s[i0]), uint32_t(res_s[i0 + 1]), uint32_t(res_s[i0 + 2]), uint32_t(res_s[i0 + 3]));
        } else {
#pragma unroll
          for (uint32_t j = 0; j < 4; j++) if (i0 + j < valid) o[j] = uint32_t(res_s[i0 + j]);
        }
      }
    }
  } else {
    // offsets[i+1] = inclusive sum; offsets[0] = 0 written by the chunk's first tile
    int32_t* o = reinterpret_cast<int32_t*>(D.out) + tile_start + 1;
    for (uint32_t i = tid; i < valid; i += kThreads) o[i] = int32_t(uint32_t(res_s[i]));
    if (lt == 0 && tid == 0) reinterpret_cast<int32_t*>(D.out)[0] = 0;
  }
  __syncthreads();
  trace_stamp(B.trace, gt, 4);
}

}  // namespace

cudaError_t launch_scan(const ScanBatch& b, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  scan_kernel<<<b.total_tiles, kThreads, 0, s>>>(b);
  return cudaGetLastError();
}

}  // namespace cdm
