// kernels_strdict.cu -- NEXT-2: String-dictionary decode (reading R34).
//
// The paper puts String-dictionary in the Group-Parallel (RLE) family: every token occurrence is a
// group whose items are the bytes of its dictionary entry, and the group offsets are the prefix sum of the
// token lengths (P:276's presum).  Three launches per batch, all on the chunk-sequential family's stream:
//   sd_sums   one CTA per 2048-token tile: unpack the w-bit ids, look up the lengths, tile byte sum;
//   sd_scan   one CTA per descriptor: exclusive scan of its tile sums in place (a few thousand values);
//   sd_expand one CTA per tile: ids -> (dictionary offset, length), block scan of the lengths gives every
//             token's byte position in the tile; the bytes are assembled in shared memory at the tile's
//             global alignment (the staged image and the output agree mod 16) and leave as aligned 16-byte
//             stores, the two partial edge words byte by byte; tiles of more than 32 KB store directly.
// The dictionary offsets were checked on the host (0, non-decreasing, ending at the token bytes), so a
// token id < entries always names bytes inside the dictionary; an id >= entries sets CDM_ERR_DICT_INDEX and
// expands to nothing; tokens that do not total the node's bytes set CDM_ERR_LENGTHS and a tile that would
// end past them writes nothing.
#include "device_util.cuh"
#include "kernels.h"

namespace cdm {
namespace {

using namespace dev;

constexpr int kSdPer = kSdTile / kThreads;  // 8 tokens per thread

__device__ __forceinline__ int find_desc_sd(const SdBatch& B, uint32_t tile) {
  int lo = 0, hi = int(B.n) - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (B.d[mid].tile0 <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// this thread's tokens kb .. kb + 7 of the tile: dictionary offsets and lengths (0 for a bad id)
__device__ __forceinline__ uint32_t load_tokens(const SdDesc& D, uint32_t g0, uint32_t nt, uint32_t kb,
                                                uint32_t (&a)[kSdPer], uint32_t (&len)[kSdPer], bool& bad) {
  const uint32_t* offs = reinterpret_cast<const uint32_t*>(D.dict);
  const uint32_t* pk = reinterpret_cast<const uint32_t*>(D.ids_packed);
  uint32_t sum = 0;
#pragma unroll
  for (int r = 0; r < kSdPer; r++) {
    a[r] = 0;
    len[r] = 0;
    const uint32_t k = kb + r;
    if (k < nt) {
      const uint64_t id = D.id_base + extract_bits_global(pk, uint64_t(g0 + k) * D.w, D.w);
      if (id < D.entries) {
        a[r] = __ldg(offs + id);
        len[r] = __ldg(offs + id + 1) - a[r];
      } else {
        bad = true;
      }
    }
    sum += len[r];
  }
  return sum;
}

__global__ void __launch_bounds__(kThreads) sd_sums_kernel(const __grid_constant__ SdBatch B) {
  __shared__ uint64_t warp_s[kThreads / 32];
  const SdDesc& D = B.d[find_desc_sd(B, blockIdx.x)];
  const uint32_t lt = blockIdx.x - D.tile0, g0 = lt * kSdTile;
  const uint32_t nt = min(uint32_t(kSdTile), D.ntok - g0);
  uint32_t a[kSdPer], len[kSdPer];
  bool bad = false;
  const uint64_t s = load_tokens(D, g0, nt, threadIdx.x * kSdPer, a, len, bad);
  uint64_t tot;
  block_excl_scan_u64<kThreads>(s, warp_s, &tot);
  if (threadIdx.x == 0) D.tsum[lt] = tot;
  if (bad) atomicOr(B.err + D.err_idx, 0x1u);
}

// one CTA per descriptor: tsum <- exclusive prefix of tsum (the tile's output offset)
__global__ void __launch_bounds__(kThreads) sd_scan_kernel(const __grid_constant__ SdBatch B) {
  __shared__ uint64_t warp_s[kThreads / 32];
  const SdDesc& D = B.d[blockIdx.x];
  uint64_t carry = 0;
  for (uint32_t i0 = 0; i0 < D.ntiles; i0 += kThreads) {
    const uint32_t i = i0 + threadIdx.x;
    const uint64_t v = i < D.ntiles ? D.tsum[i] : 0ull;
    uint64_t tot;
    const uint64_t ex = block_excl_scan_u64<kThreads>(v, warp_s, &tot);
    if (i < D.ntiles) D.tsum[i] = carry + ex;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && carry != D.n_out) atomicOr(B.err + D.err_idx, 0x8u);
}

__global__ void __launch_bounds__(kThreads) sd_expand_kernel(const __grid_constant__ SdBatch B) {
  __shared__ __align__(16) uint8_t stage_s[kSdStage + 32];
  __shared__ uint64_t warp_s[kThreads / 32];
  const SdDesc& D = B.d[find_desc_sd(B, blockIdx.x)];
  const uint32_t lt = blockIdx.x - D.tile0, g0 = lt * kSdTile;
  const uint32_t nt = min(uint32_t(kSdTile), D.ntok - g0);
  const uint32_t kb = threadIdx.x * kSdPer;
  uint32_t a[kSdPer], len[kSdPer];
  bool bad = false;
  const uint64_t s = load_tokens(D, g0, nt, kb, a, len, bad);
  uint64_t T;
  const uint32_t ex = uint32_t(block_excl_scan_u64<kThreads>(s, warp_s, &T));
  const uint64_t O64 = __ldcg(D.tsum + lt);
  if (O64 + T > D.n_out) return;  // inconsistent lengths (sd_scan reports them): never write outside
  const uint32_t O = uint32_t(O64), Tt = uint32_t(T);
  const uint8_t* tok = D.dict + 4ull * (D.entries + 1ull);
  uint8_t* const out = D.out;
  if (Tt > kSdStage) {  // long tokens: direct byte stores
    uint32_t p = O + ex;
#pragma unroll
    for (int r = 0; r < kSdPer; r++) {
      for (uint32_t j = 0; j < len[r]; j++) out[p + j] = __ldg(tok + a[r] + j);
      p += len[r];
    }
    return;
  }
  // staged image: stage_s[sh + q] = tile byte q, sh = O mod 16, so stage word i is output word (O - sh)/16 + i
  const uint32_t sh = O & 15u;
  uint32_t p = sh + ex;
#pragma unroll
  for (int r = 0; r < kSdPer; r++) {
    const uint8_t* src = tok + a[r];
    for (uint32_t j = 0; j < len[r]; j++) stage_s[p + j] = __ldg(src + j);
    p += len[r];
  }
  __syncthreads();
  const uint32_t nw = (sh + Tt + 15) / 16;
  uint4* const ow = reinterpret_cast<uint4*>(out + (O - sh));
  const uint4* const sw = reinterpret_cast<const uint4*>(stage_s);
  for (uint32_t i = threadIdx.x; i < nw; i += kThreads) {
    const uint32_t lo = 16 * i, hi = lo + 16;
    if (lo >= sh && hi <= sh + Tt) {
      ow[i] = sw[i];
    } else {  // an edge word shared with the neighbouring tiles: only this tile's bytes
      uint8_t* const ob = reinterpret_cast<uint8_t*>(ow + i);
      for (uint32_t q = max(lo, sh); q < min(hi, sh + Tt); q++) ob[q - lo] = stage_s[q];
    }
  }
}

}  // namespace

cudaError_t launch_strdict(const SdBatch& b, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  sd_sums_kernel<<<b.total_tiles, kThreads, 0, s>>>(b);
  sd_scan_kernel<<<b.n, kThreads, 0, s>>>(b);
  sd_expand_kernel<<<b.total_tiles, kThreads, 0, s>>>(b);
  return cudaGetLastError();
}

}  // namespace cdm
