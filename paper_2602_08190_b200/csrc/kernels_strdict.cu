// kernels_strdict.cu -- NEXT-2: String-dictionary decode (reading R34).
//
// The paper puts String-dictionary in the Group-Parallel (RLE) family: every token occurrence is a
// group whose items are the bytes of its dictionary entry, and the group offsets are the prefix sum of the
// token lengths (P:276's presum).  Three launches per batch, all on the chunk-sequential family's stream:
//   sd_sums   one CTA per 2048-token tile: stage the w-bit ids (coalesced), look up the lengths, tile sum;
//   sd_scan   one CTA per descriptor: exclusive scan of its tile sums in place (a few thousand values);
//   sd_expand_b (default) persistent CTAs over contiguous tile ranges with the chunk's dictionary in shared
//             memory once per chunk; a block scan of the lengths places every token; each thread copies its 4
//             tokens' bytes into a shared image at the tile's global alignment, which leaves as aligned 16-byte
//             stores.  Tested alternatives (CDM_SD_EXPAND=1 / 2, measured slower): round 1's per-tile sd_expand
//             (word assembly in registers, dictionary through L1) and the word-parallel sd_expand2.
// The dictionary offsets were checked on the host (0, non-decreasing, ending at the token bytes), so a
// token id < entries always names bytes inside the dictionary; an id >= entries sets CDM_ERR_DICT_INDEX and
// expands to nothing; tokens that do not total the node's bytes set CDM_ERR_LENGTHS and a tile that would
// end past them writes nothing.
#include "device_util.cuh"
#include "kernels.h"

#include <algorithm>
#include <cstdlib>

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

constexpr uint32_t kIdsWords = kSdTile * 32 / 32 + 4;  // packed ids of one tile (w <= 32) + extraction slack

// dictionary stream (offsets + token bytes) of descriptor D -> shared memory (16-byte copies)
__device__ __forceinline__ void load_dict(const SdDesc& D, uint32_t bytes, uint32_t* dict_s) {
  const uint4* src = reinterpret_cast<const uint4*>(D.dict);
  for (uint32_t i = threadIdx.x; i < (bytes + 15) / 16; i += blockDim.x) reinterpret_cast<uint4*>(dict_s)[i] = __ldg(src + i);
}

// this thread's tokens kb .. kb + 7 of a tile (ids staged in shared words): dictionary offsets and lengths
// (0 for a bad id).  `offs` is the dictionary in shared memory or global memory (generic loads).
// A thread's N consecutive w-bit ids (w <= 32) from staged words through a sliding two-word window (one shared load
// per 32 bits consumed instead of a 64-bit extraction per id); ids past nt read as 0.
template <int N>
__device__ __forceinline__ void window_ids(const uint32_t* ids_s, uint32_t kb, uint32_t nt, uint32_t w, uint32_t (&f)[N]) {
  if (w == 0) {
#pragma unroll
    for (int r = 0; r < N; r++) f[r] = 0;
    return;
  }
  const uint32_t m = w >= 32 ? 0xFFFFFFFFu : (1u << w) - 1u;
  uint32_t q = (kb * w) >> 5, sh = (kb * w) & 31;  // kb * w < 2^32: a tile holds 2048 ids of <= 32 bits
  uint32_t lo = ids_s[q], hi = ids_s[q + 1];
#pragma unroll
  for (int r = 0; r < N; r++) {
    f[r] = kb + r < nt ? __funnelshift_r(lo, hi, sh) & m : 0u;
    sh += w;
    if (sh >= 32) {
      sh -= 32;
      q++;
      lo = hi;
      hi = kb + r + 1 < nt ? ids_s[q + 1] : 0u;  // (stage_bits copies two words past the last id)
    }
  }
}

__device__ __forceinline__ uint32_t load_tokens(const SdDesc& D, const uint32_t* offs, const uint32_t* ids_s, uint32_t nt,
                                                uint32_t kb, uint32_t (&a)[kSdPer], uint32_t (&len)[kSdPer], bool& bad) {
  const uint32_t w = D.w;
  uint32_t sum = 0;
  uint32_t fid[kSdPer];
  window_ids<kSdPer>(ids_s, kb, nt, w, fid);
#pragma unroll
  for (int r = 0; r < kSdPer; r++) {
    a[r] = 0;
    len[r] = 0;
    const uint32_t k = kb + r;
    if (k < nt) {
      const uint64_t id = D.id_base + fid[r];
      if (id < D.entries) {
        a[r] = offs[id];
        len[r] = offs[id + 1] - a[r];
      } else {
        bad = true;
      }
    }
    sum += len[r];
  }
  return sum;
}

// one CTA per tile; the dictionary offsets are read through L1 (a shared copy per CTA or persistent CTAs
// with one copy measured slower: 0.30 vs 0.25 ms, o_comment SF 10)
__global__ void __launch_bounds__(kThreads) sd_sums_kernel(const __grid_constant__ SdBatch B) {
  __shared__ uint32_t ids_s[kIdsWords];
  __shared__ uint64_t warp_s[kThreads / 32];
  const SdDesc& D = B.d[find_desc_sd(B, blockIdx.x)];
  const uint32_t lt = blockIdx.x - D.tile0, g0 = lt * kSdTile;
  const uint32_t nt = min(uint32_t(kSdTile), D.ntok - g0);
  stage_bits<kThreads>(ids_s, D.ids_packed, g0, nt, D.w);
  __syncthreads();
  uint32_t a[kSdPer], len[kSdPer];
  bool bad = false;
  const uint64_t s = load_tokens(D, reinterpret_cast<const uint32_t*>(D.dict), ids_s, nt, threadIdx.x * kSdPer, a,
                                 len, bad);
  uint64_t tot;
  block_excl_scan_u64<kThreads>(s, warp_s, &tot);
  if (threadIdx.x == 0) D.tsum[lt] = tot;
  if (bad) atomicOr(B.err + D.err_idx, 0x1u);
}

// one CTA per descriptor: tsum <- exclusive prefix of tsum (the tile's output offset); thread t scans a
// contiguous segment, so the loads of a segment are independent
__global__ void __launch_bounds__(kThreads) sd_scan_kernel(const __grid_constant__ SdBatch B) {
  __shared__ uint64_t warp_s[kThreads / 32];
  const SdDesc& D = B.d[blockIdx.x];
  const uint32_t per = (D.ntiles + kThreads - 1) / kThreads;
  const uint32_t i0 = min(D.ntiles, threadIdx.x * per), i1 = min(D.ntiles, i0 + per);
  uint64_t s = 0;
  for (uint32_t i = i0; i < i1; i++) s += __ldcg(D.tsum + i);
  uint64_t tot;
  uint64_t run = block_excl_scan_u64<kThreads>(s, warp_s, &tot);
  for (uint32_t i = i0; i < i1; i++) {
    const uint64_t v = __ldcg(D.tsum + i);
    D.tsum[i] = run;
    run += v;
  }
  if (threadIdx.x == 0 && tot != D.n_out) atomicOr(B.err + D.err_idx, 0x8u);
}

// sd_expand (one CTA per tile; the dictionary is read through L1): a thread's 8 tokens are contiguous in the
// output, so it builds the 32-bit words of its byte range one at a time (4 dictionary bytes per token piece:
// two aligned dictionary words + a funnel shift) and stores them into the zeroed shared image; only its
// first and last words, shared with the neighbouring threads, are merged with shared-memory atomicOr.
__global__ void __launch_bounds__(kThreads) sd_expand_kernel(const __grid_constant__ SdBatch B) {
  extern __shared__ __align__(16) uint32_t dict_s[];  // B.dict_smem > 0: this tile's dictionary
  __shared__ __align__(16) uint32_t stage_s[(kSdStage + 32) / 4];
  __shared__ uint32_t ids_s[kIdsWords];
  __shared__ uint64_t warp_s[kThreads / 32];
  const SdDesc& D = B.d[find_desc_sd(B, blockIdx.x)];
  const uint32_t lt = blockIdx.x - D.tile0, g0 = lt * kSdTile;
  const uint32_t nt = min(uint32_t(kSdTile), D.ntok - g0);
  const uint32_t kb = threadIdx.x * kSdPer;
  stage_bits<kThreads>(ids_s, D.ids_packed, g0, nt, D.w);
  const uint64_t O64 = __ldcg(D.tsum + lt);
  const uint32_t sh = uint32_t(O64) & 15u;
  for (uint32_t i = threadIdx.x; i < (kSdStage + 32) / 16; i += kThreads)
    reinterpret_cast<uint4*>(stage_s)[i] = make_uint4(0u, 0u, 0u, 0u);
  const uint32_t* offs = reinterpret_cast<const uint32_t*>(D.dict);
  if (B.dict_smem) {
    load_dict(D, 4u * (D.entries + 1u) + __ldg(offs + D.entries), dict_s);
    offs = dict_s;
  }
  __syncthreads();
  uint32_t a[kSdPer], len[kSdPer];
  bool bad = false;
  const uint32_t s = load_tokens(D, offs, ids_s, nt, kb, a, len, bad);
  uint64_t T;
  const uint32_t ex = uint32_t(block_excl_scan_u64<kThreads>(s, warp_s, &T));
  if (O64 + T > D.n_out) return;  // inconsistent lengths (sd_scan reports them): never write outside
  const uint32_t O = uint32_t(O64), Tt = uint32_t(T);
  const uint32_t* tw = offs + D.entries + 1u;  // token bytes, 4-byte aligned
  uint8_t* const out = D.out;
  if (Tt > kSdStage) {  // long tokens: direct byte stores
    const uint8_t* tb = reinterpret_cast<const uint8_t*>(tw);
    uint32_t p = O + ex;
#pragma unroll
    for (int r = 0; r < kSdPer; r++) {
      for (uint32_t j = 0; j < len[r]; j++) out[p + j] = tb[a[r] + j];
      p += len[r];
    }
    return;
  }
  // staged image: stage byte sh + q = tile byte q, so stage word i (16 B) is output word (O - sh)/16 + i.
  // Word-driven: the thread walks the 4-byte words of its range [P, P + s); each word takes 4 dictionary
  // bytes from each token it overlaps (usually one or two); consumed tokens shift out of the register arrays.
  if (s) {
    const uint32_t P = sh + ex, Pe = P + s;
    uint32_t tpos = P;
    auto shift = [&]() {
#pragma unroll
      for (int r = 0; r + 1 < kSdPer; r++) { a[r] = a[r + 1]; len[r] = len[r + 1]; }
      len[kSdPer - 1] = 0;
    };
#pragma unroll 1
    for (int g = 0; g < kSdPer && len[0] == 0; g++) shift();
#pragma unroll 1
    for (uint32_t wpos = P & ~3u; wpos < Pe; wpos += 4) {
      uint32_t word = 0;
      uint32_t b = max(wpos, P);
      const uint32_t be = min(wpos + 4u, Pe);
#pragma unroll 1
      while (b < be) {
        const uint32_t off = a[0] + (b - tpos);
        const uint32_t piece = __funnelshift_r(tw[off >> 2], tw[(off >> 2) + 1], (off & 3u) * 8u);
        const uint32_t m = min(be - b, tpos + len[0] - b);
        word |= (m >= 4u ? piece : piece & ((1u << (8u * m)) - 1u)) << (8u * (b - wpos));
        b += m;
        if (b == tpos + len[0]) {  // next non-empty token of this thread
          tpos += len[0];
          shift();
#pragma unroll 1
          for (int g = 0; g < kSdPer && len[0] == 0 && b < Pe; g++) shift();
        }
      }
      if (wpos < P || wpos + 4u > Pe) atomicOr(stage_s + (wpos >> 2), word);  // shared with a neighbour
      else stage_s[wpos >> 2] = word;
    }
  }
  __syncthreads();
  const uint32_t nw = (sh + Tt + 15) / 16;
  uint4* const ow = reinterpret_cast<uint4*>(out + (O - sh));
  const uint4* const sw = reinterpret_cast<const uint4*>(stage_s);
  const uint8_t* const sb = reinterpret_cast<const uint8_t*>(stage_s);
  for (uint32_t i = threadIdx.x; i < nw; i += kThreads) {
    const uint32_t lo = 16 * i, hi = lo + 16;
    if (lo >= sh && hi <= sh + Tt) {
      ow[i] = sw[i];
    } else {  // an edge word shared with the neighbouring tiles: only this tile's bytes
      uint8_t* const ob = reinterpret_cast<uint8_t*>(ow + i);
      for (uint32_t q = max(lo, sh); q < min(hi, sh + Tt); q++) ob[q - lo] = sb[q];
    }
  }
}

// sd_expand2 (opt-in, CDM_SD_EXPAND=2; measured slower, see launch_strdict): word-parallel, the paper's Group-Parallel item loop turned around -- every output
// word is an item, found in its group (token) by rank.  Per tile: the block scan of (non-empty tokens << 32 |
// bytes) places every non-empty token (start position, dictionary offset; a sentinel end) in shared arrays and
// marks its start in a bitmap; per-bitmap-word prefix counts make rank(p) = #starts <= p one popcount away.
// Thread i then builds staged 32-bit word i: the token holding its first byte by rank, 4 dictionary bytes
// per piece (two aligned words + a funnel shift), the next token when this one ends -- consecutive lanes take
// consecutive words (no divergence beyond the 1-2 pieces a word needs, no atomics: a word has one owner).
// The dictionary (offsets + token bytes) is copied into shared memory once per CTA of kSdCtaTiles tiles
// (bank conflicts instead of one L1 wavefront per distinct line); larger ones are read through L1.
constexpr int kSdT2 = 512;                      // threads per CTA
constexpr int kSdPer2 = kSdTile / kSdT2;        // 4 tokens per thread
constexpr uint32_t kSdBmWords = kSdStage / 32 + 2;

__global__ void __launch_bounds__(kSdT2) sd_expand2_kernel(const __grid_constant__ SdBatch B) {
  extern __shared__ __align__(16) uint32_t dyn_s[];  // stage image, then (B.dict_smem) the dictionary
  uint32_t* const stage_s = dyn_s;
  uint32_t* const dict_s = dyn_s + (kSdStage + 32) / 4;
  __shared__ uint32_t ids_s[kIdsWords];
  __shared__ uint32_t pos_s[kSdTile + 1], a_s[kSdTile];
  __shared__ uint32_t bm_s[kSdBmWords], cnt_s[kSdBmWords];
  __shared__ uint64_t warp_s[kSdT2 / 32];
  const uint32_t tid = threadIdx.x;
  // this CTA's descriptor and tiles
  int lo = 0, hi = int(B.n) - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (B.d[mid].cta0 <= blockIdx.x) lo = mid; else hi = mid - 1;
  }
  const SdDesc& D = B.d[lo];
  const uint32_t t0 = (blockIdx.x - D.cta0) * kSdCtaTiles, t1 = min(D.ntiles, t0 + kSdCtaTiles);
  const uint32_t* offs = reinterpret_cast<const uint32_t*>(D.dict);
  if (B.dict_smem) {
    load_dict(D, 4u * (D.entries + 1u) + __ldg(offs + D.entries), dict_s);
    offs = dict_s;
  }
  const uint32_t* tw = offs + D.entries + 1u;  // token bytes, 4-byte aligned
  const uint32_t kb = tid * kSdPer2;
  for (uint32_t lt = t0; lt < t1; lt++) {
    const uint32_t g0 = lt * kSdTile;
    const uint32_t nt = min(uint32_t(kSdTile), D.ntok - g0);
    __syncthreads();  // previous tile's arrays are dead (and the dictionary copy is complete)
    stage_bits<kSdT2>(ids_s, D.ids_packed, g0, nt, D.w);
    for (uint32_t i = tid; i < kSdBmWords; i += kSdT2) bm_s[i] = 0u;
    __syncthreads();
    uint32_t a[kSdPer2], len[kSdPer2];
    uint32_t s = 0, ne = 0;
#pragma unroll
    for (int r = 0; r < kSdPer2; r++) {
      a[r] = 0;
      len[r] = 0;
      const uint32_t k = kb + r;
      if (k < nt) {
        const uint64_t id = D.id_base + extract_bits(ids_s, uint64_t(k) * D.w, D.w);
        if (id < D.entries) {
          a[r] = offs[id];
          len[r] = offs[id + 1] - a[r];
        }
      }
      s += len[r];
      ne += len[r] != 0u;
    }
    uint64_t T;
    const uint64_t ex = block_excl_scan_u64<kSdT2>((uint64_t(ne) << 32) | s, warp_s, &T);
    const uint64_t O64 = __ldcg(D.tsum + lt);
    const uint32_t Tt = uint32_t(T), NE = uint32_t(T >> 32);
    if (O64 + Tt > D.n_out) continue;  // inconsistent lengths (sd_scan reports them): never write outside
    const uint32_t O = uint32_t(O64), sh = O & 15u;
    uint8_t* const out = D.out;
    if (Tt > kSdStage) {  // long tokens: direct byte stores
      const uint8_t* tb = reinterpret_cast<const uint8_t*>(tw);
      uint32_t p = O + uint32_t(ex);
#pragma unroll
      for (int r = 0; r < kSdPer2; r++) {
        for (uint32_t j = 0; j < len[r]; j++) out[p + j] = tb[a[r] + j];
        p += len[r];
      }
      continue;
    }
    {  // non-empty tokens: start position (stage coordinates), dictionary offset, start bit
      uint32_t p = sh + uint32_t(ex), k = uint32_t(ex >> 32);
#pragma unroll
      for (int r = 0; r < kSdPer2; r++) {
        if (len[r]) {
          pos_s[k] = p;
          a_s[k] = a[r];
          atomicOr(bm_s + (p >> 5), 1u << (p & 31));
          k++;
        }
        p += len[r];
      }
      if (tid == 0) pos_s[NE] = sh + Tt;  // sentinel: the end of the last token
    }
    __syncthreads();
    const uint32_t nbw = (sh + Tt + 31) / 32;
    {  // cnt_s[j] = number of token starts in bitmap words < j (two words per thread)
      const uint32_t j0 = 2 * tid;
      const uint32_t c0 = j0 < nbw ? __popc(bm_s[j0]) : 0u, c1 = j0 + 1 < nbw ? __popc(bm_s[j0 + 1]) : 0u;
      uint64_t tot;
      const uint32_t e = uint32_t(block_excl_scan_u64<kSdT2>(c0 + c1, warp_s, &tot));
      if (j0 < nbw) cnt_s[j0] = e;
      if (j0 + 1 < nbw) cnt_s[j0 + 1] = e + c0;
    }
    __syncthreads();
    const uint32_t end = sh + Tt, nw4 = (end + 3) / 4;
    for (uint32_t i = (sh >> 2) + tid; i < nw4; i += kSdT2) {
      uint32_t b = max(4 * i, sh);
      const uint32_t be = min(4 * i + 4, end);
      const uint32_t wj = b >> 5;
      uint32_t k = cnt_s[wj] + __popc(bm_s[wj] & uint32_t((2ull << (b & 31)) - 1ull)) - 1u;
      uint32_t word = 0;
      while (b < be) {
        const uint32_t ts = pos_s[k], te = pos_s[k + 1];
        const uint32_t off = a_s[k] + (b - ts);
        const uint32_t piece = __funnelshift_r(tw[off >> 2], tw[(off >> 2) + 1], (off & 3u) * 8u);
        const uint32_t m = min(be, te) - b;
        word |= (m >= 4u ? piece : piece & ((1u << (8u * m)) - 1u)) << (8u * (b - 4 * i));
        b += m;
        k++;
      }
      stage_s[i] = word;
    }
    __syncthreads();
    const uint32_t nw = (end + 15) / 16;
    uint4* const ow = reinterpret_cast<uint4*>(out + (O - sh));
    const uint4* const sw = reinterpret_cast<const uint4*>(stage_s);
    const uint8_t* const sb = reinterpret_cast<const uint8_t*>(stage_s);
    for (uint32_t i = tid; i < nw; i += kSdT2) {
      const uint32_t lo16 = 16 * i, hi16 = lo16 + 16;
      if (lo16 >= sh && hi16 <= end) {
        ow[i] = sw[i];
      } else {  // an edge word shared with the neighbouring tiles: only this tile's bytes
        uint8_t* const ob = reinterpret_cast<uint8_t*>(ow + i);
        for (uint32_t q = max(lo16, sh); q < min(hi16, end); q++) ob[q - lo16] = sb[q];
      }
    }
  }
}

// sd_expand_b (CDM_SD_EXPAND=3): persistent CTAs over contiguous tile ranges, the chunk's dictionary (offsets +
// token bytes) in shared memory once per chunk, and the simplest possible copy: each thread moves its 4 tokens'
// bytes one byte at a time from the shared dictionary into the shared output image (one LDS.U8 + one STS.U8 per
// byte; no word assembly, no atomics: every image byte has one writer), which leaves as 16-byte stores.
constexpr int kSdBT = 512;                  // threads per CTA
constexpr int kSdBPer = kSdTile / kSdBT;    // 4 tokens per thread

__global__ void __launch_bounds__(kSdBT) sd_expand_b_kernel(const __grid_constant__ SdBatch B) {
  extern __shared__ __align__(16) uint32_t dyn_s[];  // stage image, then the dictionary (B.dict_smem > 0)
  uint8_t* const stage_b = reinterpret_cast<uint8_t*>(dyn_s);
  uint32_t* const dict_s = dyn_s + (kSdStage + 32) / 4;
  __shared__ uint32_t ids2_s[2][kIdsWords];
  __shared__ uint64_t warp_s[kSdBT / 32];
  const uint32_t tid = threadIdx.x;
  const uint32_t per = (B.total_tiles + gridDim.x - 1) / gridDim.x;
  const uint32_t t0 = blockIdx.x * per, t1 = min(B.total_tiles, t0 + per);
  int di = -1;
  const uint32_t* offs = nullptr;
  // the next tile's packed ids and output offset are loaded into registers while this tile expands, and
  // written to the other ids buffer at the top of the next iteration (their latency hides behind a tile)
  constexpr int kPre = (kIdsWords + kSdBT - 1) / kSdBT;
  uint32_t pre[kPre];
  uint64_t pre_o = 0;
  int dnext = t0 < t1 ? find_desc_sd(B, t0) : 0, dcur = dnext;  // tiles increase: descriptors move forward
  auto issue = [&](uint32_t t) {
    while (dnext + 1 < int(B.n) && B.d[dnext + 1].tile0 <= t) dnext++;
    const SdDesc& Dn = B.d[dnext];
    const uint32_t ltn = t - Dn.tile0, ntn = min(uint32_t(kSdTile), Dn.ntok - ltn * kSdTile);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(Dn.ids_packed) + ((uint64_t(ltn) * kSdTile * Dn.w) >> 5);
    const uint32_t nw = Dn.w ? uint32_t((uint64_t(ntn) * Dn.w + 31) / 32) + 2 : 0u;
#pragma unroll
    for (int i = 0; i < kPre; i++) {
      const uint32_t k = tid + uint32_t(i) * kSdBT;
      pre[i] = k < nw ? __ldg(src + k) : 0u;
    }
    pre_o = __ldcg(Dn.tsum + ltn);
  };
  auto commit = [&](uint32_t buf) {
#pragma unroll
    for (int i = 0; i < kPre; i++) {
      const uint32_t k = tid + uint32_t(i) * kSdBT;
      if (k < kIdsWords) ids2_s[buf][k] = pre[i];
    }
  };
  if (t0 < t1) issue(t0);
  for (uint32_t gt = t0, it = 0; gt < t1; gt++, it++) {
    while (dcur + 1 < int(B.n) && B.d[dcur + 1].tile0 <= gt) dcur++;
    const int dn = dcur;
    const SdDesc& D = B.d[dn];
    uint32_t* const ids_s = ids2_s[it & 1];
    commit(it & 1);   // this tile's ids (its buffer was last read two tiles ago, before the previous barrier)
    const uint64_t O64 = pre_o;
    __syncthreads();  // the previous tile is done with the image (and the dictionary); this tile's ids are in
    if (gt + 1 < t1) issue(gt + 1);
    if (dn != di) {
      di = dn;
      offs = reinterpret_cast<const uint32_t*>(D.dict);
      if (B.dict_smem) {
        const uint4* src = reinterpret_cast<const uint4*>(D.dict);
        const uint32_t bytes = 4u * (D.entries + 1u) + __ldg(offs + D.entries);
        for (uint32_t i = tid; i < (bytes + 15) / 16; i += kSdBT) reinterpret_cast<uint4*>(dict_s)[i] = __ldg(src + i);
        offs = dict_s;
      }
    }
    const uint32_t lt = gt - D.tile0, g0 = lt * kSdTile;
    const uint32_t nt = min(uint32_t(kSdTile), D.ntok - g0);
    __syncthreads();  // the dictionary staged above (when the chunk changed) is complete
    uint32_t a[kSdBPer], len[kSdBPer];
    uint32_t s = 0;
    uint32_t fid[kSdBPer];
    window_ids<kSdBPer>(ids_s, tid * kSdBPer, nt, D.w, fid);
#pragma unroll
    for (int r = 0; r < kSdBPer; r++) {
      a[r] = 0;
      len[r] = 0;
      const uint32_t k = tid * kSdBPer + r;
      if (k < nt) {
        const uint64_t id = D.id_base + fid[r];
        if (id < D.entries) {  // (an out-of-range id was reported by sd_sums: it expands to nothing)
          a[r] = offs[id];
          len[r] = offs[id + 1] - a[r];
        }
      }
      s += len[r];
    }
    uint64_t T;
    const uint32_t ex = uint32_t(block_excl_scan_u64<kSdBT>(s, warp_s, &T));
    if (O64 + T > D.n_out) continue;  // inconsistent lengths (sd_scan reports them): never write outside
    const uint32_t O = uint32_t(O64), Tt = uint32_t(T), sh = O & 15u;
    const uint8_t* tb = reinterpret_cast<const uint8_t*>(offs + D.entries + 1u);  // token bytes
    uint8_t* const out = D.out;
    if (Tt > kSdStage) {  // long tokens: direct byte stores
      uint32_t p = O + ex;
#pragma unroll
      for (int r = 0; r < kSdBPer; r++) {
        for (uint32_t j = 0; j < len[r]; j++) out[p + j] = tb[a[r] + j];
        p += len[r];
      }
      continue;
    }
    // image byte sh + q = tile byte q.  The image is zeroed, then every token is moved 16 bytes at a time (the
    // dictionary read at any alignment: five words + funnel shifts) and written as whole words, its edge words
    // OR-ed in (the neighbouring tokens' bytes in them belong to other threads)
    const uint32_t simg = smem_addr(stage_b);
    for (uint32_t i = tid; 16 * i < sh + Tt; i += kSdBT) sts_v4(simg + 16 * i, make_uint4(0u, 0u, 0u, 0u));
    __syncthreads();
    {
      uint32_t p = simg + sh + ex;
      const bool dsm = B.dict_smem != 0;
      const uint32_t stb = dsm ? smem_addr(tb) : 0u;
#pragma unroll
      for (int r = 0; r < kSdBPer; r++) {
        for (uint32_t t = 0; t < len[r]; t += 16) {
          const uint32_t kk = min(16u, len[r] - t);
          uint32_t v[4];
          if (dsm) sload16(stb + a[r] + t, v);
          else load16<true>(tb + a[r] + t, kk, v);
          sstore16(p + t, v, kk);
        }
        p += len[r];
      }
    }
    __syncthreads();
    const uint32_t end = sh + Tt, nw = (end + 15) / 16;
    uint4* const ow = reinterpret_cast<uint4*>(out + (O - sh));
    const uint4* const swp = reinterpret_cast<const uint4*>(stage_b);
    for (uint32_t i = tid; i < nw; i += kSdBT) {
      const uint32_t lo16 = 16 * i, hi16 = lo16 + 16;
      if (lo16 >= sh && hi16 <= end) {
        ow[i] = swp[i];
      } else {  // an edge word shared with the neighbouring tiles: only this tile's bytes
        uint8_t* const ob = reinterpret_cast<uint8_t*>(ow + i);
        for (uint32_t q = max(lo16, sh); q < min(hi16, end); q++) ob[q - lo16] = stage_b[q];
      }
    }
  }
}

}  // namespace

cudaError_t launch_strdict(const SdBatch& b, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  static bool configured[kMaxDevices] = {};
  const int dev = current_device();
  if (!configured[dev]) {
    cudaFuncSetAttribute(sd_expand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSdDictSmem);
    cudaFuncSetAttribute(sd_expand2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSdStage + 32 + kSdDictSmem);
    configured[dev] = true;
  }
  SdBatch l1 = b;
  l1.dict_smem = 0;
  sd_sums_kernel<<<b.total_tiles, kThreads, 0, s>>>(l1);
  sd_scan_kernel<<<b.n, kThreads, 0, s>>>(b);
  // CDM_SD_EXPAND: 3 (default) sd_expand_b, 1 round 1's per-tile sd_expand (dictionary through L1; 1.62 ms for
  // o_comment SF 10 vs 1.57), 2 the word-parallel sd_expand2 (1.68 ms)
  static const int variant = std::getenv("CDM_SD_EXPAND") ? std::atoi(std::getenv("CDM_SD_EXPAND")) : 3;
  if (variant == 3) {
    static bool conf3[kMaxDevices] = {};
    static int occ3[kMaxDevices] = {};
    const int dev3 = current_device();
    if (!conf3[dev3]) {
      cudaFuncSetAttribute(sd_expand_b_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSdStage + 64 + kSdDictSmem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3[dev3], sd_expand_b_kernel, kSdBT, kSdStage + 64 + kSdDictSmem);
      if (occ3[dev3] < 1) occ3[dev3] = 1;
      conf3[dev3] = true;
    }
    const uint32_t grid = std::min<uint32_t>(b.total_tiles, uint32_t(device_sms() * occ3[dev3]));
    sd_expand_b_kernel<<<grid, kSdBT, kSdStage + 32 + b.dict_smem + (b.dict_smem ? 32 : 0), s>>>(b);
  } else if (variant != 2) {
    sd_expand_kernel<<<b.total_tiles, kThreads, 0, s>>>(l1);
  } else {
    const uint32_t dyn = kSdStage + 32 + b.dict_smem;
    sd_expand2_kernel<<<b.total_ctas, kSdT2, dyn, s>>>(b);
  }
  return cudaGetLastError();
}

}  // namespace cdm
