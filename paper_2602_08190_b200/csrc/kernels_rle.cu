// kernels_rle.cu -- H7: scan-dependent ("Group-Parallel") RLE expansion.
//
//   out[offs_g .. offs_g + count_g) = V(g),   offs = exclusive_scan(count)
//
// The paper runs PyTorch cumsum on the counts, then a Group-Parallel kernel whose <L,S,C> geometry lets
// several blocks co-process one big group or one block walk several small groups.  The
// B200 design splits the family into:
//  * rle_sums_kernel: NO look-back, no scan.  Every warp sums one 1024-run tile fully in parallel (sum of
//    counts, plus sum dv*count for arithmetic runs).
//  * rle_kernel: one CTA per tile, no inter-tile dependency: it stages the tile's packed counts and values
//    in shared memory (overlapping rle_sums through programmatic dependent launch), reduces the tile sums
//    before its own into its output offset (no scan kernel, no look-back), computes the run
//    values through the fused nested provider (BitPack, Dict|BitPack, Float2Int|BitPack, arithmetic runs for
//    a root Delta|RLE), scans the counts in the CTA and expands the runs through a run-start bitmap: lane l
//    of a warp owns row 32k + l, finds its run with one popc and stores it (coalesced 32-row stores).
//    A Delta|RLE value lineage (l_orderkey's RLE|[Delta|RLE|[BP,BP],BP]) is two levels of the same kernel:
//    level 0 expands the inner arithmetic runs into the outer run values (an L2-resident u64 array, 1/4 of
//    the output rows for l_orderkey), level 1 expands the outer runs reading them (V_RAW).
//  * rle_big_kernel: tiles with more than kRleBigLimit output rows (giant runs: o_shippriority is one run
//    per chunk) are split into 8192-row pieces over every SM ("multiple GPU blocks
//    co-process a single group"); launched only when a chunk header's max run allows it.
// Invariant checked on the device: sum(count) == n (CDM_ERR_RUN_SUM); writes never leave [0, n).
#include <cstdlib>

#include "device_util.cuh"
#include "kernels.h"

namespace cdm {
namespace {

using namespace dev;

constexpr int K = kRleTile;

__constant__ double kPow10r[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                   1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};

template <typename BatchT>
__device__ __forceinline__ int find_desc(const BatchT& B, uint32_t tile) {
  int lo = 0, hi = int(B.n) - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (B.d[mid].tile0 <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Copy a descriptor from parameter space into shared memory once per CTA (dynamic param indexing would
// re-issue constant-bank loads for every field access).
template <typename T>
__device__ __forceinline__ void stage_desc(T* dst, const T* src) {
  static_assert(sizeof(T) % 4 == 0 && sizeof(T) / 4 <= kThreads, "descriptor copy");
  if (threadIdx.x < sizeof(T) / 4)
    reinterpret_cast<uint32_t*>(dst)[threadIdx.x] = reinterpret_cast<const uint32_t*>(src)[threadIdx.x];
}

// ------------------------------------------------------------------------------------------ expansion
__device__ __forceinline__ uint32_t run_search(const uint32_t* soffs, uint32_t lo, uint32_t hi, uint32_t p) {
  while (lo < hi) {  // last run in [lo, hi] with soffs[run] <= p
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (soffs[mid] <= p) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ uint64_t run_value(const uint64_t* vals, const uint64_t* slopes, const uint32_t* soffs,
                                              uint32_t r, uint32_t p) {
  uint64_t v = vals[r];
  if (slopes) v += uint64_t(p - soffs[r]) * slopes[r];
  return v;
}

__device__ __forceinline__ void store_row(uint8_t* out, uint32_t p, uint64_t v, uint32_t ob) {
  if (ob == 8) reinterpret_cast<uint64_t*>(out)[p] = v;
  else reinterpret_cast<uint32_t*>(out)[p] = uint32_t(v);
}

// Expand tile rows [pb, pe) (tile-relative) of a tile whose runs start at soffs[0..nr] (soffs[0] = 0,
// soffs[nr] = T); element p of run r is vals[r] + (p - soffs[r]) * slopes[r] (slopes == nullptr: plain
// RLE).  `out` points at row 0 of the tile and `gO` is the tile's first global row: rows up to the first
// 4-aligned global row go one per lane, then 128-row windows in which lane l writes rows 4l..4l+3 with one
// 16-byte store (4-byte rows) or two (8-byte rows).  Called by a full warp.
__device__ __forceinline__ void expand_warp(const uint32_t* soffs, uint32_t nr, const uint64_t* vals, const uint64_t* slopes,
                            uint32_t pb, uint32_t pe, uint8_t* out, uint32_t ob, uint32_t gO) {
  const uint32_t lane = threadIdx.x & 31;
  if (pb >= pe || nr == 0) return;
  const uint32_t a = min(pe, pb + ((4u - ((gO + pb) & 3u)) & 3u));
  if (lane < a - pb) {
    const uint32_t p = pb + lane;
    const uint32_t r = run_search(soffs, 0, nr - 1, p);
    store_row(out, p, run_value(vals, slopes, soffs, r, p), ob);
  }
  if (a >= pe) return;
  uint32_t r = run_search(soffs, 0, nr - 1, a);  // run holding the window's first row (warp-uniform)
  for (uint32_t p0 = a; p0 < pe; p0 += 128) {
    // candidate run starts r+1+lane+32k (k = 0..3), every one > p0
    uint32_t contrib[4] = {0u, 0u, 0u, 0u};
    uint32_t cnt127 = 0, cnt128 = 0;
    bool full127 = false, full128 = false;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const uint32_t j = r + 1 + lane + 32 * k;
      const uint32_t c = (j <= nr) ? soffs[j] : 0xFFFFFFFFu;
      const bool in = c <= p0 + 127;
      const uint32_t m = __ballot_sync(FULL, in);
      const uint32_t m2 = __ballot_sync(FULL, c <= p0 + 128);
      cnt127 += __popc(m);
      cnt128 += __popc(m2);
      if (k == 3) { full127 = m == FULL; full128 = m2 == FULL; }
      if (in) {
        const uint32_t pos = c - p0;  // 1..127
#pragma unroll
        for (int wd = 0; wd < 4; wd++)
          if ((pos >> 5) == uint32_t(wd)) contrib[wd] |= 1u << (pos & 31);
      }
    }
    uint32_t M[4];
#pragma unroll
    for (int wd = 0; wd < 4; wd++) M[wd] = __reduce_or_sync(FULL, contrib[wd]);
    const uint32_t distinct = __popc(M[0]) + __popc(M[1]) + __popc(M[2]) + __popc(M[3]);
    const uint32_t q0 = p0 + 4 * lane;  // this lane's rows q0 .. q0+3
    uint64_t v[4];
    if (distinct == cnt127 && !full127) {
      const uint32_t wl = lane >> 3;  // mask word holding rows 4*lane .. 4*lane+3
      uint32_t base = 0;
#pragma unroll
      for (int wd = 0; wd < 3; wd++)
        if (uint32_t(wd) < wl) base += __popc(M[wd]);
      const uint32_t Mw = wl == 0 ? M[0] : wl == 1 ? M[1] : wl == 2 ? M[2] : M[3];
#pragma unroll
      for (int jj = 0; jj < 4; jj++) {
        const uint32_t bit = (4 * lane + jj) & 31;
        const uint32_t rr = r + base + __popc(Mw & (FULL >> (31 - bit)));
        v[jj] = run_value(vals, slopes, soffs, rr, q0 + jj);
      }
    } else {  // zero-length runs or >= 128 starts in the window: per-row search
#pragma unroll
      for (int jj = 0; jj < 4; jj++) {
        const uint32_t q = min(q0 + jj, pe - 1);
        const uint32_t rr = run_search(soffs, r, nr - 1, q);
        v[jj] = run_value(vals, slopes, soffs, rr, q);
      }
    }
    if (q0 + 3 < pe) {
      if (ob == 8) {
        st_v2_u64(reinterpret_cast<uint64_t*>(out) + q0, v[0], v[1]);
        st_v2_u64(reinterpret_cast<uint64_t*>(out) + q0 + 2, v[2], v[3]);
      } else {
        st_v4_u32(reinterpret_cast<uint32_t*>(out) + q0, uint32_t(v[0]), uint32_t(v[1]), uint32_t(v[2]),
                  uint32_t(v[3]));
      }
    } else {
#pragma unroll
      for (int jj = 0; jj < 4; jj++)
        if (q0 + jj < pe) store_row(out, q0 + jj, v[jj], ob);
    }
    r += cnt128;  // run holding row p0 + 128
    if (full128) {
      while (r + 1 <= nr && soffs[r + 1] <= p0 + 128) r++;
    }
  }
}

// ------------------------------------------------------------------------------------------ sums
__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Sums of items [i0, i1) of stream a (and sum of b*a when with_b): lane-strided, 8 items per lane per step
// with all their loads in flight.  Returns the warp totals in every lane; `bad` flags an a > cap.
__device__ __forceinline__ void warp_range_sums(const uint32_t* ap, uint64_t abase, uint32_t aw, const uint32_t* bp,
                                                uint64_t bbase, uint32_t bw, bool with_b, uint64_t i0, uint64_t i1,
                                                uint64_t cap, uint64_t* sa, uint64_t* sba, bool* bad) {
  const uint32_t lane = threadIdx.x & 31;
  constexpr int U = 8;
  uint64_t s1 = 0, s2 = 0;
  for (uint64_t k = i0; k < i1; k += 32 * U) {
    uint64_t offa[U], offb[U], av[U], bv[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t j = min(k + u * 32 + lane, i1 - 1);
      offa[u] = j * aw;
      offb[u] = j * bw;
    }
    extract_bits_global_batch<U>(ap, offa, aw, av);
    if (with_b) extract_bits_global_batch<U>(bp, offb, bw, bv);
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (k + u * 32 + lane < i1) {
        uint64_t x = abase + av[u];
        if (x > cap) { *bad = true; x = 0; }
        s1 += x;
        if (with_b) s2 += (bbase + bv[u]) * x;
      }
    }
  }
  *sa = warp_sum(s1);
  *sba = warp_sum(s2);
}

// Cooperative copy of `nw` 32-bit words starting at word index w0 of `src` into shared memory (16-byte
// vector loads: w0 is a multiple of 4 and the stream base is 16-byte aligned).
__device__ __forceinline__ void stage_words(uint32_t* dst, const uint8_t* src, uint64_t w0, uint32_t nw) {
  const uint4* s4 = reinterpret_cast<const uint4*>(src) + (w0 >> 2);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (uint32_t k = threadIdx.x; k < (nw + 3) / 4; k += kThreads) d4[k] = __ldg(s4 + k);
}

constexpr uint32_t kSumsWarpRuns = 1024;                    // runs per rle_sums warp (half a tile)
constexpr uint32_t kSumsRuns = 8 * kSumsWarpRuns;           // runs per rle_sums CTA (4 tiles)
constexpr uint32_t kSumsTiles = kSumsRuns / K;
constexpr uint32_t kWarpsPerTile = K / kSumsWarpRuns;
constexpr uint32_t kSumsWords = kSumsRuns * 16 / 32 + 8;  // staged words per stream for w <= 16

__global__ void __launch_bounds__(kThreads, 3) rle_sums_kernel(const __grid_constant__ SumsBatch B) {
  __shared__ SumsChunk D;
  __shared__ __align__(16) uint32_t cw_s[kSumsWords];  // the CTA's packed counts (w <= 16)
  __shared__ __align__(16) uint32_t vw_s[kSumsWords];  // ... and packed slopes (root Delta|RLE, w <= 16)
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t unit = blockIdx.x;
  {
    int lo = 0, hi = int(B.n) - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (B.d[mid].unit0 <= unit) lo = mid; else hi = mid - 1;
    }
    stage_desc(&D, &B.d[lo]);
  }
  __syncthreads();
  trace_stamp(B.trace, unit, 0);
  trace_stamp(B.trace, unit, 7);
  grid_launch_dependents();  // rle_kernel may start staging now
  __shared__ uint64_t part_s[8][2];
  const uint32_t t0 = (unit - D.unit0) * kSumsTiles;
  const uint64_t r0 = uint64_t(t0) * K, r1 = min(r0 + kSumsRuns, uint64_t(D.nruns));
  const uint32_t t = t0 + warp / kWarpsPerTile;  // the warps of tile t0 + t' sum its 1024-run parts
  bool bad = false;
  uint64_t s1 = 0, s2 = 0;
  const bool staged = D.cnt_w <= 16 && (!D.linear || D.dv_w <= 16);
  if (staged) {
    // the CTA's 8 tiles are one contiguous bit range: stage it with coalesced 16-byte loads (one round trip)
    const uint32_t n = uint32_t(r1 - r0);
    if (D.cnt_w) stage_words(cw_s, D.cnt_packed, r0 * D.cnt_w / 32, (n * D.cnt_w + 31) / 32 + 2);
    else if (threadIdx.x < 2) cw_s[threadIdx.x] = 0;
    if (D.linear && D.dv_w) stage_words(vw_s, D.dv_packed, r0 * D.dv_w / 32, (n * D.dv_w + 31) / 32 + 2);
    else if (threadIdx.x < 2) vw_s[threadIdx.x] = 0;
    __syncthreads();
    if (t < D.tiles) {
      const uint32_t k0 = min(n, warp * kSumsWarpRuns), k1 = min(k0 + kSumsWarpRuns, n);
      const uint32_t cw = D.cnt_w, vw = D.dv_w, cap = D.rows;
      const uint32_t cm = (1u << cw) - 1u, vm = (1u << vw) - 1u;  // w <= 16
      const uint64_t cb = D.cnt_base, vb = D.dv_base;
      if (D.linear) {
#pragma unroll 4
        for (uint32_t k = k0 + lane; k < k1; k += 32) {
          const uint32_t bc = k * cw, bv = k * vw;
          uint64_t c = cb + (__funnelshift_r(cw_s[bc >> 5], cw_s[(bc >> 5) + 1], bc & 31) & cm);
          if (c > cap) { bad = true; c = 0; }
          s1 += c;
          s2 += (vb + (__funnelshift_r(vw_s[bv >> 5], vw_s[(bv >> 5) + 1], bv & 31) & vm)) * c;
        }
      } else {
#pragma unroll 4
        for (uint32_t k = k0 + lane; k < k1; k += 32) {
          const uint32_t bc = k * cw;
          uint64_t c = cb + (__funnelshift_r(cw_s[bc >> 5], cw_s[(bc >> 5) + 1], bc & 31) & cm);
          if (c > cap) { bad = true; c = 0; }
          s1 += c;
        }
      }
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
    }
  } else if (t < D.tiles) {
    const uint64_t i0 = min(r1, r0 + uint64_t(warp) * kSumsWarpRuns), i1 = min(i0 + kSumsWarpRuns, r1);
    warp_range_sums(reinterpret_cast<const uint32_t*>(D.cnt_packed), D.cnt_base, D.cnt_w,
                    reinterpret_cast<const uint32_t*>(D.dv_packed), D.dv_base, D.dv_w, D.linear, i0, i1, D.rows,
                    &s1, &s2, &bad);
  }
  if (lane == 0) { part_s[warp][0] = s1; part_s[warp][1] = s2; }
  __syncthreads();
  if (threadIdx.x < kSumsTiles && t0 + threadIdx.x < D.tiles) {
    uint64_t a = 0, b = 0;
#pragma unroll
    for (uint32_t h = 0; h < kWarpsPerTile; h++) {
      a += part_s[threadIdx.x * kWarpsPerTile + h][0];
      b += part_s[threadIdx.x * kWarpsPerTile + h][1];
    }
    D.tsum[2 * (t0 + threadIdx.x)] = a;
    D.tsum[2 * (t0 + threadIdx.x) + 1] = b;
  }
  if (threadIdx.x == 0) {  // the group's total (its kSumsTiles tiles), after the tile sums: tsum[2 (tiles + g)]
    uint64_t a = 0, b = 0;
#pragma unroll
    for (int w = 0; w < 8; w++) { a += part_s[w][0]; b += part_s[w][1]; }
    D.tsum[2 * (D.tiles + (unit - D.unit0))] = a;
    D.tsum[2 * (D.tiles + (unit - D.unit0)) + 1] = b;
  }
  if (bad) atomicOr(B.err + D.err_idx, 0x2u);
  trace_stamp(B.trace, unit, 4);
}

// ------------------------------------------------------------------------------------------ main
// One CTA per 1024-run tile; thread t owns runs 4t..4t+3.
//  1. stage the tile's packed counts/values (chunk data: overlaps rle_sums under PDL), then wait;
//  2. output offset O = sum of the tile sums before this tile; run values through the fused nested provider (V_RAW: the run values a
//     level-0 launch decoded from a Delta|RLE value lineage, read after the wait);
//  3. the tile's non-empty runs are compacted (first row, first value, slope) and a bitmap marks the row
//     where each one starts; row p of the tile belongs to compact run popc(bitmap[0..p]) - 1.  Each warp
//     owns a contiguous range of 64-row windows aligned to even global rows: a warp-wide popcount of the
//     words before its range gives the compact run it starts in, then per window lane l takes rows
//     2l, 2l+1 with two popcounts and one aligned vector store, so a warp stores 64 consecutive rows per
//     instruction (coalesced, no shared-memory output image).
// Descriptor fields are copied into registers once (the shared copy would otherwise be re-read inside
// every loop), and the compact tables are plain shared arrays (no generic-pointer address arithmetic).
constexpr int kRPer = K / kThreads;  // 4 runs per thread
constexpr uint32_t kBmWords = kRleSegRows / 64 + 2;  // 64-bit bitmap words of one segment (+ the shift bit)

__device__ __forceinline__ void stg_u64(void* p, uint64_t v) {
  asm volatile("st.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_v2_u32(void* p, uint32_t a, uint32_t b) {
  asm volatile("st.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void stg_u32(void* p, uint32_t v) {
  asm volatile("st.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// LIN: the batch has arithmetic-run (V_LINEAR or strided) descriptors; their slope table lives in dynamic shared memory.
// Occupancy OCC: 4 CTAs/SM (64 registers) for LIN (5 measured slower: config 2 level 0 13 -> 15 us) and for
// long runs; 5 (48 registers) for short-run batches (<= 16 rows per run: config 2 level 1 23.1 -> 21.8 us,
// 2700 -> 2820 GB/s; E3 even-1/even-4/random-1-8 +9-12 %; but even-32 / random-1-64 -6 %, hence the split;
// 6 / 40 registers measured slower)
template <bool TR, bool LIN, int OCC = 4>
__global__ void __launch_bounds__(kThreads, OCC) rle_kernel(const __grid_constant__ RleBatch B) {
  __shared__ RleDesc D;
  __shared__ uint32_t cnt_s[K / 2 + 8];             // staged packed counts when w <= 16 (else read via L1)
  __shared__ __align__(16) uint64_t aux_s[K + 8];   // staged packed values (V_BP/DICT/F2I); then compact values
  extern __shared__ __align__(16) uint64_t cslope_s[];  // [K] compact run slopes (V_LINEAR batches only)
  __shared__ uint32_t cstart_s[K];                  // compact run first rows (tile-relative)
  __shared__ __align__(16) uint64_t bm_s[kBmWords];  // run-start bitmap of one output segment
  __shared__ uint64_t warp_s[2 * kThreads / 32];
  uint64_t* const trace = TR ? B.trace : nullptr;

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t gt = blockIdx.x;
  trace_stamp(trace, gt, 0);
  trace_stamp(trace, gt, 7);
  stage_desc(&D, &B.d[find_desc(B, gt)]);
  for (uint32_t q = tid; q < kBmWords / 2; q += kThreads) reinterpret_cast<uint4*>(bm_s)[q] = make_uint4(0, 0, 0, 0);
  static_assert(kBmWords % 2 == 0, "bitmap cleared in 16-byte words");
  __syncthreads();
  const uint32_t lt = gt - D.tile0;
  const uint32_t g0 = lt * K;
  const uint32_t nr = min(uint32_t(K), D.nruns - g0);
  const uint32_t vmode = D.vmode;
  const bool linear = LIN && vmode == V_LINEAR;
  const bool strided = LIN && D.strided;  // DeltaStride: arithmetic runs with a per-node stride
  const bool arith = linear || strided;
  const uint64_t stride = D.stride;
  const uint32_t ob = D.out_bytes;
  const uint32_t n = D.n;
  const uint32_t cw = D.cnt_w, vw = D.val_w;
  const uint64_t cbase = D.cnt_base, vbase = D.val_base;
  const uint8_t* const cpk = D.cnt_packed;
  const uint8_t* const vpk = D.val_packed;
  uint32_t errbits = 0;
  const bool cnt_staged = cw <= 16;
  const bool val_staged = vmode == V_BP || vmode == V_DICT || vmode == V_F2I;
  if (cnt_staged) stage_bits<kThreads>(cnt_s, cpk, g0, nr, cw);
  if (val_staged) stage_bits<kThreads>(reinterpret_cast<uint32_t*>(aux_s), vpk, g0, nr, vw);
  grid_launch_dependents();  // a following level-1 launch may start its own staging
  grid_dependency_wait();    // rle_sums (and a level-0 launch) complete: tile sums / V are valid

  // ---- 2. output offset (and the wrapping dv*count prefix of a root Delta|RLE) of this tile: the sum of the
  // tile sums before it (L2-resident, written by rle_sums; loaded through L2 only)
  uint64_t O64, Pw;
  {
    // the group sums of the rle_sums groups before this tile's group, plus the tile sums of its group before it
    // (one round of independent L2 loads however deep the tile is in its chunk)
    uint64_t pc = 0, pw = 0;
    const ulonglong2* ts = reinterpret_cast<const ulonglong2*>(D.tsum);
    const uint32_t grp = lt / kSumsTiles, tg0 = grp * kSumsTiles;
    for (uint32_t i = tid; i < grp; i += kThreads) {
      const ulonglong2 v = __ldcg(ts + D.ntiles + i);
      pc += v.x;
      pw += v.y;
    }
    if (tid < lt - tg0) {
      const ulonglong2 v = __ldcg(ts + tg0 + tid);
      pc += v.x;
      pw += v.y;
    }
    pc = warp_sum(pc);
    if (linear) pw = warp_sum(pw);
    if (lane == 0) { warp_s[2 * warp] = pc; warp_s[2 * warp + 1] = pw; }
    __syncthreads();  // also: the staged counts / values are complete
    O64 = 0;
    Pw = 0;
#pragma unroll
    for (int k = 0; k < kThreads / 32; k++) { O64 += warp_s[2 * k]; Pw += warp_s[2 * k + 1]; }
    __syncthreads();  // warp_s is reused by the count scan
  }
  trace_stamp(trace, gt, 5);

  // phase A: this thread's 4 consecutive runs -- counts and values through the fused nested provider
  const uint32_t kb = tid * kRPer;
  uint32_t cnt[kRPer];
  uint64_t val[kRPer];
  uint64_t sc = 0, sw = 0;
  uint32_t ne = 0;
  const uint32_t cmask = cw >= 32 ? 0xFFFFFFFFu : (1u << cw) - 1u;
  uint64_t raw[kRPer];
  if (vmode == V_RAW) {  // level-0 output: 4 consecutive u64 (32-byte aligned)
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(vpk) + g0 + kb;
    if (kb + kRPer <= nr) {
      const ulonglong2 a = __ldcg(reinterpret_cast<const ulonglong2*>(src));
      const ulonglong2 b = __ldcg(reinterpret_cast<const ulonglong2*>(src) + 1);
      raw[0] = a.x; raw[1] = a.y; raw[2] = b.x; raw[3] = b.y;
    } else {
#pragma unroll
      for (int r = 0; r < kRPer; r++) raw[r] = kb + r < nr ? __ldcg(src + r) : 0ull;
    }
  }
#pragma unroll
  for (int r = 0; r < kRPer; r++) {
    const uint32_t k = kb + r;
    uint64_t c = 0, v = 0;
    if (k < nr) {
      const uint64_t g = g0 + k;
      if (cnt_staged) {
        const uint32_t bit = k * cw;
        c = cbase + (__funnelshift_r(cnt_s[bit >> 5], cnt_s[(bit >> 5) + 1], bit & 31) & cmask);
      } else {
        c = cbase + extract_bits_global(reinterpret_cast<const uint32_t*>(cpk), g * cw, cw);
      }
      if (c > n) { errbits |= 0x2u; c = 0; }
      if (linear) {
        v = vbase + extract_bits_global(reinterpret_cast<const uint32_t*>(vpk), g * vw, vw);
      } else if (vmode == V_RAW) {
        v = raw[r];
      } else {
        const uint64_t x = vbase + (vw ? extract_bits(reinterpret_cast<const uint32_t*>(aux_s), uint64_t(k) * vw, vw) : 0ull);
        if (vmode == V_BP) {
          v = x;
        } else if (vmode == V_DICT) {
          uint64_t idx = x;
          if (idx >= D.entries) { errbits |= 0x1u; idx = 0; }
          v = ob == 8 ? __ldg(reinterpret_cast<const unsigned long long*>(D.dict) + idx)
                      : uint64_t(__ldg(reinterpret_cast<const uint32_t*>(D.dict) + idx));
        } else {  // V_F2I
          v = uint64_t(__double_as_longlong(double(int64_t(x)) / kPow10r[D.d]));
        }
      }
    }
    cnt[r] = uint32_t(c);
    val[r] = v;
    sc += c;
    ne += c != 0;
    if (linear) sw += v * c;
  }
  trace_stamp(trace, gt, 1);
  // ---- 3. block scan of (non-empty runs << 44 | rows): this thread's first row and first compact index
  uint64_t T, W, ex, ew = 0;
  if (linear) block_excl_scan_pair<kThreads>((uint64_t(ne) << 44) | sc, sw, warp_s, &ex, &ew, &T, &W);
  else ex = block_excl_scan_u64<kThreads>((uint64_t(ne) << 44) | sc, warp_s, &T);
  const uint32_t ec = uint32_t(ex & ((1ull << 44) - 1)), ce = uint32_t(ex >> 44);
  const uint32_t nce = uint32_t(T >> 44);
  T &= (1ull << 44) - 1;
  trace_stamp(trace, gt, 2);
  const bool overflow = O64 + T > n;
  if (tid == 0 && (overflow || (lt + 1 == D.ntiles && O64 + T != n))) errbits |= 0x2u;
  if (errbits) atomicOr(B.err + D.err_idx, errbits);
  if (overflow) return;  // corrupt counts: never write outside [0, n) (uniform across the CTA)
  const uint32_t O = uint32_t(O64);
  const uint32_t Tt = uint32_t(T);

  if (Tt > kRleBigLimit && B.big_enabled) {  // giant runs: hand the tile's run table to rle_big
    __shared__ uint32_t slot_s;
    if (tid == 0) {
      const uint64_t pieces = (Tt + kRleBigPiece - 1) / kRleBigPiece;
      const unsigned long long old = atomicAdd(B.big.counter, (1ull << 44) | pieces);
      const uint32_t e = uint32_t(old >> 44);
      slot_s = e;
      if (e < B.big.max_slots) {
        RleBig::Entry& en = B.big.entries[e];
        en.out = D.out;
        en.O = O;
        en.T = Tt;
        en.nr = nr;
        en.slot = e;
        en.piece0 = old & ((1ull << 44) - 1);
        en.out_bytes = ob;
        en.linear = arith;
      } else {
        atomicOr(B.err + D.err_idx, 0x2u);
      }
    }
    __syncthreads();
    const uint32_t e = slot_s;
    if (e < B.big.max_slots) {
      uint32_t* so = B.big.soffs + uint64_t(e) * (K + 1);
      uint64_t* va = B.big.vals + uint64_t(e) * K;
      uint64_t* sl = B.big.slopes + uint64_t(e) * K;
      uint32_t row = ec;
      uint64_t wv = Pw + ew;
#pragma unroll
      for (int r = 0; r < kRPer; r++) {
        const uint32_t k = kb + r;
        if (k < nr) {
          so[k] = row;
          va[k] = linear ? D.delta_base + wv + val[r] : val[r];
          sl[k] = linear ? val[r] : stride;
        }
        if (linear) wv += val[r] * cnt[r];
        row += cnt[r];
      }
      if (tid == 0) so[nr] = Tt;
    }
    trace_stamp(trace, gt, 4);
    return;
  }

  // compact run table: first row, first value, slope of every non-empty run
  __syncthreads();  // the staged values are dead from here on
  {
    uint32_t row = ec, c = ce;
    uint64_t wv = Pw + ew;
    const uint64_t dbase = D.delta_base;
#pragma unroll
    for (int r = 0; r < kRPer; r++) {
      if (cnt[r]) {
        cstart_s[c] = row;
        aux_s[c] = linear ? dbase + wv + val[r] : val[r];
        if (arith) cslope_s[c] = linear ? val[r] : stride;
        c++;
      }
      if (linear) wv += val[r] * cnt[r];
      row += cnt[r];
    }
  }
  trace_stamp(trace, gt, 3);
  uint8_t* const gout = reinterpret_cast<uint8_t*>(D.out) + uint64_t(O) * ob;
  // 64-row windows aligned to EVEN global rows: bit b of a segment's bitmap is segment row b - a, a = parity
  // of the segment's first global row, so lane l's pair of rows (bits 2l, 2l+1) is one aligned 16-byte
  // (8-byte rows) or 8-byte (4-byte rows) store
  const uint32_t b0 = 2 * lane;
  const uint64_t lm0 = (2ull << b0) - 1ull;  // bits <= 2l
  for (uint32_t s0 = 0; s0 < Tt; s0 += kRleSegRows) {  // one segment unless the tile holds > 32 K rows
    const uint32_t rows = min(Tt - s0, kRleSegRows);
    const uint32_t a = (O + s0) & 1u;
    const uint32_t nw = (rows + a + 63) / 64;
    if (s0) {  // later segments: clear the previous segment's bits
      __syncthreads();
      for (uint32_t q = tid; q < kBmWords / 2; q += kThreads) reinterpret_cast<uint4*>(bm_s)[q] = make_uint4(0, 0, 0, 0);
      __syncthreads();
    }
    {
      uint32_t row = ec;
#pragma unroll
      for (int r = 0; r < kRPer; r++) {
        const uint32_t p = row - s0;
        if (cnt[r] && row >= s0 && p < rows) {
          const uint32_t bb = p + a;
          atomicOr(reinterpret_cast<uint32_t*>(bm_s) + (bb >> 5), 1u << (bb & 31));
        }
        row += cnt[r];
      }
    }
    __syncthreads();  // bitmap + compact run table complete
    // warp w: windows [k0, k1); cb = compact index of the row before its first window
    const uint32_t per = (nw + kThreads / 32 - 1) / (kThreads / 32);
    const uint32_t k0 = min(nw, warp * per), k1 = min(nw, k0 + per);
    uint32_t c_lt = 0;  // compact runs starting before s0 (later segments only)
    if (s0) {
      uint32_t lo = 0, hi = nce;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (cstart_s[mid] < s0) lo = mid + 1; else hi = mid;
      }
      c_lt = lo;
    }
    uint32_t pc = 0;
    for (uint32_t k = lane; k < k0; k += 32) pc += __popcll(bm_s[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pc += __shfl_xor_sync(FULL, pc, o);
    uint32_t cb = c_lt + pc - 1;
    uint8_t* const gseg = gout + uint64_t(s0) * ob;
    for (uint32_t k = k0; k < k1; k++) {
      const uint64_t wv = bm_s[k];
      const uint32_t c0 = cb + __popcll(wv & lm0);
      const uint32_t c1 = c0 + uint32_t((wv >> (b0 + 1)) & 1ull);
      cb += __popcll(wv);
      const int32_t p0 = int32_t(64 * k + b0) - int32_t(a);  // segment row of bit 2l
      uint64_t v0 = aux_s[c0 == 0xFFFFFFFFu ? 0u : c0], v1 = aux_s[c1];
      if (arith) {
        v0 += uint64_t(int64_t(s0) + p0 - cstart_s[c0 == 0xFFFFFFFFu ? 0u : c0]) * cslope_s[c0 == 0xFFFFFFFFu ? 0u : c0];
        v1 += uint64_t(int64_t(s0) + p0 + 1 - cstart_s[c1]) * cslope_s[c1];
      }
      const bool ok0 = p0 >= 0 && p0 < int32_t(rows), ok1 = p0 + 1 < int32_t(rows) && p0 + 1 >= 0;
      if (ob == 8) {
        uint64_t* const o = reinterpret_cast<uint64_t*>(gseg) + p0;
        if (ok0 && ok1) st_v2_u64(o, v0, v1);
        else {
          if (ok0) stg_u64(o, v0);
          if (ok1) stg_u64(o + 1, v1);
        }
      } else {
        uint32_t* const o = reinterpret_cast<uint32_t*>(gseg) + p0;
        if (ok0 && ok1) st_v2_u32(o, uint32_t(v0), uint32_t(v1));
        else {
          if (ok0) stg_u32(o, uint32_t(v0));
          if (ok1) stg_u32(o + 1, uint32_t(v1));
        }
      }
    }
  }
  trace_stamp(trace, gt, 4);
}

// ------------------------------------------------------------------------------------------ big tiles
__global__ void __launch_bounds__(kThreads) rle_big_kernel(const __grid_constant__ RleBatch B) {
  const RleBig& G = B.big;
  const unsigned long long c = *reinterpret_cast<volatile unsigned long long*>(G.counter);
  const uint32_t nent = min(uint32_t(c >> 44), G.max_slots);
  const uint64_t total = c & ((1ull << 44) - 1);
  const uint32_t warp = threadIdx.x >> 5;
  for (uint64_t piece = blockIdx.x; piece < total && nent; piece += gridDim.x) {
    uint32_t lo = 0, hi = nent - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (G.entries[mid].piece0 <= piece) lo = mid; else hi = mid - 1;
    }
    const RleBig::Entry en = G.entries[lo];
    const uint32_t k = uint32_t(piece - en.piece0);
    const uint32_t pb0 = k * kRleBigPiece;
    if (pb0 >= en.T) continue;
    const uint32_t pe0 = min(en.T, pb0 + kRleBigPiece);
    // 8192-row piece: warps take 1024-row spans (multiples of 128 keep windows aligned)
    const uint32_t pb = min(pe0, pb0 + warp * (kRleBigPiece / 8)), pe = min(pe0, pb + kRleBigPiece / 8);
    uint8_t* out = reinterpret_cast<uint8_t*>(en.out) + uint64_t(en.O) * en.out_bytes;
    expand_warp(G.soffs + uint64_t(en.slot) * (K + 1), en.nr, G.vals + uint64_t(en.slot) * K,
                en.linear ? G.slopes + uint64_t(en.slot) * K : nullptr, pb, pe, out, en.out_bytes, en.O);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(G.done, 1u) == gridDim.x - 1) {  // every CTA has read the queue: reset it
      atomicExch(G.counter, 0ull);
      atomicExch(G.done, 0u);
    }
  }
}

bool pdl_enabled() {
  static const bool pdl = !(std::getenv("CDM_PDL") && std::getenv("CDM_PDL")[0] == '0');
  return pdl;
}

}  // namespace

cudaError_t launch_rle_sums(const SumsBatch& b, cudaStream_t s) {
  if (!b.total_units) return cudaSuccess;
  rle_sums_kernel<<<b.total_units, kThreads, 0, s>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_rle(const RleBatch& b, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  // programmatic dependent launch: rle_kernel's prologue overlaps rle_sums (CDM_PDL=0 disables)
  const bool pdl = pdl_enabled();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(b.total_tiles);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = b.any_linear ? K * sizeof(uint64_t) : 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void (*kern)(RleBatch);
  if (b.any_linear) kern = b.trace ? rle_kernel<true, true> : rle_kernel<false, true>;
  else if (b.short_runs) kern = b.trace ? rle_kernel<true, false, 5> : rle_kernel<false, false, 5>;
  else kern = b.trace ? rle_kernel<true, false> : rle_kernel<false, false>;
  // NEXT-3 G.P. knob (Table 3's G.P. row): resident rle_kernel CTAs per SM, enforced by
  // padding the launch's dynamic shared memory (0 = the kernel's own occupancy)
  const int cap = tune_get(TUNE_GP_CTAS_PER_SM);
  const int dev = current_device();
  if (cap > 0) {
    static int smem_sm[kMaxDevices] = {};
    if (!smem_sm[dev]) cudaDeviceGetAttribute(&smem_sm[dev], cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    const long want = long(smem_sm[dev]) / cap - long(fa.sharedSizeBytes) - 1024;  // 1 KB reserved per CTA
    if (want > long(cfg.dynamicSmemBytes)) cfg.dynamicSmemBytes = size_t(want);
  }
  static size_t configured[kMaxDevices][6] = {};
  const int ki = kern == rle_kernel<true, true> ? 0 : kern == rle_kernel<false, true> ? 1
               : kern == rle_kernel<true, false, 5> ? 2 : kern == rle_kernel<false, false, 5> ? 3
               : kern == rle_kernel<true, false> ? 4 : 5;
  if (cfg.dynamicSmemBytes > 48 * 1024 && cfg.dynamicSmemBytes > configured[dev][ki]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(cfg.dynamicSmemBytes));
    configured[dev][ki] = cfg.dynamicSmemBytes;
  }
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, b);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_rle_big(const RleBatch& b, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  // every resident CTA slot: a piece's windows are latency-bound (dependent run-table loads), so occupancy
  // hides them (2 CTAs/SM measured 1.58 TB/s on E3 even-1024)
  static int occ[kMaxDevices] = {};
  int& o = occ[current_device()];
  if (!o) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, rle_big_kernel, kThreads, 0);
    if (o < 1) o = 1;
  }
  rle_big_kernel<<<device_sms() * o, kThreads, 0, s>>>(b);
  return cudaGetLastError();
}

}  // namespace cdm
