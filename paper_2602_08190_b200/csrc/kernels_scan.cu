// kernels_scan.cu -- H6: scan-dependent delta decode / VARCHAR offsets.
//
//   DELTA   out[i] = base + sum_{k<=i} (FOR + bits_k)            (mod 2^bits)
//   OFFSETS out[i] = sum_{k<i} (FOR + bits_k), out[n] = the total (lengths -> int32 offsets, reading R17)
//   DELTA over Dict|BitPack (Table 2 PS_SUPPKEY): the k-th delta is dict[FOR + bits_k]
//
// The paper decodes delta with PyTorch's cumsum as a separate pass.  Here the unpack is
// fused into the scan, in one of two schedules (NEXT-3 knob TUNE_SCAN_MODE):
//
//  * reduce-then-scan (default): scan_sums_kernel writes every 4096-element tile's sum (one warp per tile,
//    fully parallel: the packed stream is read once more, w/8 bytes per element); scan_kernel_rts is a
//    persistent, programmatically dependent launch whose CTAs each walk a contiguous range of tiles with the
//    next tile's packed bytes staged by the TMA engine (double buffer): the first tile's prefix is the sum of
//    the chunk's tile sums before it, later tiles carry the running prefix.  No inter-CTA waits.
//  * single-pass decoupled look-back: scan_kernel<true>, one tile per CTA in ticket order (epoch|ticket
//    counter: no memset, CUDA-graph safe), warp 0 publishes the tile aggregate and looks back over 32
//    predecessors at a time (device_util.cuh lb_tile).
//
// Both: a blocked thread-local scan of 16 values, a CTA scan of the thread totals, results transposed through
// shared memory so every warp store is a contiguous 16-byte-per-lane write; offsets are the EXCLUSIVE scan,
// aligned with the tile (16-byte stores), plus out[n] written by the chunk's last tile.
#include <cstdlib>

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

constexpr int kRtsThreads = 512;  // reduce-then-scan CTA: 8 values per thread (more warps in flight per SM)

__device__ __forceinline__ uint32_t scan_stage_bytes(const ScanDesc& D, uint64_t tile_start) {
  const uint64_t stream_bytes = ((uint64_t(D.n) * D.w + 7) / 8 + 15) & ~15ull;
  const uint64_t start = tile_start / 8 * D.w;
  const uint64_t want = uint64_t(kScanTile / 8) * D.w;
  const uint64_t have = stream_bytes > start ? stream_bytes - start : 0ull;
  return uint32_t(want < have ? want : have);
}

// Tile sums for reduce-then-scan: one 256-thread CTA per tile, thread t sums the 16 consecutive fields
// [16t, 16t + 16) through a two-word bit window that slides over the packed words (one load per 32 bits consumed,
// adjacent threads read adjacent words: coalesced), then a block reduction.  Exact in u64 (the offsets check
// compares the chunk's total).
__global__ void __launch_bounds__(kThreads) scan_sums_kernel(const __grid_constant__ ScanBatch B) {
  grid_launch_dependents();  // scan_kernel's CTAs may be scheduled (they stage their first tile, then wait)
  __shared__ uint64_t warp_s[kThreads / 32];
  const uint32_t gt = blockIdx.x, tid = threadIdx.x;
  const ScanDesc& D = B.d[find_desc_scan(B, gt)];
  const uint32_t lt = gt - D.tile0, w = D.w;
  const uint64_t tile_start = uint64_t(lt) * kScanTile;
  const uint32_t valid = uint32_t(min(uint64_t(kScanTile), uint64_t(D.n) - tile_start));
  const uint32_t* wd = reinterpret_cast<const uint32_t*>(D.packed + tile_start / 8 * w);
  constexpr uint32_t kPerS = kScanTile / kThreads;  // 16 fields per thread
  const uint32_t i0 = tid * kPerS, i1 = min(valid, i0 + kPerS);
  uint64_t acc = 0;
  if (D.dict) {  // Delta|Dict|BitPack: the deltas are dictionary entries (an index out of range adds 0)
    for (uint32_t i = i0; i < i1; i++) {
      const uint64_t ix = D.for_base + (w ? extract_bits_global(wd, uint64_t(i) * w, w) : 0ull);
      if (ix < D.entries) acc += __ldg(D.dict + ix);
    }  // scan_tile flags it (the look-back schedule has no sums pass)
  } else if (w && i0 < i1) {
    if (w <= 32) {
      const uint32_t m = w == 32 ? 0xFFFFFFFFu : (1u << w) - 1u;
      uint32_t q = (i0 * w) >> 5, sh = (i0 * w) & 31;
      uint32_t lo = __ldg(wd + q), hi = __ldg(wd + q + 1);
#pragma unroll
      for (uint32_t j = 0; j < kPerS; j++) {
        if (i0 + j >= i1) break;  // never read past the tile's last field (its word + 1 is in the stream padding)
        acc += __funnelshift_r(lo, hi, sh) & m;
        sh += w;
        if (sh >= 32 && i0 + j + 1 < i1) {
          sh -= 32;
          q++;
          lo = hi;
          hi = __ldg(wd + q + 1);
        }
      }
    } else {
      for (uint32_t i = i0; i < i1; i++) acc += extract_bits_global(wd, uint64_t(i) * w, w);
    }
  }
  if (!D.dict) acc += D.for_base * uint64_t(i1 > i0 ? i1 - i0 : 0u);
  uint64_t tot;
  block_excl_scan_u64<kThreads>(acc, warp_s, &tot);
  if (tid == 0) B.tsum[gt] = tot;
}

// One tile: unpack + scan + prefix + transposed 16-byte stores.  T = uint32_t when every output of the launch is
// 4 bytes (the values are needed mod 2^32 only: 32-bit arithmetic, the low 32 bits of each field), else
// uint64_t.  LB: the prefix comes from the decoupled look-back (warp 0) and the chunk's LENGTHS check uses the
// tile total; else `prefix` is the CTA's running prefix and `tsum_tile` this tile's exact sum (B.tsum).
constexpr uint32_t kResPad = kScanTile + kScanTile / 16;  // results in shared memory, one pad slot per 16
__device__ __forceinline__ uint32_t rpad(uint32_t i) { return i + (i >> 4); }

template <bool LB, typename T, int NT>
__device__ __forceinline__ void scan_tile(const ScanBatch& B, const ScanDesc& D, uint32_t gt, uint32_t epoch,
                                          const uint32_t* wd, T* res_s, uint64_t* warp_s, uint64_t* prefix_s,
                                          uint64_t prefix, uint64_t tsum_tile) {
  constexpr bool W64 = sizeof(T) == 8;
  constexpr int kPer = kScanTile / NT;  // values per thread
  const uint32_t tid = threadIdx.x;
  const uint32_t lt = gt - D.tile0, w = D.w;
  const uint64_t tile_start = uint64_t(lt) * kScanTile;
  const uint32_t valid = uint32_t(min(uint64_t(kScanTile), uint64_t(D.n) - tile_start));
  const T fb = T(D.for_base);
  const uint32_t m32 = w >= 32 ? 0xFFFFFFFFu : (1u << w) - 1u;

  // blocked: thread t owns values [kPer t, kPer (t+1)); v[j] = exclusive prefix within the thread
  T v[kPer + 1];
  T run = 0;
  const uint32_t i0 = tid * kPer;
  if (D.dict) {  // Delta|Dict|BitPack: an out-of-range index adds 0 and sets CDM_ERR_DICT_INDEX
    bool bad = false;
#pragma unroll
    for (int j = 0; j < kPer; j++) {
      T f = 0;
      if (i0 + j < valid) {
        const uint64_t ix = D.for_base + extract_bits(wd, uint64_t(i0 + j) * w, w);
        if (ix < D.entries) f = T(__ldg(D.dict + ix)); else bad = true;
      }
      v[j] = run;
      run += f;
    }
    if (bad) atomicOr(B.err + D.err_idx, 0x1u);
  } else if (!W64 || w <= 32) {
    // a two-word bit window slides over the thread's 16 fields (one shared load per 32 bits consumed)
    uint32_t q = (i0 * w) >> 5, sh = (i0 * w) & 31;
    uint32_t lo = wd[q], hi = wd[q + 1];
    const bool full = valid == kScanTile;
#pragma unroll
    for (int j = 0; j < kPer; j++) {
      const uint32_t f = __funnelshift_r(lo, hi, sh) & m32;
      v[j] = run;
      run += (full || i0 + j < valid) ? fb + T(f) : T(0);
      sh += w;
      if (sh >= 32) {
        sh -= 32;
        q++;
        lo = hi;
        hi = wd[q + 1];
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < kPer; j++) {
      const T f = (i0 + j < valid) ? fb + T(extract_bits(wd, uint64_t(i0 + j) * w, w)) : T(0);
      v[j] = run;
      run += f;
    }
  }
  v[kPer] = run;
  uint64_t tile_total;
  uint64_t texcl;
  if (LB) {
    texcl = block_excl_scan_u64<NT>(uint64_t(run), warp_s, &tile_total);
  } else {  // in T arithmetic (the LENGTHS check uses the exact tile sum from scan_sums_kernel)
    T tt;
    texcl = uint64_t(block_excl_scan_log<NT, T>(run, reinterpret_cast<T*>(warp_s), &tt));
    tile_total = uint64_t(tt);
  }
  if (LB) {
    if (tid < 32) {
      uint64_t pc, p0;
      lb_tile(B.lb, gt, D.tile0, epoch, 0, tile_total, &pc, &p0);
      if (tid == 0) *prefix_s = p0;
    }
    __syncthreads();
    prefix = *prefix_s;
    tsum_tile = tile_total;
  }
  if (tid == 0 && D.mode == SCAN_OFFSETS && lt + 1 == D.ntiles) {
    if (prefix + tsum_tile != D.base) atomicOr(B.err + D.err_idx, 0x8u);  // CDM_ERR_LENGTHS
    reinterpret_cast<int32_t*>(D.out)[D.n] = int32_t(uint32_t(prefix + tsum_tile));  // offsets[n]
  }
  // DELTA: out[i] = base + inclusive sum; OFFSETS: out[i] = exclusive sum
  const bool delta = D.mode == SCAN_DELTA;
  const T add = T((delta ? D.base : 0ull) + prefix + texcl);
#pragma unroll
  for (int j = 0; j < kPer; j++) res_s[rpad(i0 + j)] = add + (delta ? v[j + 1] : v[j]);
  __syncthreads();
  // striped: thread t stores values k*4NT + 4t .. +3 (16 or 32 contiguous bytes per lane, whole lines per warp)
#pragma unroll
  for (uint32_t k = 0; k < kScanTile / (4 * NT); k++) {
    const uint32_t e0 = k * 4 * NT + tid * 4;
    if (e0 >= valid) break;
    const uint64_t gi = tile_start + e0;
    const T r0 = res_s[rpad(e0)], r1 = res_s[rpad(e0 + 1)], r2 = res_s[rpad(e0 + 2)], r3 = res_s[rpad(e0 + 3)];
    if (D.out_bytes == 8) {
      uint64_t* o = reinterpret_cast<uint64_t*>(D.out) + gi;
      if (e0 + 4 <= valid) {
        st_v2_u64(o, uint64_t(r0), uint64_t(r1));
        st_v2_u64(o + 2, uint64_t(r2), uint64_t(r3));
      } else {
        const T r[4] = {r0, r1, r2, r3};
#pragma unroll
        for (uint32_t j = 0; j < 4; j++) if (e0 + j < valid) o[j] = uint64_t(r[j]);
      }
    } else {
      uint32_t* o = reinterpret_cast<uint32_t*>(D.out) + gi;
      if (e0 + 4 <= valid) {
        st_v4_u32(o, uint32_t(r0), uint32_t(r1), uint32_t(r2), uint32_t(r3));
      } else {
        const T r[4] = {r0, r1, r2, r3};
#pragma unroll
        for (uint32_t j = 0; j < 4; j++) if (e0 + j < valid) o[j] = uint32_t(r[j]);
      }
    }
  }
  __syncthreads();  // res_s and the staged tile are free
}

// reduce-then-scan: persistent CTAs, each over a CONTIGUOUS range of tiles, the next tile's packed bytes staged by
// the TMA engine while the current one is scanned.  A CTA needs the tile sums once for its first tile (the sum of
// the chunk's tiles before it, block-reduced); after that the running prefix grows by each tile's sum (and
// restarts at 0 at a chunk's first tile).
constexpr uint32_t kRtsStages = 4;  // packed-tile stages: the TMA engine runs up to 3 tiles ahead

template <typename T>
__global__ void __launch_bounds__(kRtsThreads, sizeof(T) == 4 ? 3 : 2) scan_kernel_rts(const __grid_constant__ ScanBatch B, uint32_t stage_alloc) {
  extern __shared__ __align__(128) uint8_t smem[];  // [kRtsStages x stage_alloc packed][kResPad x T results]
  T* res_s = reinterpret_cast<T*>(smem + kRtsStages * stage_alloc);
  __shared__ uint64_t warp_s[kRtsThreads / 32];
  __shared__ __align__(8) uint64_t bar[kRtsStages];
  const uint32_t tid = threadIdx.x;
  const uint32_t per = (B.total_tiles + gridDim.x - 1) / gridDim.x;
  const uint32_t t0 = blockIdx.x * per, t1 = min(B.total_tiles, t0 + per);
  if (t0 >= t1) return;
  // the descriptor of a tile: the CTA's tiles are contiguous, so the index only moves forward
  int di = find_desc_scan(B, t0);
  int sdi = di;  // the staging cursor (kRtsStages - 1 tiles ahead)
  auto stage = [&](uint32_t t, uint32_t s) {  // tid 0: TMA the packed bytes of tile t into stage s
    while (sdi + 1 < int(B.n) && B.d[sdi + 1].tile0 <= t) sdi++;
    const ScanDesc& D = B.d[sdi];
    const uint64_t tile_start = uint64_t(t - D.tile0) * kScanTile;
    const uint32_t nb = scan_stage_bytes(D, tile_start);
    fence_proxy_async();  // generic reads of this stage (kRtsStages tiles ago) precede the TMA refill
    mbar_arrive_expect_tx(&bar[s], nb);
    if (nb) tma_load_1d(smem + s * stage_alloc, D.packed + tile_start / 8 * D.w, nb, &bar[s]);
  };
  if (tid == 0) {
    for (uint32_t k = 0; k < kRtsStages; k++) mbar_init(&bar[k], 1);
    fence_mbar_init();
    for (uint32_t k = 0; k + 1 < kRtsStages && t0 + k < t1; k++) stage(t0 + k, k);
  }
  __syncthreads();
  grid_dependency_wait();  // scan_sums_kernel complete: the tile sums are valid
  uint64_t prefix;
  {
    uint64_t part = 0;
    for (uint32_t k = B.d[di].tile0 + tid; k < t0; k += kRtsThreads) part += B.tsum[k];
    uint64_t tot;
    block_excl_scan_u64<kRtsThreads>(part, warp_s, &tot);
    prefix = tot;
  }
  uint32_t it = 0;
  uint64_t ts = B.tsum[t0];
  for (uint32_t gt = t0; gt < t1; gt++, it++) {
    const uint32_t s = it % kRtsStages;
    // the stage of tile gt - 1 was freed by its barriers: refill it with tile gt + kRtsStages - 1
    if (tid == 0 && gt + kRtsStages - 1 < t1) stage(gt + kRtsStages - 1, (it + kRtsStages - 1) % kRtsStages);
    const uint64_t ts_next = gt + 1 < t1 ? B.tsum[gt + 1] : 0ull;  // in flight during this tile
    while (di + 1 < int(B.n) && B.d[di + 1].tile0 <= gt) di++;
    const ScanDesc& D = B.d[di];
    if (gt == D.tile0) prefix = 0;  // a chunk's first tile
    mbar_wait(&bar[s], (it / kRtsStages) & 1);
    scan_tile<false, T, kRtsThreads>(B, D, gt, 0, reinterpret_cast<const uint32_t*>(smem + s * stage_alloc), res_s,
                                     warp_s, nullptr, prefix, ts);
    prefix += ts;
    ts = ts_next;
  }
}

// single-pass decoupled look-back: one tile per CTA, tiles in ticket order
__global__ void __launch_bounds__(kThreads) scan_kernel_lb(const __grid_constant__ ScanBatch B) {
  __shared__ __align__(128) uint64_t buf_s[kResPad + 4];  // the staged tile, then the results
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
  const ScanDesc& D = B.d[find_desc_scan(B, gt)];
  if (tid == 0) {
    const uint64_t tile_start = uint64_t(gt - D.tile0) * kScanTile;
    const uint32_t nb = scan_stage_bytes(D, tile_start);
    mbar_arrive_expect_tx(&bar, nb);
    if (nb) tma_load_1d(buf_s, D.packed + tile_start / 8 * D.w, nb, &bar);
  }
  mbar_wait(&bar, 0);
  // the unpack reads the staged bytes into registers before the results overwrite the buffer (scan_tile's
  // first barrier sits between the two)
  scan_tile<true, uint64_t, kThreads>(B, D, gt, epoch, reinterpret_cast<const uint32_t*>(buf_s), buf_s, warp_s, &prefix_s, 0,
                                   0);
}

// ------------------------------------------------------------------------------------------ warp tiles (3 passes)
// scan_mode 2: the scan without any CTA-wide barrier.  Warp tiles of kSub = 512 values (16 per
// lane): pass 1 (scan_wsums_kernel) writes every warp tile's exact sum, pass 2 (scan_wprefix_kernel, one CTA per
// chunk) scans a chunk's warp-tile sums in place (and checks / writes the offsets' total), pass 3
// (scan_warp_kernel) gives every warp tile to one warp: its 16 fields per lane are unpacked from global memory
// through a sliding two-word window, scanned in registers and across the warp with shuffles, offset by the tile's
// prefix, and leave through a per-warp shared stage as 16-byte stores (__syncwarp only).
constexpr uint32_t kSub = 512;
constexpr uint32_t kSubPer = kSub / 32;  // 16 values per lane
constexpr uint32_t kSubPerTile = kScanTile / kSub;

// the lane's kSubPer fields (FOR added; dictionary entries for Delta|Dict|BitPack) of elements [e0, e0 + nv),
// unpacked from global memory through a sliding two-word window
template <typename T>
__device__ __forceinline__ void lane_fields(const ScanDesc& D, uint64_t e0, uint32_t nv, T (&f)[kSubPer], bool& bad) {
  const uint32_t w = D.w;
  const uint32_t* wd = reinterpret_cast<const uint32_t*>(D.packed);
  if (D.dict) {
#pragma unroll
    for (uint32_t j = 0; j < kSubPer; j++) {
      f[j] = 0;
      if (j < nv) {
        const uint64_t ix = D.for_base + (w ? extract_bits_global(wd, (e0 + j) * w, w) : 0ull);
        if (ix < D.entries) f[j] = T(__ldg(D.dict + ix)); else bad = true;
      }
    }
    return;
  }
  const T fb = T(D.for_base);
  if (w == 0) {
#pragma unroll
    for (uint32_t j = 0; j < kSubPer; j++) f[j] = j < nv ? fb : T(0);
  } else if (w <= 32) {
    const uint32_t m = w == 32 ? 0xFFFFFFFFu : (1u << w) - 1u;
    const uint64_t b0 = e0 * w;
    uint64_t q = b0 >> 5;
    uint32_t sh = uint32_t(b0 & 31);
    uint32_t lo = nv ? __ldg(wd + q) : 0u, hi = nv ? __ldg(wd + q + 1) : 0u;
#pragma unroll
    for (uint32_t j = 0; j < kSubPer; j++) {
      f[j] = j < nv ? fb + T(__funnelshift_r(lo, hi, sh) & m) : T(0);
      sh += w;
      if (sh >= 32) {
        sh -= 32;
        q++;
        lo = hi;
        hi = j + 1 < nv ? __ldg(wd + q + 1) : 0u;  // never past the last field's word + 1 (stream padding)
      }
    }
  } else {
#pragma unroll
    for (uint32_t j = 0; j < kSubPer; j++) f[j] = j < nv ? fb + T(extract_bits_global(wd, (e0 + j) * w, w)) : T(0);
  }
}

__device__ __forceinline__ uint32_t chunk_subs(const ScanDesc& D) { return (D.n + kSub - 1) / kSub; }

// pass 1: one warp per warp tile (sub-tiles of a chunk are numbered from kSubPerTile * tile0)
__global__ void __launch_bounds__(kThreads) scan_wsums_kernel(const __grid_constant__ ScanBatch B) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gs = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (gs >= B.total_tiles * kSubPerTile) return;
  const ScanDesc& D = B.d[find_desc_scan(B, gs / kSubPerTile)];
  const uint32_t ls = gs - D.tile0 * kSubPerTile;
  if (ls >= chunk_subs(D)) return;
  const uint64_t e0 = uint64_t(ls) * kSub + lane * kSubPer;
  const uint32_t nv = e0 < D.n ? uint32_t(min(uint64_t(kSubPer), uint64_t(D.n) - e0)) : 0u;
  bool bad = false;
  uint64_t acc = 0;
  if (!D.dict && D.w <= 27) {  // 16 fields < 2^27 sum in 32 bits; the FOR base is added once per field after
    ScanDesc Dz = D;
    Dz.for_base = 0;
    uint32_t f[kSubPer];
    lane_fields<uint32_t>(Dz, e0, nv, f, bad);
    uint32_t a32 = 0;
#pragma unroll
    for (uint32_t j = 0; j < kSubPer; j++) a32 += f[j];
    acc = uint64_t(a32) + D.for_base * uint64_t(nv);
  } else {
    uint64_t f[kSubPer];
    lane_fields<uint64_t>(D, e0, nv, f, bad);
#pragma unroll
    for (uint32_t j = 0; j < kSubPer; j++) acc += f[j];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
  if (lane == 0) B.tsum[gs] = acc;
  if (bad) atomicOr(B.err + D.err_idx, 0x1u);
}

// pass 2: one CTA per chunk: exclusive scan of its warp-tile sums in place; the offsets' total is checked against
// the node's byte count (CDM_ERR_LENGTHS) and written as out[n]
constexpr int kPfxThreads = 1024;
__global__ void __launch_bounds__(kPfxThreads) scan_wprefix_kernel(const __grid_constant__ ScanBatch B) {
  __shared__ uint64_t warp_s[kPfxThreads / 32];
  const ScanDesc& D = B.d[blockIdx.x];
  uint64_t* ts = B.tsum + uint64_t(D.tile0) * kSubPerTile;
  const uint32_t ns = chunk_subs(D), per = (ns + kPfxThreads - 1) / kPfxThreads;
  const uint32_t i0 = min(ns, threadIdx.x * per), i1 = min(ns, i0 + per);
  // up to 8 sums per thread (chunks of <= 4 M values) are read once, all loads in flight together
  constexpr uint32_t R = 8;
  uint64_t v[R];
  uint64_t sum = 0;
  if (per <= R) {
#pragma unroll
    for (uint32_t r = 0; r < R; r++) {
      v[r] = i0 + r < i1 ? __ldcg(ts + i0 + r) : 0ull;
      sum += v[r];
    }
  } else {
    for (uint32_t i = i0; i < i1; i++) sum += __ldcg(ts + i);
  }
  uint64_t tot;
  uint64_t run = block_excl_scan_u64<kPfxThreads>(sum, warp_s, &tot);
  if (per <= R) {
#pragma unroll
    for (uint32_t r = 0; r < R; r++) {
      if (i0 + r < i1) ts[i0 + r] = run;
      run += v[r];
    }
  } else {
    for (uint32_t i = i0; i < i1; i++) {
      const uint64_t x = __ldcg(ts + i);
      ts[i] = run;
      run += x;
    }
  }
  if (threadIdx.x == 0 && D.mode == SCAN_OFFSETS) {
    if (tot != D.base) atomicOr(B.err + D.err_idx, 0x8u);  // CDM_ERR_LENGTHS
    reinterpret_cast<int32_t*>(D.out)[D.n] = int32_t(uint32_t(tot));
  }
}

// pass 3: one warp per warp tile
template <typename T>
__global__ void __launch_bounds__(kThreads, 4) scan_warp_kernel(const __grid_constant__ ScanBatch B) {
  __shared__ __align__(16) T stage_s[kThreads / 32][kSub];  // a warp tile's results as 16-byte chunks
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t gs = blockIdx.x * (kThreads / 32) + wib;
  if (gs >= B.total_tiles * kSubPerTile) return;
  const ScanDesc& D = B.d[find_desc_scan(B, gs / kSubPerTile)];
  const uint32_t ls = gs - D.tile0 * kSubPerTile;
  if (ls >= chunk_subs(D)) return;
  const uint64_t s0 = uint64_t(ls) * kSub, e0 = s0 + lane * kSubPer;
  const uint32_t valid = uint32_t(min(uint64_t(kSub), uint64_t(D.n) - s0));
  const uint32_t nv = e0 < D.n ? uint32_t(min(uint64_t(kSubPer), uint64_t(D.n) - e0)) : 0u;
  T f[kSubPer];
  bool bad = false;  // (reported by pass 1)
  lane_fields<T>(D, e0, nv, f, bad);
  T run = 0;
#pragma unroll
  for (uint32_t j = 0; j < kSubPer; j++) {
    const T x = f[j];
    f[j] = run;  // exclusive within the lane
    run += x;
  }
  T incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T v = __shfl_up_sync(FULL, incl, o);
    if (lane >= uint32_t(o)) incl += v;
  }
  const bool delta = D.mode == SCAN_DELTA;
  const T add = T((delta ? D.base : 0ull) + B.tsum[gs]) + (incl - run);
  // DELTA: base + inclusive sum (exclusive + own field); OFFSETS: the exclusive sum
#pragma unroll
  for (uint32_t j = 0; j < kSubPer; j++) {
    const T nxt = j + 1 < kSubPer ? f[j + 1] : run;
    f[j] = add + (delta ? nxt : f[j]);
  }
  // the lane's 16 results leave through the warp's stage as 16-byte chunks: lane L writes its chunks c at slot
  // L * CPL + (c ^ swizzle(L)) (conflict-free), then every lane stores the warp tile's chunks 32 apart (coalesced)
  uint4* const stq = reinterpret_cast<uint4*>(stage_s[wib]);
  if (sizeof(T) == 8 && D.out_bytes == 8) {
#pragma unroll
    for (uint32_t c = 0; c < 8; c++) {
      const uint64_t a = uint64_t(f[2 * c]), b = uint64_t(f[2 * c + 1]);
      stq[lane * 8 + (c ^ (lane & 7))] = make_uint4(uint32_t(a), uint32_t(a >> 32), uint32_t(b), uint32_t(b >> 32));
    }
    __syncwarp();
    uint64_t* o = reinterpret_cast<uint64_t*>(D.out) + s0;
#pragma unroll
    for (uint32_t k = 0; k < 8; k++) {
      const uint32_t q = k * 32 + lane, L = q >> 3, c = q & 7;
      if (2 * q >= valid) break;
      const uint4 x = stq[L * 8 + (c ^ (L & 7))];
      const uint64_t a = uint64_t(x.x) | (uint64_t(x.y) << 32), b = uint64_t(x.z) | (uint64_t(x.w) << 32);
      if (2 * q + 2 <= valid) st_v2_u64(o + 2 * q, a, b);
      else o[2 * q] = a;
    }
  } else {  // 4-byte outputs (values mod 2^32)
#pragma unroll
    for (uint32_t c = 0; c < 4; c++)
      stq[lane * 4 + (c ^ ((lane >> 1) & 3))] =
          make_uint4(uint32_t(f[4 * c]), uint32_t(f[4 * c + 1]), uint32_t(f[4 * c + 2]), uint32_t(f[4 * c + 3]));
    __syncwarp();
    uint32_t* o = reinterpret_cast<uint32_t*>(D.out) + s0;
#pragma unroll
    for (uint32_t k = 0; k < 4; k++) {
      const uint32_t q = k * 32 + lane, L = q >> 2, c = q & 3;
      if (4 * q >= valid) break;
      const uint4 x = stq[L * 4 + (c ^ ((L >> 1) & 3))];
      if (4 * q + 4 <= valid) {
        st_v4_u32(o + 4 * q, x.x, x.y, x.z, x.w);
      } else {
        const uint32_t r[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (uint32_t j = 0; j < 4; j++) if (4 * q + j < valid) o[4 * q + j] = r[j];
      }
    }
  }
}

bool pdl_on() {
  static const bool pdl = !(std::getenv("CDM_PDL") && std::getenv("CDM_PDL")[0] == '0');
  return pdl;
}

}  // namespace

cudaError_t launch_scan(const ScanBatch& b, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  if (tune_get(TUNE_SCAN_MODE) == 1) {
    scan_kernel_lb<<<b.total_tiles, kThreads, 0, s>>>(b);
    return cudaGetLastError();
  }
  if (tune_get(TUNE_SCAN_MODE) == 2) {
    bool w64 = false;
    for (uint32_t i = 0; i < b.n; i++) w64 = w64 || b.d[i].out_bytes == 8;
    const uint32_t grid = (b.total_tiles * kSubPerTile + kThreads / 32 - 1) / (kThreads / 32);
    scan_wsums_kernel<<<grid, kThreads, 0, s>>>(b);
    scan_wprefix_kernel<<<b.n, kPfxThreads, 0, s>>>(b);
    if (w64) scan_warp_kernel<uint64_t><<<grid, kThreads, 0, s>>>(b);
    else scan_warp_kernel<uint32_t><<<grid, kThreads, 0, s>>>(b);
    return cudaGetLastError();
  }
  scan_sums_kernel<<<b.total_tiles, kThreads, 0, s>>>(b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  uint32_t max_w = 0;
  bool w64 = false;  // some output of the launch is 8 bytes: 64-bit arithmetic
  for (uint32_t i = 0; i < b.n; i++) {
    max_w = std::max<uint32_t>(max_w, b.d[i].w);
    w64 = w64 || b.d[i].out_bytes == 8;
  }
  const uint32_t stage = ((kScanTile / 8) * (max_w ? max_w : 1) + 16 + 127) & ~127u;  // + slack words
  const uint32_t smem = kRtsStages * stage + kResPad * (w64 ? 8 : 4);
  auto kern = w64 ? scan_kernel_rts<uint64_t> : scan_kernel_rts<uint32_t>;
  static uint32_t configured[kMaxDevices][2] = {};
  uint32_t& conf = configured[current_device()][w64];
  if (smem > conf) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    conf = smem;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRtsThreads, smem);
  if (per_sm < 1) per_sm = 1;
  uint32_t grid = uint32_t(device_sms() * per_sm);
  if (grid > b.total_tiles) grid = b.total_tiles;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kRtsThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, b, stage);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace cdm
