// kernels_rle.cu -- H7: scan-dependent ("Group-Parallel") RLE expansion.
//
//   out[offs_g .. offs_g + count_g) = V(g),   offs = exclusive_scan(count)
//
// The paper runs PyTorch cumsum on the counts, then a Group-Parallel kernel whose <L,S,C> geometry lets
// several blocks co-process one big group or one block walk several small groups.  The
// B200 design splits the family into:
//  * rle_prep_kernel: ALL look-backs of the family in one launch, over tiny aggregates only: per outer tile
//    of 2048 runs the sum of counts (plus sum dv*count for arithmetic runs), and for the Delta|RLE value
//    lineage of l_orderkey the inner run table S_j, Q_j = base + sum_{k<j} dv_k dc_k, dv_j.  Its tiles do no
//    expansion, so their look-back chains resolve in a few microseconds.
//  * rle_kernel: one CTA per outer tile, no inter-tile dependency: it stages the tile's packed counts and
//    values in shared memory, computes the run values through the fused nested provider (BitPack,
//    Dict|BitPack, Float2Int|BitPack, the Delta|RLE closed form value(g) = Q_j + (g - S_j + 1) dv_j, or
//    arithmetic runs for a root Delta|RLE), scans the counts in the CTA, reads its output offset from the
//    prep prefix and expands: each warp maps a 128-row window to runs with 4 ballots + 4 redux.or over the
//    next 128 run starts and every lane writes 4 consecutive rows with 16-byte stores.
//  * rle_big_kernel: tiles with more than kRleBigLimit output rows (giant runs: o_shippriority is one run
//    per chunk) are split into 8192-row pieces over every SM ("multiple GPU blocks
//    co-process a single group"); launched only when a chunk header's max run allows it.
// Invariant checked on the device: sum(count) == n (CDM_ERR_RUN_SUM); writes never leave [0, n).
#include "device_util.cuh"
#include "kernels.h"

namespace cdm {
namespace {

using namespace dev;

constexpr int K = kRleTile;
static_assert(kPrepOuterTile == 16 * kRleTile, "two rle tiles per prep warp");

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

// Cooperative, coalesced copy of the packed bits of items [i0, i0 + cnt) of a w-bit stream into shared
// words.  i0 is a multiple of 2048, so i0 * w is word aligned.  Copies two words past the last field
// (extraction reads up to word k+2); the stream's 16-byte slack keeps that in bounds.
__device__ __forceinline__ void stage_bits(uint32_t* dst, const uint8_t* packed, uint64_t i0, uint32_t cnt,
                                           uint32_t w) {
  if (w == 0) return;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(packed) + (i0 * w >> 5);
  const uint32_t nw = uint32_t((uint64_t(cnt) * w + 31) / 32) + 2;
  for (uint32_t k = threadIdx.x; k < nw; k += kThreads) dst[k] = __ldg(src + k);
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
                            uint32_t pb, uint32_t pe, uint8_t* out, uint32_t ob, uint32_t gO, bool nostore = false) {
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
    if (nostore) {
      if ((v[0] ^ v[1] ^ v[2] ^ v[3]) == 0x123456789ull) store_row(out, q0, 0, ob);
    } else if (q0 + 3 < pe) {
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

// ------------------------------------------------------------------------------------------ prep
// Warp-level sums over lane-strided items (coalesced extraction of consecutive fields).
__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ uint64_t warp_incl_scan(uint64_t v) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(FULL, v, o);
    if (lane >= uint32_t(o)) v += y;
  }
  return v;
}

__global__ void __launch_bounds__(kThreads) rle_prep_kernel(const __grid_constant__ PrepBatch B) {
  __shared__ PrepDesc D;
  __shared__ uint64_t wc_s[kThreads / 32], ww_s[kThreads / 32];
  __shared__ uint32_t tile_s, epoch_s;
  __shared__ uint64_t pc_s, pw_s;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    uint32_t t, e;
    take_ticket(B.ticket, B.total_tiles - 1, &t, &e);
    tile_s = t;
    epoch_s = e;
  }
  __syncthreads();
  const uint32_t gt = tile_s, epoch = epoch_s;
  if (gt >= B.total_tiles) return;
  trace_stamp(B.trace, gt, 0);
  trace_stamp(B.trace, gt, 7);
  stage_desc(&D, &B.d[find_desc(B, gt)]);
  __syncthreads();
  const uint32_t lt = gt - D.tile0;
  const bool inner = D.kind == PREP_INNER;
  const bool with_b = inner || D.linear;
  const uint32_t IW = inner ? kPrepInnerTile / 8 : kPrepOuterTile / 8;  // items per warp
  const uint64_t wbase = uint64_t(lt) * (8 * IW) + uint64_t(warp) * IW;
  const uint32_t* ap = reinterpret_cast<const uint32_t*>(D.a_packed);
  const uint32_t* bp = reinterpret_cast<const uint32_t*>(D.b_packed);

  // pass 1: per-warp sums (lane l takes items wbase + 32k + l: consecutive lanes read consecutive fields);
  // 8 items per lane per step with all their loads in flight
  uint64_t sc = 0, sw = 0, sc0 = 0, sw0 = 0;  // sc0/sw0: the warp's first rle tile (OUTER)
  bool bad = false;
  constexpr int U = 8;
  static_assert(kRleTile % (32 * U) == 0, "batches must not straddle rle tiles");
  for (uint32_t k = 0; k < IW; k += 32 * U) {
    if (k == uint32_t(K)) { sc0 = sc; sw0 = sw; }
    uint64_t offa[U], offb[U], av[U], bv[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t j = min(wbase + k + u * 32 + lane, uint64_t(D.n_items ? D.n_items - 1 : 0));
      offa[u] = j * D.a_w;
      offb[u] = j * D.b_w;
    }
    extract_bits_global_batch<U>(ap, offa, D.a_w, av);
    if (with_b) extract_bits_global_batch<U>(bp, offb, D.b_w, bv);
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t j = wbase + k + u * 32 + lane;
      if (j < D.n_items) {
        uint64_t a = D.a_base + av[u];
        const uint64_t b = with_b ? D.b_base + bv[u] : 0ull;
        if (a > D.total) { bad = true; a = 0; }
        sc += a;
        sw += b * a;
      }
    }
  }
  if (IW <= uint32_t(K)) { sc0 = sc; sw0 = sw; }
  sc = warp_sum(sc);
  sw = warp_sum(sw);
  sc0 = warp_sum(sc0);
  sw0 = warp_sum(sw0);
  if (lane == 0) { wc_s[warp] = sc; ww_s[warp] = sw; }
  __syncthreads();
  uint64_t ec = 0, ew = 0, tc = 0, tw = 0;
#pragma unroll
  for (int w2 = 0; w2 < kThreads / 32; w2++) {
    if (uint32_t(w2) < warp) { ec += wc_s[w2]; ew += ww_s[w2]; }
    tc += wc_s[w2];
    tw += ww_s[w2];
  }
  trace_stamp(B.trace, gt, 1);
  trace_stamp(B.trace, gt, 2);
  if (warp == 0) {
    uint64_t p0, p1;
    lb_tile(B.lb, gt, D.tile0, epoch, tc, tw, &p0, &p1);
    if (lane == 0) {
      pc_s = p0;
      pw_s = p1;
      if (lt + 1 == D.ntiles && p0 + tc != D.total) atomicOr(B.err + D.err_idx, 0x2u);
      if (inner && lt + 1 == D.ntiles) D.tstart[D.outer_tiles] = D.n_items - 1;  // closes the last window
    }
    trace_stamp(B.trace, gt, 3);
  }
  if (bad) atomicOr(B.err + D.err_idx, 0x2u);
  __syncthreads();
  uint64_t cc = pc_s + ec, cw = pw_s + ew;  // prefix at this warp's first item
  if (!inner) {  // the warp's rle tiles (IW / K of them): exclusive prefixes
    if (lane == 0) {
      for (uint32_t h = 0; h * K < IW; h++) {
        const uint64_t first = wbase + uint64_t(h) * K;
        if (first >= D.n_items) break;
        const uint64_t c = h ? cc + sc0 : cc, w = h ? cw + sw0 : cw;
        D.prefix[first / K] = make_uint4(0u, sat32(c), uint32_t(w), uint32_t(w >> 32));
      }
    }
  } else {  // pass 2: S_j, Q_j, DV_j per inner run (warp scans), tile starts
    constexpr int U2 = 4;
    for (uint32_t k = 0; k < IW; k += 32 * U2) {
      uint64_t offa[U2], offb[U2], avs[U2], bvs[U2];
#pragma unroll
      for (int u = 0; u < U2; u++) {
        const uint64_t j = min(wbase + k + u * 32 + lane, uint64_t(D.n_items ? D.n_items - 1 : 0));
        offa[u] = j * D.a_w;
        offb[u] = j * D.b_w;
      }
      extract_bits_global_batch<U2>(ap, offa, D.a_w, avs);
      extract_bits_global_batch<U2>(bp, offb, D.b_w, bvs);
#pragma unroll
      for (int u = 0; u < U2; u++) {
        const uint64_t j = wbase + k + u * 32 + lane;
        uint64_t av = 0, bv = 0;
        if (j < D.n_items) {
          av = D.a_base + avs[u];
          bv = D.b_base + bvs[u];
          if (av > D.total) av = 0;
        }
        const uint64_t ic = warp_incl_scan(av), iw = warp_incl_scan(bv * av);
        const uint64_t c = cc + ic - av, wv = cw + iw - bv * av;
        if (j < D.n_items) {
          D.S[j] = uint32_t(min(c, uint64_t(D.total)));
          D.Q[j] = D.base + wv;
          D.DV[j] = bv;
          if (av && c < D.total) {  // outer tiles whose first run lies in this inner run
            const uint64_t last = min(c + av, uint64_t(D.total)) - 1;
            for (uint64_t t = (c + K - 1) / K; t <= last / K && t < D.outer_tiles; t++) D.tstart[t] = uint32_t(j);
          }
        }
        cc += __shfl_sync(FULL, ic, 31);
        cw += __shfl_sync(FULL, iw, 31);
      }
    }
  }
  __syncthreads();
  trace_stamp(B.trace, gt, 4);
}

// ------------------------------------------------------------------------------------------ main
// One CTA per 1024-run tile; thread t owns runs 4t..4t+3.  The tile's output rows are written by each
// thread for its own runs (one shared-memory store per row, no searching) into a shared-memory image of
// the tile's output, which the CTA then copies out with aligned 16-byte stores.
constexpr int kRPer = K / kThreads;  // 4 runs per thread

__global__ void __launch_bounds__(kThreads, 3) rle_kernel(const __grid_constant__ RleBatch B) {
  extern __shared__ __align__(16) uint8_t outbuf[];  // kRleOutBytes + 16: the tile's output image
  __shared__ RleDesc D;
  __shared__ uint32_t cnt_s[K / 2 + 8];  // staged packed counts when w <= 16 (else read through L1)
  // aux: inner-run window (V_DRLE) | staged packed values (V_BP/V_DICT/V_F2I) | slopes (V_LINEAR)
  __shared__ __align__(16) uint8_t aux_s[K * 8 + 64];
  __shared__ uint32_t rc_s[K];  // run counts
  __shared__ uint64_t rv_s[K];  // run first values
  uint64_t* iQ_s = reinterpret_cast<uint64_t*>(aux_s);
  uint64_t* iDV_s = iQ_s + (kRleWindow + 1);
  uint32_t* iS_s = reinterpret_cast<uint32_t*>(iDV_s + (kRleWindow + 1));
  uint32_t* valbits_s = reinterpret_cast<uint32_t*>(aux_s);
  uint64_t* slope_s = reinterpret_cast<uint64_t*>(aux_s);
  static_assert((kRleWindow + 1) * 20 <= K * 8, "window must fit the aux buffer");
  __shared__ uint64_t warp_s[kThreads / 32];
  __shared__ uint32_t skip_s, win_s, j0i_s;
  const uint32_t tid = threadIdx.x;
  const uint32_t gt = blockIdx.x;
  trace_stamp(B.trace, gt, 0);
  trace_stamp(B.trace, gt, 7);
  stage_desc(&D, &B.d[find_desc(B, gt)]);
  __syncthreads();
  const uint32_t lt = gt - D.tile0;
  const uint32_t g0 = lt * K;
  const uint32_t nr = min(uint32_t(K), D.nruns - g0);
  const uint8_t vmode = D.vmode;
  const bool linear = vmode == V_LINEAR;
  const uint32_t ob = D.out_bytes;
  uint32_t errbits = 0;
  const uint4 pf = D.prefix[lt];  // tile output offset from rle_prep, issued early

  // stage packed counts (and values) of this tile; V_DRLE stages inner runs [tstart[lt], tstart[lt+1]]
  const bool cnt_staged = D.cnt_w <= 16;
  if (cnt_staged) stage_bits(cnt_s, D.cnt_packed, g0, nr, D.cnt_w);
  if (vmode == V_BP || vmode == V_DICT || vmode == V_F2I) stage_bits(valbits_s, D.val_packed, g0, nr, D.val_w);
  const uint32_t* wS = iS_s;
  const uint64_t* wQ = iQ_s;
  const uint64_t* wDV = iDV_s;
  if (vmode == V_DRLE) {
    if (tid == 0) {
      uint32_t j0i = D.tstart[lt], j1i = D.tstart[lt + 1];
      if (j0i >= D.n_inner) { j0i = 0; errbits |= 0x2u; }
      if (j1i >= D.n_inner || j1i < j0i) j1i = D.n_inner - 1;
      j0i_s = j0i;
      win_s = j1i - j0i + 1;
    }
    __syncthreads();
    const uint32_t j0i = j0i_s, win = win_s;
    if (win <= kRleWindow + 1) {
      for (uint32_t k = tid; k < win; k += kThreads) {
        iS_s[k] = D.S[j0i + k];
        iQ_s[k] = D.Q[j0i + k];
        iDV_s[k] = D.DV[j0i + k];
      }
    } else {  // unusual data (many tiny inner runs): search the prep arrays in global memory
      wS = D.S + j0i;
      wQ = D.Q + j0i;
      wDV = D.DV + j0i;
    }
  }
  __syncthreads();
  trace_stamp(B.trace, gt, 5);

  // phase A: this thread's 4 consecutive runs -- counts and values through the fused nested provider
  const uint32_t kb = tid * kRPer;
  uint32_t cnt[kRPer];
  uint64_t val[kRPer];
  uint64_t sc = 0, sw = 0;
  {
    uint32_t a = 0;
    if (vmode == V_DRLE && kb < nr) a = run_search(wS, 0, win_s - 1, g0 + kb);
#pragma unroll
    for (int r = 0; r < kRPer; r++) {
      const uint32_t k = kb + r;
      uint64_t c = 0, v = 0;
      if (k < nr) {
        const uint64_t g = g0 + k;
        c = D.cnt_base +
            (cnt_staged ? (D.cnt_w ? extract_bits(cnt_s, uint64_t(k) * D.cnt_w, D.cnt_w) : 0ull)
                        : extract_bits_global(reinterpret_cast<const uint32_t*>(D.cnt_packed), g * D.cnt_w, D.cnt_w));
        if (c > D.n) { errbits |= 0x2u; c = 0; }
        if (vmode == V_DRLE) {
          while (a + 1 < win_s && wS[a + 1] <= g) a++;
          v = wQ[a] + (g - wS[a] + 1) * wDV[a];
        } else if (linear) {
          v = D.val_base + extract_bits_global(reinterpret_cast<const uint32_t*>(D.val_packed), g * D.val_w, D.val_w);
        } else {
          const uint64_t x = D.val_base + (D.val_w ? extract_bits(valbits_s, uint64_t(k) * D.val_w, D.val_w) : 0ull);
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
      if (linear) sw += v * c;
    }
  }
  trace_stamp(B.trace, gt, 1);
  uint64_t T, W = 0;
  const uint64_t ec = block_excl_scan_u64<kThreads>(sc, warp_s, &T);  // this thread's first row
  uint64_t ew = 0;
  if (linear) ew = block_excl_scan_u64<kThreads>(sw, warp_s, &W);
  trace_stamp(B.trace, gt, 2);
  const uint64_t O64 = pf.y;
  const uint64_t Pw = (uint64_t(pf.w) << 32) | pf.z;
  if (tid == 0) {
    const bool overflow = O64 + T > D.n;
    skip_s = overflow;
    if (overflow || (lt + 1 == D.ntiles && O64 + T != D.n)) atomicOr(B.err + D.err_idx, 0x2u);
  }
  if (errbits) atomicOr(B.err + D.err_idx, errbits);
  // run table (the thread's own runs): first value and slope (arithmetic runs of a root Delta|RLE)
  {
    uint64_t wv = Pw + ew;
#pragma unroll
    for (int r = 0; r < kRPer; r++) {
      uint64_t first = val[r];
      if (linear) {
        slope_s[kb + r] = val[r];
        first = D.delta_base + wv + val[r];
        wv += val[r] * cnt[r];
      }
      rc_s[kb + r] = cnt[r];
      rv_s[kb + r] = first;
    }
  }
  __syncthreads();
  trace_stamp(B.trace, gt, 3);
  if (skip_s) return;  // corrupt counts: never write outside [0, n)

  const uint32_t O = uint32_t(O64);
  const uint32_t Tt = uint32_t(T);
  const uint32_t my = uint32_t(sc);
  if (Tt <= kRleBigLimit || !B.big_enabled) {
    const uint32_t cap_rows = (kRleOutBytes - 16) / ob;
    uint8_t* gout = reinterpret_cast<uint8_t*>(D.out);
    for (uint32_t s0 = 0; s0 < Tt; s0 += cap_rows) {  // one segment for all but unusually long tiles
      const uint32_t s1 = min(Tt, s0 + cap_rows);
      const uint64_t gbyte = uint64_t(O + s0) * ob;
      const uint32_t sh = uint32_t(gbyte & 15);
      uint8_t* buf = outbuf + sh;
      // rows of this thread's runs inside [s0, s1): a flat loop, one shared store per row
      const uint32_t q0 = max(uint32_t(ec), s0), q1 = min(uint32_t(ec) + my, s1);
      if (q0 < q1) {
        uint32_t r = 0, row = uint32_t(ec);
        while (row + rc_s[kb + r] <= q0) { row += rc_s[kb + r]; r++; }
        uint32_t rem = row + rc_s[kb + r] - q0;
        uint64_t v = rv_s[kb + r], sl = 0;
        if (linear) {
          sl = slope_s[kb + r];
          v += uint64_t(q0 - row) * sl;
        }
        uint8_t* p = buf + uint64_t(q0 - s0) * ob;
        uint8_t* const pe = buf + uint64_t(q1 - s0) * ob;
        if (ob == 8) {
          for (; p < pe; p += 8) {
            while (rem == 0) { r++; rem = rc_s[kb + r]; v = rv_s[kb + r]; if (linear) sl = slope_s[kb + r]; }
            *reinterpret_cast<uint64_t*>(p) = v;
            v += sl;
            rem--;
          }
        } else {
          for (; p < pe; p += 4) {
            while (rem == 0) { r++; rem = rc_s[kb + r]; v = rv_s[kb + r]; if (linear) sl = slope_s[kb + r]; }
            *reinterpret_cast<uint32_t*>(p) = uint32_t(v);
            v += sl;
            rem--;
          }
        }
      }
      __syncthreads();
      const uint32_t bytes = (s1 - s0) * ob;
      const uint32_t h = min(bytes, (16u - sh) & 15u);  // unaligned head (a multiple of ob)
      const uint32_t body = (bytes - h) & ~15u;
      uint8_t* dst = gout + gbyte;
      if (tid * ob < h) {
        if (ob == 8) *reinterpret_cast<uint64_t*>(dst + tid * 8) = *reinterpret_cast<const uint64_t*>(buf + tid * 8);
        else *reinterpret_cast<uint32_t*>(dst + tid * 4) = *reinterpret_cast<const uint32_t*>(buf + tid * 4);
      }
      for (uint32_t o = h + tid * 16; o < h + body; o += kThreads * 16) {
        const uint4 x = *reinterpret_cast<const uint4*>(buf + o);
        st_v4_u32(dst + o, x.x, x.y, x.z, x.w);
      }
      const uint32_t t0 = h + body + tid * ob;
      if (t0 < bytes) {
        if (ob == 8) *reinterpret_cast<uint64_t*>(dst + t0) = *reinterpret_cast<const uint64_t*>(buf + t0);
        else *reinterpret_cast<uint32_t*>(dst + t0) = *reinterpret_cast<const uint32_t*>(buf + t0);
      }
      if (s1 < Tt) __syncthreads();
    }
  } else {
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
        en.linear = linear;
      } else {
        atomicOr(B.err + D.err_idx, 0x2u);
      }
    }
    __syncthreads();
    const uint32_t e = slot_s;
    if (e < B.big.max_slots) {  // the tile's run table for rle_big, from this thread's runs
      uint32_t* so = B.big.soffs + uint64_t(e) * (K + 1);
      uint64_t* va = B.big.vals + uint64_t(e) * K;
      uint64_t* sl = B.big.slopes + uint64_t(e) * K;
      uint32_t row = uint32_t(ec);
#pragma unroll
      for (int r = 0; r < kRPer; r++) {
        const uint32_t k = kb + r;
        if (k < nr) {
          so[k] = row;
          va[k] = rv_s[k];
          sl[k] = linear ? slope_s[k] : 0ull;
        }
        row += cnt[r];
      }
      if (tid == 0) so[nr] = Tt;
    }
  }
  __syncthreads();
  trace_stamp(B.trace, gt, 4);
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

}  // namespace

cudaError_t launch_rle_prep(const PrepBatch& b, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  rle_prep_kernel<<<b.total_tiles, kThreads, 0, s>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_rle(const RleBatch& b, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(rle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kRleOutBytes + 16);
    configured = true;
  }
  rle_kernel<<<b.total_tiles, kThreads, kRleOutBytes + 16, s>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_rle_big(const RleBatch& b, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  rle_big_kernel<<<device_sms() * 2, kThreads, 0, s>>>(b);
  return cudaGetLastError();
}

}  // namespace cdm
