// kernels_rle.cu -- H7: scan-dependent ("Group-Parallel") RLE expansion.
//
//   out[offs_g .. offs_g + count_g) = V(g),   offs = exclusive_scan(count)
//
// The paper runs PyTorch cumsum on the counts, then a Group-Parallel kernel whose <L,S,C> geometry makes
// several blocks co-process one big group or one block walk several small groups.
// B200 design, one pass over the runs:
//  * rle_kernel: a CTA owns 2048 consecutive runs (ticketed).  It unpacks the counts (FOR + bits), the
//    run values through the fused nested provider (BitPack, Dict|BitPack, Float2Int|BitPack, the
//    closed form of Delta|RLE, or arithmetic runs for a root Delta|RLE), scans the counts in the CTA
//    and obtains the tile's output offset by decoupled look-back -- the cumsum never touches HBM.
//    Small tiles are expanded in place: each warp takes a contiguous output span and maps 32 output
//    rows at a time to runs with one ballot + one redux.or over the next 32 run starts.
//  * tiles whose output exceeds kRleBigLimit rows (giant runs: o_shippriority is one run per chunk,
//    SPEC.md:167) are queued with their run table; rle_big_kernel splits them into 8192-row pieces
//    spread over every SM ("multiple GPU blocks co-process a single group").
//  * inner_kernel: for RLE|[Delta|RLE|[BitPack,BitPack], BitPack] (l_orderkey) the outer run values
//    are value(g) = base + Q_j + (g - S_j + 1) * dv_j with j the inner run holding g, so only the inner
//    run table (S, Q, dv; ~n/16 entries, L2-resident) is materialised -- never the n/4 outer values.
// Invariant checked on the device: sum(count) == n (CDM_ERR_RUN_SUM); writes never leave [0, n).
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

// Expand output rows [pb, pe) of a tile whose runs start at soffs[0..nr] (soffs[0] = 0, soffs[nr] = T).
// Element p of run r is vals[r] + (p - soffs[r]) * slopes[r] (slopes == nullptr: plain RLE).
// Called by a full warp; rows are written by consecutive lanes (coalesced 4/8-byte stores).
__device__ __forceinline__ void expand_warp(const uint32_t* soffs, uint32_t nr, const uint64_t* vals,
                                            const uint64_t* slopes, uint32_t pb, uint32_t pe, uint8_t* out,
                                            uint32_t ob) {
  const uint32_t lane = threadIdx.x & 31;
  if (pb >= pe || nr == 0) return;
  uint32_t lo = 0, hi = nr - 1;  // last run with soffs[r] <= pb
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (soffs[mid] <= pb) lo = mid; else hi = mid - 1;
  }
  uint32_t r = lo;
  for (uint32_t p0 = pb; p0 < pe; p0 += 32) {
    const uint32_t j = r + 1 + lane;
    const uint32_t s = (j <= nr) ? soffs[j] : 0xFFFFFFFFu;  // s > p0 for every candidate
    const bool in31 = s <= p0 + 31;
    const uint32_t m31 = __ballot_sync(FULL, in31);
    const uint32_t M = __reduce_or_sync(FULL, in31 ? (1u << (s - p0)) : 0u);
    const uint32_t p = p0 + lane;
    uint32_t rr;
    if (m31 != FULL && __popc(M) == __popc(m31)) {
      rr = r + __popc(M & (FULL >> (31 - lane)));  // run starts at or before p0 + lane
    } else {  // zero-length runs or >= 32 starts in the window: per-lane search
      uint32_t a = r, b = nr - 1;
      while (a < b) {
        const uint32_t mid = (a + b + 1) >> 1;
        if (soffs[mid] <= p) a = mid; else b = mid - 1;
      }
      rr = a;
    }
    if (p < pe) {
      uint64_t v = vals[rr];
      if (slopes) v += uint64_t(p - soffs[rr]) * slopes[rr];
      if (ob == 8) reinterpret_cast<uint64_t*>(out)[p] = v;
      else reinterpret_cast<uint32_t*>(out)[p] = uint32_t(v);
    }
    const uint32_t c2 = __popc(__ballot_sync(FULL, s <= p0 + 32));
    r += c2;
    if (c2 == 32) {
      while (r + 1 <= nr && soffs[r + 1] <= p0 + 32) r++;
    }
  }
}

// ------------------------------------------------------------------------------------------ pre-pass
constexpr int kIPer = kInnerTile / kThreads;  // 8 inner runs per thread

__global__ void __launch_bounds__(kThreads) inner_kernel(const __grid_constant__ InnerBatch B) {
  __shared__ uint64_t warp_s[kThreads / 32];
  __shared__ uint32_t tile_s, epoch_s;
  __shared__ uint64_t pc_s, pw_s;
  const uint32_t tid = threadIdx.x;
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
  const InnerDesc& D = B.d[find_desc(B, gt)];
  const uint32_t lt = gt - D.tile0;
  const uint32_t j0 = lt * kInnerTile;
  const uint32_t nvalid = min(uint32_t(kInnerTile), D.n_inner - j0);
  if (B.trace && tid == 0) {  // stamp 5: descriptor fields resident
    volatile uint64_t sink = D.dc_base + D.dv_base + D.dc_w + D.dv_w + uint64_t(D.dc_packed) + D.n_outer;
    (void)sink;
    trace_stamp(B.trace, gt, 5);
  }

  uint64_t dc[kIPer], dv[kIPer];
  uint64_t sc = 0, sw = 0;
  bool bad = false;
#pragma unroll
  for (int r = 0; r < kIPer; r++) {
    const uint32_t k = tid * kIPer + r;
    dc[r] = 0;
    dv[r] = 0;
    if (k < nvalid) {
      const uint64_t j = j0 + k;
      dc[r] = D.dc_base + extract_bits_global(reinterpret_cast<const uint32_t*>(D.dc_packed), j * D.dc_w, D.dc_w);
      dv[r] = D.dv_base + extract_bits_global(reinterpret_cast<const uint32_t*>(D.dv_packed), j * D.dv_w, D.dv_w);
      if (dc[r] > D.n_outer) { bad = true; dc[r] = 0; }
    }
    sc += dc[r];
    sw += dv[r] * dc[r];
  }
  trace_stamp(B.trace, gt, 1);
  uint64_t tc, tw;
  const uint64_t ec = block_excl_scan_u64<kThreads>(sc, warp_s, &tc);
  const uint64_t ew = block_excl_scan_u64<kThreads>(sw, warp_s, &tw);
  trace_stamp(B.trace, gt, 2);
  if (tid < 32) {
    uint64_t p0, p1;
    lb_tile(B.lb, gt, D.tile0, epoch, tc, tw, &p0, &p1);
    trace_stamp(B.trace, gt, 3);
    if (tid == 0) {
      pc_s = p0;
      pw_s = p1;
      if (lt + 1 == D.ntiles) {
        if (p0 + tc != D.n_outer) atomicOr(B.err + D.err_idx, 0x2u);
        D.tstart[D.outer_tiles] = D.n_inner - 1;  // closes the last outer tile's window
      }
    }
  }
  if (bad) atomicOr(B.err + D.err_idx, 0x2u);
  __syncthreads();
  uint64_t c = pc_s + ec, wsum = pw_s + ew;
#pragma unroll
  for (int r = 0; r < kIPer; r++) {
    const uint32_t k = tid * kIPer + r;
    if (k < nvalid) {
      const uint32_t j = j0 + k;
      D.S[j] = uint32_t(min(c, uint64_t(D.n_outer)));
      D.Q[j] = D.base + wsum;
      D.DV[j] = dv[r];
      if (dc[r] && c < D.n_outer) {  // outer tiles whose first run lies in this inner run
        const uint64_t last = min(c + dc[r], uint64_t(D.n_outer)) - 1;
        for (uint64_t t = (c + K - 1) / K; t <= last / K && t < D.outer_tiles; t++) D.tstart[t] = j;
      }
    }
    c += dc[r];
    wsum += dv[r] * dc[r];
  }
  trace_stamp(B.trace, gt, 4);
}

// ------------------------------------------------------------------------------------------ main
constexpr int kRPer = K / kThreads;  // 8 runs per thread

__global__ void __launch_bounds__(kThreads, 4) rle_kernel(const __grid_constant__ RleBatch B) {
  __shared__ uint32_t soffs_s[K + 1];
  __shared__ uint64_t vals_s[K];
  __shared__ __align__(16) uint8_t aux_s[K * 8];  // slopes (V_LINEAR) or the inner-run window (V_DRLE)
  uint64_t* slopes_s = reinterpret_cast<uint64_t*>(aux_s);
  uint64_t* iQ_s = reinterpret_cast<uint64_t*>(aux_s);
  uint64_t* iDV_s = iQ_s + (kRleWindow + 1);
  uint32_t* iS_s = reinterpret_cast<uint32_t*>(iDV_s + (kRleWindow + 1));
  static_assert((kRleWindow + 1) * 20 <= K * 8, "window must fit the aux buffer");
  __shared__ uint64_t warp_s[kThreads / 32];
  __shared__ uint32_t tile_s, epoch_s, skip_s, win_s, j0i_s;
  __shared__ uint64_t pc_s, pw_s;
  const uint32_t tid = threadIdx.x;
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
  const RleDesc& D = B.d[find_desc(B, gt)];
  const uint32_t lt = gt - D.tile0;
  const uint32_t g0 = lt * K;
  const uint32_t nr = min(uint32_t(K), D.nruns - g0);
  const uint8_t vmode = D.vmode;
  uint32_t errbits = 0;

  // V_DRLE: inner runs [tstart[lt], tstart[lt+1]] hold every outer run of this tile
  const uint32_t* wS = iS_s;
  const uint64_t* wQ = iQ_s;
  const uint64_t* wDV = iDV_s;
  if (vmode == V_DRLE) {
    if (tid == 0) {
      uint32_t j0i = D.tstart[lt], j1i = D.tstart[lt + 1];
      if (j0i >= D.n_inner) { j0i = 0; errbits |= 0x2u; }
      if (j1i >= D.n_inner || j1i < j0i) { j1i = D.n_inner - 1; }
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
      __syncthreads();
    } else {  // unusual data (many tiny inner runs): search the pre-pass arrays in global memory
      wS = D.S + j0i;
      wQ = D.Q + j0i;
      wDV = D.DV + j0i;
    }
  }

  trace_stamp(B.trace, gt, 5);  // window staged
  uint64_t cnt[kRPer], val[kRPer];
  uint64_t sc = 0, sw = 0;
  {
    const uint32_t kb = tid * kRPer;
    uint32_t a = 0;
    if (vmode == V_DRLE && kb < nr) {  // first window run with S <= g, then walk forward
      const uint32_t g = g0 + kb;
      uint32_t hi = win_s - 1;
      while (a < hi) {
        const uint32_t mid = (a + hi + 1) >> 1;
        if (wS[mid] <= g) a = mid; else hi = mid - 1;
      }
    }
#pragma unroll
    for (int r = 0; r < kRPer; r++) {
      const uint32_t k = kb + r;
      cnt[r] = 0;
      val[r] = 0;
      if (k < nr) {
        const uint64_t g = g0 + k;
        cnt[r] = D.cnt_base + extract_bits_global(reinterpret_cast<const uint32_t*>(D.cnt_packed), g * D.cnt_w, D.cnt_w);
        if (cnt[r] > D.n) { errbits |= 0x2u; cnt[r] = 0; }
        if (vmode == V_DRLE) {
          while (a + 1 < win_s && wS[a + 1] <= g) a++;
          val[r] = wQ[a] + (g - wS[a] + 1) * wDV[a];
        } else {
          const uint64_t x = D.val_base + extract_bits_global(reinterpret_cast<const uint32_t*>(D.val_packed),
                                                              g * D.val_w, D.val_w);
          if (vmode == V_BP || vmode == V_LINEAR) {
            val[r] = x;
          } else if (vmode == V_DICT) {
            uint64_t idx = x;
            if (idx >= D.entries) { errbits |= 0x1u; idx = 0; }
            val[r] = D.out_bytes == 8 ? __ldg(reinterpret_cast<const unsigned long long*>(D.dict) + idx)
                                      : uint64_t(__ldg(reinterpret_cast<const uint32_t*>(D.dict) + idx));
          } else {  // V_F2I
            val[r] = uint64_t(__double_as_longlong(double(int64_t(x)) / kPow10r[D.d]));
          }
        }
      }
      sc += cnt[r];
      if (vmode == V_LINEAR) sw += val[r] * cnt[r];
    }
  }
  trace_stamp(B.trace, gt, 1);
  uint64_t T, W = 0;
  const uint64_t ec = block_excl_scan_u64<kThreads>(sc, warp_s, &T);
  uint64_t ew = 0;
  if (vmode == V_LINEAR) ew = block_excl_scan_u64<kThreads>(sw, warp_s, &W);
  trace_stamp(B.trace, gt, 2);

  if (tid < 32) {
    uint64_t p0, p1;
    lb_tile(B.lb, gt, D.tile0, epoch, T, W, &p0, &p1);
    trace_stamp(B.trace, gt, 3);
    if (tid == 0) {
      pc_s = p0;
      pw_s = p1;
      const bool overflow = p0 + T > D.n;
      skip_s = overflow;
      if (overflow || (lt + 1 == D.ntiles && p0 + T != D.n)) atomicOr(B.err + D.err_idx, 0x2u);
    }
  }
  if (errbits) atomicOr(B.err + D.err_idx, errbits);
  __syncthreads();
  if (skip_s) return;  // corrupt counts: never write outside [0, n)

  // run table in shared memory (tile-relative starts, < 2^31 since the tile fits the chunk)
  {
    uint64_t c = ec, wv = pw_s + ew;
#pragma unroll
    for (int r = 0; r < kRPer; r++) {
      const uint32_t k = tid * kRPer + r;
      if (k < nr) {
        soffs_s[k] = uint32_t(c);
        if (vmode == V_LINEAR) {
          vals_s[k] = D.delta_base + wv + val[r];  // first element of the arithmetic run
          slopes_s[k] = val[r];
        } else {
          vals_s[k] = val[r];
        }
      }
      c += cnt[r];
      if (vmode == V_LINEAR) wv += val[r] * cnt[r];
    }
    if (tid == 0) soffs_s[nr] = uint32_t(T);
  }
  __syncthreads();

  const uint32_t O = uint32_t(pc_s);
  const uint32_t Tt = uint32_t(T);
  const uint64_t* slopes = vmode == V_LINEAR ? slopes_s : nullptr;
  if (Tt <= kRleBigLimit || !B.big_enabled) {
    uint8_t* out = reinterpret_cast<uint8_t*>(D.out) + uint64_t(O) * D.out_bytes;
    const uint32_t warp = tid >> 5;
    const uint32_t span = ((Tt + kThreads - 1) / kThreads) * 32;
    const uint32_t pb = min(Tt, warp * span), pe = min(Tt, pb + span);
    expand_warp(soffs_s, nr, vals_s, slopes, pb, pe, out, D.out_bytes);
    __syncthreads();
    trace_stamp(B.trace, gt, 4);
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
        en.out_bytes = D.out_bytes;
        en.linear = vmode == V_LINEAR;
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
      for (uint32_t k = tid; k <= nr; k += kThreads) so[k] = soffs_s[k];
      for (uint32_t k = tid; k < nr; k += kThreads) {
        va[k] = vals_s[k];
        if (slopes) sl[k] = slopes_s[k];
      }
    }
  }
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
    const uint32_t span = ((pe0 - pb0 + kThreads - 1) / kThreads) * 32;
    const uint32_t pb = min(pe0, pb0 + warp * span), pe = min(pe0, pb + span);
    uint8_t* out = reinterpret_cast<uint8_t*>(en.out) + uint64_t(en.O) * en.out_bytes;
    expand_warp(G.soffs + uint64_t(en.slot) * (K + 1), en.nr, G.vals + uint64_t(en.slot) * K,
                en.linear ? G.slopes + uint64_t(en.slot) * K : nullptr, pb, pe, out, en.out_bytes);
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

cudaError_t launch_inner(const InnerBatch& b, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  inner_kernel<<<b.total_tiles, kThreads, 0, s>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_rle(const RleBatch& b, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  rle_kernel<<<b.total_tiles, kThreads, 0, s>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_rle_big(const RleBatch& b, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  rle_big_kernel<<<device_sms() * 2, kThreads, 0, s>>>(b);
  return cudaGetLastError();
}

}  // namespace cdm
