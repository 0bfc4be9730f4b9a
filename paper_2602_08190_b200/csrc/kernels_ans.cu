// kernels_ans.cu -- NEXT-1: chunk-sequential ("Non-Parallel") range-ANS decode.
//
// "Each intermediate decode state in ANS depends on its predecessor ... opportunities for
// parallelism arise by grouping their intermediate decode states from different chunks and dispatching
// them in a SIMT manner".  This kernel is exactly that schedule: ONE THREAD PER ANS CHUNK, a warp advances
// 32 independent chunk states in lockstep.  Format (reading R32): range ANS
// with a 32-bit state x in [2^16, 2^32), 16-bit renormalisation words, one frequency table normalised to
// 2^tl shared by the chunks of a CDM1 chunk; each ANS chunk stores its initial decoder state, its words in
// decode order, and must end at state 2^16 with every word consumed (else CDM_ERR_ANS = 0x20).
//
// il = 1 (one state per chunk): a CTA takes 256 consecutive chunks of one column chunk; it first expands the shared table
// into a shared-memory slot table (2^tl packed entries {symbol, slot - cum, f}, tl <= 12), so the
// per-symbol step is one shared load + a multiply-add; every thread gathers 4 decoded bytes into a
// register and writes them with one 4-byte store.
#include "device_util.cuh"
#include "kernels.h"

namespace cdm {
namespace {

using namespace dev;

constexpr uint32_t kAnsMaxTl = 12;

__device__ __forceinline__ int find_desc_ans(const AnsBatch& B, uint32_t tile) {
  int lo = 0, hi = int(B.n) - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (B.d[mid].tile0 <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// The CTA's slot table from the 256 frequencies: cum_s = exclusive scan, tab_s[slot] = packed {symbol, slot - cum,
// f}; returns whether the frequencies sum to M (else every chunk reports CDM_ERR_ANS).
__device__ __forceinline__ bool build_slot_table(const uint8_t* table, uint32_t& tl, uint32_t* tab_s, uint32_t* cum_s,
                                                 uint64_t* warp_s) {
  uint32_t M = 1u << tl;
  const uint32_t tid = threadIdx.x;
  {
    const uint32_t f = tid < 256 ? uint32_t(__ldg(reinterpret_cast<const uint16_t*>(table) + tid)) : 0u;
    uint64_t tot;
    const uint32_t ex = uint32_t(block_excl_scan_u64<kThreads>(f, warp_s, &tot));
    if (tid < 256) cum_s[tid] = ex;
    if (tid == 0) cum_s[256] = uint32_t(tot);
  }
  __syncthreads();
  const bool ok = cum_s[256] == M;
  // f = 2^12 (one symbol owns the whole table) does not fit the 12-bit f field; such a step is the identity
  // x' = M (x >> tl) + (x & (M - 1)) = x for every table log, so that table decodes with tl = 11 and f = 2^11
  if (__syncthreads_or(M == 4096u && tid < 256 && cum_s[tid + 1] - cum_s[tid] == M)) { tl = 11; M = 2048; }
  for (uint32_t slot = tid; slot < M; slot += kThreads) {
    uint32_t lo = 0, hi = 255;
    while (lo < hi) {  // last symbol with cum <= slot
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (cum_s[mid] <= slot) lo = mid; else hi = mid - 1;
    }
    const uint32_t f = min(cum_s[lo + 1] - cum_s[lo], M);
    tab_s[slot] = lo | (slot - cum_s[lo]) << 8 | f << 20;
  }
  __syncthreads();
  return ok;
}

__global__ void __launch_bounds__(kThreads) ans_kernel(const __grid_constant__ AnsBatch B) {
  __shared__ uint32_t tab_s[1u << kAnsMaxTl];  // slot -> sym | (slot - cum) << 8 | f << 20
  __shared__ uint32_t cum_s[257];
  __shared__ uint64_t warp_s[kThreads / 32];
  const uint32_t tid = threadIdx.x;
  const AnsDesc& D = B.d[find_desc_ans(B, blockIdx.x)];
  uint32_t tl = D.tl;
  const uint8_t* const table = D.table;
  const bool table_ok = build_slot_table(table, tl, tab_s, cum_s, warp_s);
  const uint32_t M = 1u << tl;
  const uint32_t c = (blockIdx.x - D.tile0) * kThreads + tid;  // this thread's chunk
  if (c >= D.nchunks) return;
  bool bad = !table_ok;
  const uint8_t* ce = table + 512 + 12ull * c;
  const uint32_t w0 = __ldg(reinterpret_cast<const uint32_t*>(ce)), nw = __ldg(reinterpret_cast<const uint32_t*>(ce + 4));
  uint32_t x = __ldg(reinterpret_cast<const uint32_t*>(ce + 8));
  if (uint64_t(w0) + nw > D.n_words) bad = true;
  const uint64_t i0 = uint64_t(c) * D.chunk;
  const uint32_t len = uint32_t(min(uint64_t(D.chunk), D.n - i0));
  const uint16_t* __restrict__ wp = D.words + w0;
  uint32_t pos = 0;
  uint8_t* out = D.out + i0;
  const uint32_t mask = M - 1u;
  // the next renormalisation word is loaded as soon as the previous one is consumed, so its global-memory
  // latency overlaps the symbols decoded in between
  uint32_t wnext = nw ? uint32_t(__ldg(wp)) : 0u;
  auto step = [&](uint32_t& x) -> uint32_t {
    const uint32_t e = tab_s[x & mask];
    x = (e >> 20) * (x >> tl) + ((e >> 8) & 0xFFFu);
    if (x < (1u << 16)) {  // one step suffices: x >= 2^(16 - tl) here, tl <= 12
      bad |= pos >= nw;
      x = (x << 16) | wnext;
      pos++;
      wnext = pos < nw ? uint32_t(__ldg(wp + pos)) : 0u;
    }
    return e & 0xFFu;
  };
  if (!bad) {
    uint32_t i = 0;
    for (; i + 4 <= len; i += 4) {  // 4 symbols -> one 4-byte store (chunks are 16-byte multiples)
      uint32_t word = 0;
#pragma unroll
      for (int j = 0; j < 4; j++) word |= step(x) << (8 * j);
      *reinterpret_cast<uint32_t*>(out + i) = word;
    }
    for (; i < len; i++) out[i] = uint8_t(step(x));  // the column chunk's ragged tail
    if (x != (1u << 16) || pos != nw) bad = true;
  }
  if (bad) atomicOr(B.err + D.err_idx, 0x20u);
}


// il = 32 (the default format, SURVEY Sec. 8f NEXT-1 "interleaved rANS, warp-per-chunk"): one WARP per ANS
// chunk, lane l owns state l and decodes symbols 32s + l, so a warp emits 32 consecutive bytes per step and a
// chunk's dependency chain is chunk/32 steps long.  The states that renormalise at a step take consecutive
// words in lane order (ballot + popcount rank); the chunk's next 64 words sit in two registers per lane
// (one word per lane each) and reach the renormalising lanes by shuffle, refilled 32 words at a time from a
// third register whose coalesced load was issued one slide earlier.  A CTA's 8 warps take B.cpw rounds of 8 chunks, so the slot table is built once per
// 8 * cpw chunks.
__global__ void __launch_bounds__(kThreads) ans_warp_kernel(const __grid_constant__ AnsBatch B) {
  __shared__ uint32_t tab_s[1u << kAnsMaxTl];
  __shared__ uint32_t cum_s[257];
  __shared__ uint64_t warp_s[kThreads / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const AnsDesc& D = B.d[find_desc_ans(B, blockIdx.x)];
  uint32_t tl = D.tl;
  const uint8_t* const table = D.table;
  const bool table_ok = build_slot_table(table, tl, tab_s, cum_s, warp_s);
  const uint32_t M = 1u << tl;
  const uint32_t mask = M - 1u, lt_mask = (1u << lane) - 1u;
  for (uint32_t rnd = 0; rnd < B.cpw; rnd++) {
    const uint32_t c = ((blockIdx.x - D.tile0) * B.cpw + rnd) * (kThreads / 32) + warp;  // this warp's chunk
    if (c >= D.nchunks) break;  // warp-uniform
    const uint8_t* ce = table + 512 + 136ull * c;
    const uint32_t w0 = __ldg(reinterpret_cast<const uint32_t*>(ce)), nw = __ldg(reinterpret_cast<const uint32_t*>(ce + 4));
    uint32_t x = __ldg(reinterpret_cast<const uint32_t*>(ce + 8) + lane);
    bool bad = !table_ok || uint64_t(w0) + nw > D.n_words;
    const uint64_t i0 = uint64_t(c) * D.chunk;
    const uint32_t len = uint32_t(min(uint64_t(D.chunk), D.n - i0));
    const uint16_t* __restrict__ wp = D.words + w0;
    uint8_t* out = D.out + i0;
    auto ldw = [&](uint32_t q) -> uint32_t { return q < nw ? uint32_t(__ldg(wp + q)) : 0u; };
    // words [wbase, wbase + 64) are resident in (cur, nxt); pre holds [wbase + 64, wbase + 96), loaded one slide
    // ahead so its latency overlaps the ~10 steps that consume a 32-word slice (the shuffles never read it)
    uint32_t wbase = 0, cur = 0, nxt = 0, pre = 0, pos = 0;
    if (!bad) { cur = ldw(lane); nxt = ldw(32 + lane); pre = ldw(64 + lane); }
    // one decode step of the warp (32 symbols); words past nw read as 0 (ldw) and over-consumption shows in
    // the final pos == nw check, so the step itself carries no bounds test
    auto step = [&](uint32_t i0, bool act) {
      const uint32_t e = tab_s[x & mask];
      const uint32_t xn = (e >> 20) * (x >> tl) + ((e >> 8) & 0xFFFu);
      const bool need = act && xn < (1u << 16);  // one step suffices for tl <= 12
      const uint32_t m = __ballot_sync(FULL, need);
      const uint32_t q = pos + __popc(m & lt_mask) - wbase;  // word index relative to the window (< 64)
      const uint32_t a = __shfl_sync(FULL, cur, q & 31), b = __shfl_sync(FULL, nxt, q & 31);
      const uint32_t w = q < 32 ? a : b;
      x = need ? (xn << 16) | w : (act ? xn : x);
      if (act) out[i0 + lane] = uint8_t(e & 0xFFu);
      pos += __popc(m);
      if (pos >= wbase + 32) {  // warp-uniform: slide the window by 32 words
        wbase += 32;
        cur = nxt;
        nxt = pre;
        pre = ldw(wbase + 64 + lane);
      }
    };
    const uint32_t full = bad ? 0u : len / 32, tail = bad ? 0u : len % 32;
#pragma unroll 8  // measured: unroll 2 / 4 / 8 / 16 -> 554 / 613 / 628-644 / 640-644 GB/s (ans workload)
    for (uint32_t st = 0; st < full; st++) step(32 * st, true);
    if (tail) step(32 * full, lane < tail);
    bad |= !__all_sync(FULL, x == (1u << 16)) || pos != nw;
    if (bad && lane == 0) atomicOr(B.err + D.err_idx, 0x20u);
  }
}

}  // namespace

cudaError_t launch_ans(const AnsBatch& b, bool interleaved, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  if (interleaved) ans_warp_kernel<<<b.total_tiles, kThreads, 0, s>>>(b);
  else ans_kernel<<<b.total_tiles, kThreads, 0, s>>>(b);
  return cudaGetLastError();
}

}  // namespace cdm
