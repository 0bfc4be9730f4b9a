// device_util.cuh -- sm_100a device helpers shared by the decode kernels (never by the oracle).
//
//  * LSB-first contiguous bit-field extraction (reading R1) from shared or global words.
//  * 1-D TMA bulk copies global->shared completing on an mbarrier (cp.async.bulk + expect_tx).
//  * Tile tickets + epoch-tagged decoupled look-back (single-pass scan; Merrill & Garland style) used by
//    the scan-dependent ("Group-Parallel") kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cdm {
namespace dev {

constexpr unsigned FULL = 0xFFFFFFFFu;

// ------------------------------------------------------------------ bit extraction
// Field i of width w (0..64) from 32-bit little-endian words `wd` (bit k of the stream is bit (k&31) of
// word k>>5).  Reads words [k>>5, (k>>5)+2]; callers guarantee those words are readable.
__device__ __forceinline__ uint64_t extract_bits(const uint32_t* wd, uint64_t bitoff, uint32_t w) {
  const uint64_t wi = bitoff >> 5;
  const uint32_t sh = uint32_t(bitoff & 31);
  const uint32_t a = wd[wi], b = wd[wi + 1];
  const uint32_t lo = __funnelshift_r(a, b, sh);
  if (w <= 32) return w == 32 ? lo : (lo & ((1u << w) - 1u));
  const uint32_t c = wd[wi + 2];
  const uint32_t hi = __funnelshift_r(b, c, sh);
  const uint64_t v = (uint64_t(hi) << 32) | lo;
  return w == 64 ? v : (v & ((1ull << w) - 1ull));
}

// Same, through the read-only path from global memory (small streams: RLE counts/values).
// Cooperative, coalesced copy of the packed bits of items [i0, i0 + cnt) of a w-bit stream into shared
// words.  i0 is a multiple of 2048, so i0 * w is word aligned.  Copies two words past the last field
// (extraction reads up to word k+2); the stream's 16-byte slack keeps that in bounds.
template <int NT>
__device__ __forceinline__ void stage_bits(uint32_t* dst, const uint8_t* packed, uint64_t i0, uint32_t cnt,
                                           uint32_t w) {
  if (w == 0) return;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(packed) + (i0 * w >> 5);
  const uint32_t nw = uint32_t((uint64_t(cnt) * w + 31) / 32) + 2;
  for (uint32_t k = threadIdx.x; k < nw; k += NT) dst[k] = __ldg(src + k);
}

__device__ __forceinline__ uint64_t extract_bits_global(const uint32_t* __restrict__ wd, uint64_t bitoff,
                                                        uint32_t w) {
  if (w == 0) return 0;
  const uint64_t wi = bitoff >> 5;
  const uint32_t sh = uint32_t(bitoff & 31);
  const uint32_t a = __ldg(wd + wi), b = __ldg(wd + wi + 1);
  const uint32_t lo = __funnelshift_r(a, b, sh);
  if (w <= 32) return w == 32 ? lo : (lo & ((1u << w) - 1u));
  const uint32_t c = __ldg(wd + wi + 2);
  const uint32_t hi = __funnelshift_r(b, c, sh);
  const uint64_t v = (uint64_t(hi) << 32) | lo;
  return w == 64 ? v : (v & ((1ull << w) - 1ull));
}

// Batched form for memory-level parallelism: U fields (bit offsets off[u], same width w) -- all 3U word loads
// are issued before any use (no branches between them), then the fields are assembled.  Reads up to two
// words past a field; the 16-byte stream slack keeps that in bounds.
template <int U>
__device__ __forceinline__ void extract_bits_global_batch(const uint32_t* __restrict__ wd, const uint64_t (&off)[U],
                                                          uint32_t w, uint64_t (&out)[U]) {
  uint32_t a[U], b[U], c[U];
#pragma unroll
  for (int u = 0; u < U; u++) {
    const uint64_t wi = off[u] >> 5;
    a[u] = __ldg(wd + wi);
    b[u] = __ldg(wd + wi + 1);
    c[u] = __ldg(wd + wi + 2);
  }
  const uint64_t mask = w >= 64 ? ~0ull : ((1ull << w) - 1ull);
#pragma unroll
  for (int u = 0; u < U; u++) {
    const uint32_t sh = uint32_t(off[u] & 31);
    const uint64_t v = (uint64_t(__funnelshift_r(b[u], c[u], sh)) << 32) | __funnelshift_r(a[u], b[u], sh);
    out[u] = w ? (v & mask) : 0ull;
  }
}

// ------------------------------------------------------------------ mbarrier + TMA bulk copy
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}
// Order this thread's earlier generic-proxy shared-memory accesses (made visible CTA-wide by a preceding
// barrier) before subsequent async-proxy (TMA) writes to the same buffer.
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 1-D bulk copy (TMA engine) of `bytes` (multiple of 16, 16-aligned src/dst) completing on `bar`.
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// ------------------------------------------------------------------ vector stores
__device__ __forceinline__ void st_v4_u32(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void st_v2_u64(void* p, uint64_t a, uint64_t b) {
  asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

// ------------------------------------------------------------------ tickets + look-back
// A launch-wide 64-bit counter: high 32 bits = epoch, low 32 bits = next ticket.  One atomicAdd hands a
// CTA both its tile ticket and the launch epoch; the CTA drawing the last ticket (`last`) bumps the epoch
// and resets the ticket, so the counter needs no memset and survives CUDA-graph replays.
__device__ __forceinline__ void take_ticket(unsigned long long* ctr, uint32_t last, uint32_t* ticket,
                                            uint32_t* epoch) {
  const unsigned long long v = atomicAdd(ctr, 1ull);
  *ticket = uint32_t(v & 0xFFFFFFFFull);
  *epoch = uint32_t(v >> 32) & 0x3FFFFFFFu;
  if (*ticket == last) atomicExch(ctr, (unsigned long long)(*epoch + 1) << 32);
}

// Look-back record of tile t: three 16-byte words -- [3t] the flag word {flag = (epoch << 2) | state}, [3t+1]
// the AGG values {c (u32, saturating count), w (u64, wrapping)}, [3t+2] the INC values.  A publisher writes
// the state's value word, then the flag with a release store; a reader acquires the flag, then reads the
// value word of the state it saw.  Each value word is written once per epoch, before its flag, so a reader
// never combines a flag with values it does not belong to -- without relying on 16-byte store atomicity
// (the PTX memory model promises single-copy atomicity only up to 8 bytes).
constexpr uint32_t LB_AGG = 1, LB_INC = 2;

__device__ __forceinline__ void lb_store_vals(uint4* p, uint32_t c, uint64_t w) {
  asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(0u), "r"(c), "r"(uint32_t(w)),
               "r"(uint32_t(w >> 32))
               : "memory");
}
__device__ __forceinline__ void lb_store_flag(uint4* p, uint32_t flag) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(flag) : "memory");
}
__device__ __forceinline__ uint32_t lb_load_flag(const uint4* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint4 lb_load_vals(const uint4* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

__device__ __forceinline__ uint32_t sat32(uint64_t x) { return x > 0xFFFFFFFFull ? 0xFFFFFFFFu : uint32_t(x); }

__device__ __forceinline__ void lb_publish(uint4* words, uint32_t gt, uint32_t epoch, uint32_t state, uint64_t c,
                                           uint64_t w) {
  lb_store_vals(words + 3ull * gt + state, sat32(c), w);
  lb_store_flag(words + 3ull * gt, (epoch << 2) | state);
}

// Single-warp decoupled look-back: lanes probe 32 predecessors at a time (gt-1-lane) and fold the AGG
// values up to the nearest INC.  `first_gt` is the chunk's first tile (prefix 0).  Called by all 32 lanes
// of one warp; returns the exclusive prefix in every lane (count saturating at 2^32-1, w mod 2^64).
__device__ __forceinline__ void lb_lookback(const uint4* words, uint32_t gt, uint32_t first_gt, uint32_t epoch,
                                            uint64_t* pc, uint64_t* pw) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t acc_c = 0, acc_w = 0;
  int64_t base = int64_t(gt) - 1;  // highest predecessor not yet folded
  while (base >= int64_t(first_gt)) {
    const int64_t me = base - lane;
    uint32_t st = LB_INC;  // lanes below the chunk start act as a terminating INC with value 0
    uint64_t c = 0, w = 0;
    if (me >= int64_t(first_gt)) {
      uint32_t f;
      do {
        f = lb_load_flag(words + 3ull * me);
      } while ((f >> 2) != epoch || (f & 3u) == 0);
      st = f & 3u;
      const uint4 v = lb_load_vals(words + 3ull * me + st);
      c = v.y;
      w = (uint64_t(v.w) << 32) | v.z;
    }
    const uint32_t incmask = __ballot_sync(FULL, st == LB_INC);
    const uint32_t stop = incmask ? uint32_t(__ffs(incmask) - 1) : 32u;
    if (lane > stop) { c = 0; w = 0; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      c += __shfl_xor_sync(FULL, c, o);
      w += __shfl_xor_sync(FULL, w, o);
    }
    acc_c += c;
    acc_w += w;
    if (incmask) break;
    base -= 32;
  }
  *pc = sat32(acc_c);
  *pw = acc_w;
}

// The whole protocol for one tile, run by warp 0: publish AGG (or INC for the chunk's first tile), look
// back, publish INC.  Returns the tile's exclusive prefix (count, w) in every lane.
__device__ __forceinline__ void lb_tile(uint4* words, uint32_t gt, uint32_t first_gt, uint32_t epoch, uint64_t agg_c,
                                        uint64_t agg_w, uint64_t* pc, uint64_t* pw) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t c = 0, w = 0;
  if (gt == first_gt) {
    if (lane == 0) lb_publish(words, gt, epoch, LB_INC, agg_c, agg_w);
  } else {
    if (lane == 0) lb_publish(words, gt, epoch, LB_AGG, agg_c, agg_w);
    lb_lookback(words, gt, first_gt, epoch, &c, &w);
    if (lane == 0) lb_publish(words, gt, epoch, LB_INC, c + agg_c, w + agg_w);
  }
  *pc = c;
  *pw = w;
}

// ------------------------------------------------------------------ tracing (CDM_TRACE)
// Programmatic dependent launch (no-ops when the launch did not enable it).
__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}
// stamp phase k of tile gt (thread 0 only; no-op unless the launch carries a trace buffer)
__device__ __forceinline__ void trace_stamp(uint64_t* trace, uint32_t gt, int k) {
  if (trace && threadIdx.x == 0) trace[uint64_t(gt) * 8 + k] = k == 7 ? smid() : globaltimer();
}

// ------------------------------------------------------------------ block scans (256 threads)
// Exclusive scan of one u64 per thread across the CTA; returns the exclusive prefix, *total = sum.
template <int NT>
__device__ __forceinline__ uint64_t block_excl_scan_u64(uint64_t v, uint64_t* smem_warp /*[NT/32]*/,
                                                        uint64_t* total) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= uint32_t(o)) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  uint64_t wp = 0, tot = 0;
#pragma unroll
  for (int k = 0; k < NT / 32; k++) {
    const uint64_t s = smem_warp[k];
    if (uint32_t(k) < warp) wp += s;
    tot += s;
  }
  __syncthreads();
  *total = tot;
  return wp + x - v;
}

// Exclusive scan of one value per thread across the CTA in T arithmetic (uint32_t: mod 2^32) with log-step
// scans at both levels: a shuffle scan inside each warp, then every warp scans the NT/32 warp totals with
// shuffles (no serial loop over the warps).  Returns the exclusive prefix; *total = the CTA's sum.
template <int NT, typename T>
__device__ __forceinline__ T block_excl_scan_log(T v, T* smem_warp /*[NT/32]*/, T* total) {
  constexpr int NW = NT / 32;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(FULL, x, o);
    if (lane >= uint32_t(o)) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  T w = lane < uint32_t(NW) ? smem_warp[lane] : T(0);
#pragma unroll
  for (int o = 1; o < NW; o <<= 1) {
    const T y = __shfl_up_sync(FULL, w, o);
    if (lane >= uint32_t(o)) w += y;
  }
  const T wp = warp ? __shfl_sync(FULL, w, warp - 1) : T(0);
  *total = __shfl_sync(FULL, w, NW - 1);
  __syncthreads();
  return wp + x - v;
}

// Exclusive scan of a pair (a, b) of u64 per thread across the CTA with one barrier pair; *ta, *tb = totals.
// smem_warp holds 2 * NT/32 words.  The warp totals are scanned by every warp with one shuffle scan.
template <int NT>
__device__ __forceinline__ void block_excl_scan_pair(uint64_t a, uint64_t b, uint64_t* smem_warp, uint64_t* ea,
                                                     uint64_t* eb, uint64_t* ta, uint64_t* tb) {
  static_assert(NT % 32 == 0 && NT <= 1024, "block size");
  constexpr int NW = NT / 32;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t x = a, y = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t u = __shfl_up_sync(FULL, x, o);
    const uint64_t v = __shfl_up_sync(FULL, y, o);
    if (lane >= uint32_t(o)) { x += u; y += v; }
  }
  if (lane == 31) { smem_warp[2 * warp] = x; smem_warp[2 * warp + 1] = y; }
  __syncthreads();
  // lane k < NW holds warp k's totals; an inclusive shuffle scan over them
  uint64_t wx = lane < uint32_t(NW) ? smem_warp[2 * lane] : 0ull;
  uint64_t wy = lane < uint32_t(NW) ? smem_warp[2 * lane + 1] : 0ull;
#pragma unroll
  for (int o = 1; o < NW; o <<= 1) {
    const uint64_t u = __shfl_up_sync(FULL, wx, o);
    const uint64_t v = __shfl_up_sync(FULL, wy, o);
    if (lane >= uint32_t(o)) { wx += u; wy += v; }
  }
  const uint64_t px = warp ? __shfl_sync(FULL, wx, warp - 1) : 0ull;
  const uint64_t py = warp ? __shfl_sync(FULL, wy, warp - 1) : 0ull;
  *ta = __shfl_sync(FULL, wx, NW - 1);
  *tb = __shfl_sync(FULL, wy, NW - 1);
  __syncthreads();
  *ea = px + x - a;
  *eb = py + y - b;
}


// ---- byte-granular 16-byte moves (LZ4, String-dictionary)
__device__ __forceinline__ uint2 ld_v2_global(const void* p) {  // coherent (the thread's own earlier stores)
  uint2 v;
  asm volatile("ld.global.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint2 ld_v2_nc(const void* p) { return __ldg(reinterpret_cast<const uint2*>(p)); }

// bytes [a, a + k) (k <= 16) into v (little-endian words); only the 8-byte words holding them are read
template <bool NC>
__device__ __forceinline__ void load16(const uint8_t* a, uint32_t k, uint32_t (&v)[4]) {
  const uintptr_t p = reinterpret_cast<uintptr_t>(a);
  const uint8_t* b = reinterpret_cast<const uint8_t*>(p & ~uintptr_t(7));
  const uint32_t f = uint32_t(p & 7u);
  const uint2 z = make_uint2(0u, 0u);
  const uint2 x0 = NC ? ld_v2_nc(b) : ld_v2_global(b);
  const uint2 x1 = f + k > 8 ? (NC ? ld_v2_nc(b + 8) : ld_v2_global(b + 8)) : z;
  const uint2 x2 = f + k > 16 ? (NC ? ld_v2_nc(b + 16) : ld_v2_global(b + 16)) : z;
  const bool hi = f >= 4;
  const uint32_t sh = (f & 3u) * 8u;
  const uint32_t w0 = hi ? x0.y : x0.x, w1 = hi ? x1.x : x0.y, w2 = hi ? x1.y : x1.x, w3 = hi ? x2.x : x1.y,
                 w4 = hi ? x2.y : x2.x;
  v[0] = __funnelshift_r(w0, w1, sh);
  v[1] = __funnelshift_r(w1, w2, sh);
  v[2] = __funnelshift_r(w2, w3, sh);
  v[3] = __funnelshift_r(w3, w4, sh);
}

// explicit shared-space accesses (32-bit shared addresses): the output image is only touched through these
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_v4(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void reds_or(uint32_t a, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// 16 bytes at shared byte address a (any alignment; the 4 bytes after a + 16 must be readable)
__device__ __forceinline__ void sload16(uint32_t a, uint32_t (&v)[4]) {
  const uint32_t b = a & ~3u, sh = (a & 3u) * 8u;
  const uint32_t w0 = lds_u32(b), w1 = lds_u32(b + 4), w2 = lds_u32(b + 8), w3 = lds_u32(b + 12), w4 = lds_u32(b + 16);
  v[0] = __funnelshift_r(w0, w1, sh);
  v[1] = __funnelshift_r(w1, w2, sh);
  v[2] = __funnelshift_r(w2, w3, sh);
  v[3] = __funnelshift_r(w3, w4, sh);
}
// bytes [0, k) of v (1 <= k <= 16) to shared byte address a of a ZEROED image whose other bytes other lanes may
// be writing: whole words with one store, partial words OR-ed in (only this lane's bytes are non-zero)
__device__ __forceinline__ void sstore16(uint32_t a, const uint32_t (&v)[4], uint32_t k) {
  const uint32_t a3 = a & 3u, sh = 8u * a3, base = a & ~3u, e = a3 + k;
  uint32_t u[5];
  u[0] = v[0] << sh;
  u[1] = __funnelshift_l(v[0], v[1], sh);
  u[2] = __funnelshift_l(v[1], v[2], sh);
  u[3] = __funnelshift_l(v[2], v[3], sh);
  u[4] = sh ? (v[3] >> (32u - sh)) : 0u;
#pragma unroll
  for (int i = 0; i < 5; i++) {
    const int lo = max(int(a3) - 4 * i, 0), hi = min(int(e) - 4 * i, 4);
    if (hi > lo) {
      if (hi - lo == 4) sts_u32(base + 4 * i, u[i]);
      else reds_or(base + 4 * i, u[i] & (((1u << (8 * (hi - lo))) - 1u) << (8 * lo)));
    }
  }
}


}  // namespace dev
}  // namespace cdm
