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
#include <cstdlib>

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
  if (D.uniform) {
    off = uint64_t(s) * D.uniform;  // host-verified uniform sub-chunk sizes
  } else {
    for (uint32_t k = lane; k < s; k += 32) off += __ldg(tab + 3 * k + 2);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) off += __shfl_xor_sync(FULL, off, o);
  }
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

// ------------------------------------------------------------------------------------------ lane groups
// 32/kLzG sub-chunks per warp, kLzG lanes each (default 4: eight sub-chunks per warp; CDM_LZ4_G=8/16): the warp-per-sub-chunk schedule spends ~130
// warp instructions per LZ4 sequence of ~8 output bytes (31 lanes mostly idle on short sequences); eight
// lanes match the typical sequence and four groups share every instruction.  Per sequence a group loads one
// 8-byte window of the compressed stream (one byte per lane) that usually holds the token, the literals and
// the offset (shuffled out within the group); literal and match bytes are copied 8 per step with
// out[p + k] = out[p - o + (k mod o)] for overlapping short periods; __syncwarp(group mask) orders a
// group's stores before its match reads.  Same bounds checks and error bit as lz4_kernel.
// kWB = window bytes per lane: 1 (one compressed byte per lane), or 4 (each lane holds 4 bytes -- two
// aligned words + a funnel shift -- so a 4-lane group sees 16 bytes: token, literals and offset of most
// sequences in one load round).
template <uint32_t kLzG, uint32_t kWB>  // lanes per sub-chunk, window bytes per lane
__global__ void __launch_bounds__(kWarpsPerCta * 32) lz4_group_kernel(const __grid_constant__ Lz4Batch B) {
  constexpr uint32_t kWS = kLzG * kWB;  // window bytes per group
  const uint32_t lane = threadIdx.x & 31, gl = lane & (kLzG - 1);
  const uint32_t gmask = (kLzG == 32 ? FULL : ((1u << kLzG) - 1u)) << (lane & ~(kLzG - 1));
  const uint32_t gs = (blockIdx.x * (kWarpsPerCta * 32) + threadIdx.x) / kLzG;
  if (gs >= B.total_subs) return;  // uniform within a group
  const Lz4Desc& D = B.d[find_desc_lz4(B, gs)];
  const uint32_t s = gs - D.sub0;
  const uint32_t* tab = reinterpret_cast<const uint32_t*>(D.table);
  uint64_t off = 0;
  if (D.uniform) {
    off = uint64_t(s) * D.uniform;
  } else {
    for (uint32_t k = gl; k < s; k += kLzG) off += __ldg(tab + 3 * k + 2);
#pragma unroll
    for (int o = kLzG / 2; o > 0; o >>= 1) off += __shfl_xor_sync(gmask, off, o, kLzG);
  }
  const uint32_t co = __ldg(tab + 3 * s), cl = __ldg(tab + 3 * s + 1), dl = __ldg(tab + 3 * s + 2);
  bool bad = uint64_t(co) + cl > D.payload_bytes || off + dl > D.n;
  if (s + 1 == D.n_sub && off + dl != D.n) bad = true;
  if (bad) {
    if (gl == 0) atomicOr(B.err + D.err_idx, 0x4u);
    return;
  }
  const uint8_t* __restrict__ in = D.payload + co;
  uint8_t* out = D.out + off;
  uint32_t ip = 0, op = 0;
  for (;;) {
    if (ip >= cl) { bad = true; break; }
    // window: compressed bytes [ip, ip + kWS), kWB per lane (bytes past cl are never used: every use below
    // is bounds-checked against cl; the stream's 16 slack bytes keep the aligned word reads in bounds)
    uint32_t wb;
    if (kWB == 1) {
      wb = ip + gl < cl ? uint32_t(__ldg(in + ip + gl)) : 0u;
    } else {
      const uintptr_t a = reinterpret_cast<uintptr_t>(in + ip + kWB * gl);
      const uint32_t* pw = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
      wb = ip + kWB * gl < cl ? __funnelshift_r(__ldg(pw), __ldg(pw + 1), uint32_t(a & 3u) * 8u) : 0u;
    }
    // window byte j (j < kWS for a meaningful value; the lane index wraps modulo the group otherwise)
    auto wbyte = [&](uint32_t j) -> uint32_t {
      const uint32_t v = __shfl_sync(gmask, wb, j / kWB, kLzG);
      return kWB == 1 ? v : (v >> ((j % kWB) * 8u)) & 0xFFu;
    };
    const uint32_t token = wbyte(0);
    uint32_t lit = token >> 4;
    uint32_t q = ip + 1;
    if (lit == 15) {
      uint32_t b;
      do {
        if (q >= cl) { bad = true; break; }
        b = __ldg(in + q++);
        lit += b;
      } while (b == 255);
      if (bad) break;
    }
    if (lit > cl - q || lit > dl - op) { bad = true; break; }
    if (q + lit <= ip + kWS) {  // literals inside the window: lane gl takes window bytes (q - ip) + gl + kLzG*t
      for (uint32_t base = 0; base < lit; base += kLzG) {  // group-uniform trip count (shuffles inside)
        const uint32_t v = wbyte(q - ip + base + gl);
        if (base + gl < lit) out[op + base + gl] = uint8_t(v);
      }
    } else {
      for (uint32_t k = gl; k < lit; k += kLzG) out[op + k] = __ldg(in + q + k);
    }
    q += lit;
    op += lit;
    if (q == cl) break;  // the last sequence carries literals only
    if (cl - q < 2) { bad = true; break; }
    uint32_t moff;
    if (q + 2 <= ip + kWS) {
      moff = wbyte(q - ip) | (wbyte(q - ip + 1) << 8);
    } else {
      moff = uint32_t(__ldg(in + q)) | (uint32_t(__ldg(in + q + 1)) << 8);
    }
    q += 2;
    if (moff == 0 || moff > op) { bad = true; break; }
    uint32_t ml = token & 15;
    if (ml == 15) {
      uint32_t b;
      do {
        if (q >= cl) { bad = true; break; }
        b = __ldg(in + q++);
        ml += b;
      } while (b == 255);
      if (bad) break;
    }
    ml += 4;
    if (ml > dl - op) { bad = true; break; }
    __syncwarp(gmask);  // literal bytes written by the group are visible to its match reads
    if (moff >= ml && ml <= 2 * kLzG) {
      // no overlap, short match (the common case): two loads per lane, then the stores
      const uint32_t k1 = gl + kLzG;
      const uint32_t v0 = (kLzG <= 4 || gl < ml) ? uint32_t(out[op - moff + gl]) : 0u;  // ml >= 4
      const uint32_t v1 = k1 < ml ? uint32_t(out[op - moff + k1]) : 0u;
      if (kLzG <= 4 || gl < ml) out[op + gl] = uint8_t(v0);
      if (k1 < ml) out[op + k1] = uint8_t(v1);
      __syncwarp(gmask);
    } else if (moff >= ml) {
      // no overlap: the whole match is already written -- issue up to 4 batches of loads, then the stores
      // (one L2 round trip per 4*kLzG bytes instead of one per batch)
      for (uint32_t base = 0; base < ml; base += 4 * kLzG) {
        uint32_t v[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint32_t k = base + j * kLzG + gl;
          v[j] = k < ml ? uint32_t(out[op - moff + k]) : 0u;
        }
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint32_t k = base + j * kLzG + gl;
          if (k < ml) out[op + k] = uint8_t(v[j]);
        }
      }
      __syncwarp(gmask);
    } else if (moff >= kLzG) {
      // overlapping, period >= kLzG: the sources of a batch lie before the batch -> batches in order
      for (uint32_t base = 0; base < ml; base += kLzG) {
        const uint32_t k = base + gl;
        if (k < ml) out[op + k] = out[op - moff + k];
        __syncwarp(gmask);
      }
    } else {  // overlapping short period (moff < kLzG): every source byte lies in [op - moff, op)
      uint32_t m = gl;  // gl mod moff without a division (gl < kLzG <= 16, moff >= 1)
      while (m >= moff) m -= moff;
      uint32_t st = kLzG;  // kLzG mod moff
      while (st >= moff) st -= moff;
      for (uint32_t k = gl; k < ml; k += kLzG) {
        out[op + k] = out[op - moff + m];
        m += st;
        if (m >= moff) m -= moff;
      }
      __syncwarp(gmask);
    }
    op += ml;
    ip = q;
  }
  if (!bad && op != dl) bad = true;
  if (bad && gl == 0) atomicOr(B.err + D.err_idx, 0x4u);
}

// ------------------------------------------------------------------------------------------ thread per sub-chunk
// The paper's Non-Parallel schedule, one thread per chunk, built around the per-sub-chunk
// latency chain: a sub-chunk's sequences decode one after another, so its decode time is
// (sequences) x (latency per sequence), and a launch lasts as long as its slowest sub-chunk.  Per sequence this
// kernel has at most one dependent global round trip (a far match source); everything else is shared memory:
//  * the compressed stream is prefetched 16-byte block by block into a 64-byte per-thread input ring, two
//    blocks ahead in registers (the loads are in flight while earlier sequences decode);
//  * output bytes go to an OR-byte per-thread output ring (128) indexed by global address bits; a completed
//    FB-byte block (32: a whole L2 sector) of the global output leaves the ring with FB / 16 vector stores (byte
//    stores only at the sub-chunk's unaligned head and tail);
//  * a literal run or match moves up to 16 bytes per step; match sources within kLzNear bytes (96) come from the
//    output ring, farther ones from global memory (three 8-byte loads in flight together), where the thread's own
//    earlier 16-byte stores already are (same-thread program order).  An overlapping match (offset < 16)
//    moves `offset` bytes per step, so every source byte precedes the bytes being written.
// A warp instruction advances 32 sub-chunks (vs one per warp for lz4_kernel).
constexpr uint32_t kLzRing = 64;   // input ring bytes per thread

// far-match source loads: L1::evict_first (the window of one thread is re-read at most a few times; measured on
// config 3's l_comment: 4.71 vs 4.84 ms and 20.1 vs 22.0 GB of DRAM reads; .cg / L1::no_allocate: 6.2 / 5.9 ms)
__device__ __forceinline__ uint2 ld_v2_far(const void* p) {
  uint2 v;
  asm volatile("ld.global.L1::evict_first.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
  return v;
}

// OR: output ring bytes per thread, FB: output block bytes (flushed with FB / 16 vector stores once complete)
template <uint32_t OR, uint32_t FB>
__global__ void __launch_bounds__(kWarpsPerCta * 32, 3) lz4_thread_kernel(const __grid_constant__ Lz4Batch B) {
  static_assert((OR == 64 && FB == 16) || (OR == 128 && FB == 32), "ring / block pairs");
  constexpr uint32_t kLzNear = OR == 64 ? 48 : 96;  // match offsets up to this are read from the output ring
  __shared__ __align__(16) uint8_t oring_s[kWarpsPerCta * 32 * OR];
  __shared__ __align__(16) uint8_t iring_s[kWarpsPerCta * 32 * kLzRing];
  const uint32_t gs = blockIdx.x * (kWarpsPerCta * 32) + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31;
  const bool live = gs < B.total_subs;
  const Lz4Desc& D = B.d[find_desc_lz4(B, live ? gs : B.total_subs - 1)];
  const uint32_t s = gs - D.sub0;
  const uint32_t* tab = reinterpret_cast<const uint32_t*>(D.table);
  uint64_t off = 0;
  if (D.uniform) {
    off = uint64_t(s) * D.uniform;
  } else {
    // sum of the preceding sub-chunks' lengths, the warp cooperating on each lane's sum in turn
    const uint32_t act = __ballot_sync(FULL, live);
    for (uint32_t L = 0; L < 32; L++) {
      if (!(act >> L & 1u)) continue;
      const uint32_t sL = __shfl_sync(FULL, s, L);
      const uint64_t tL = __shfl_sync(FULL, reinterpret_cast<uint64_t>(tab), L);
      const uint32_t uL = __shfl_sync(FULL, D.uniform, L);
      uint64_t acc = 0;
      if (!uL)
        for (uint32_t k = lane; k < sL; k += 32) acc += __ldg(reinterpret_cast<const uint32_t*>(tL) + 3 * k + 2);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
      if (lane == L && !uL) off = acc;
    }
  }
  if (!live) return;
  const uint32_t co = __ldg(tab + 3 * s), cl = __ldg(tab + 3 * s + 1), dl = __ldg(tab + 3 * s + 2);
  bool bad = uint64_t(co) + cl > D.payload_bytes || off + dl > D.n;
  if (s + 1 == D.n_sub && off + dl != D.n) bad = true;
  if (bad) {
    atomicOr(B.err + D.err_idx, 0x4u);
    return;
  }
  uint8_t* const oring = oring_s + threadIdx.x * OR;
  uint8_t* const iring = iring_s + threadIdx.x * kLzRing;
  const uint32_t* const orw = reinterpret_cast<const uint32_t*>(oring);
  const uint32_t* const irw = reinterpret_cast<const uint32_t*>(iring);

  // ---- compressed input: global addresses [ia0, ia0 + cl); 16-byte blocks below `ihave` are in the input
  // ring (the last four of them), blocks ihave and ihave + 16 are in flight in nb0 / nb1
  const uintptr_t ia0 = reinterpret_cast<uintptr_t>(D.payload + co);
  // blocks at or past the stream's padded end (16-byte padding + 16 slack bytes) are never loaded
  const uintptr_t istop = (reinterpret_cast<uintptr_t>(D.payload) + D.payload_bytes + 31) & ~uintptr_t(15);
  auto ldblk = [&](uintptr_t a) -> uint4 {
    return a < istop ? __ldg(reinterpret_cast<const uint4*>(a)) : make_uint4(0, 0, 0, 0);
  };
  uintptr_t ihave = ia0 & ~uintptr_t(15);
  uint4 nb0 = ldblk(ihave), nb1 = ldblk(ihave + 16);
  auto ensure = [&](uintptr_t end) {  // input bytes below `end` are in the ring
    while (ihave < end) {
      *reinterpret_cast<uint4*>(iring + (ihave & (kLzRing - 1))) = nb0;
      nb0 = nb1;
      nb1 = ldblk(ihave + 32);
      ihave += 16;
    }
  };
  auto in_u8 = [&](uint32_t p) -> uint32_t { return iring[(ia0 + p) & (kLzRing - 1)]; };
  // 16 ring bytes from global address a (words q..q+4 of a ring of RB bytes, funnel-shifted)
  auto ring16 = [&](const uint32_t* rw, uint32_t rb, uintptr_t a, uint32_t (&v)[4]) {
    const uint32_t q = uint32_t(a >> 2), sh = uint32_t(a & 3u) * 8u;
    uint32_t w[5];
#pragma unroll
    for (int i = 0; i < 5; i++) w[i] = rw[(q + i) & (rb / 4 - 1)];
#pragma unroll
    for (int i = 0; i < 4; i++) v[i] = __funnelshift_r(w[i], w[i + 1], sh);
  };

  // ---- output: global addresses [ga0, ga0 + dl)
  uint8_t* const out = D.out + off;
  const uintptr_t ga0 = reinterpret_cast<uintptr_t>(out), ge = ga0 + dl;
  auto flush = [&](uintptr_t blk) {  // block [blk, blk + FB) leaves the ring (bytes inside [ga0, ge) only)
    const uint8_t* r = oring + (blk & (OR - 1));
    if (blk >= ga0 && blk + FB <= ge) {
#pragma unroll
      for (uint32_t h = 0; h < FB; h += 16) {
        const uint4 v = *reinterpret_cast<const uint4*>(r + h);
        st_v4_u32(reinterpret_cast<void*>(blk + h), v.x, v.y, v.z, v.w);
      }
    } else {
      for (uint32_t b = 0; b < FB; b++)
        if (blk + b >= ga0 && blk + b < ge) reinterpret_cast<uint8_t*>(blk)[b] = r[b];
    }
  };

  // ---- one LZ4 sequence: header fields, parsed in two parts (head: token + literal length; tail: offset +
  // match length), and a match source preloaded from global memory one sequence ahead
  struct Seq {
    uint32_t token, lit, lit_src, ipx, moff, ml;
    bool last, tail, pre;
    uint2 x0, x1, x2;
  };
  auto head = [&](uint32_t ip, Seq& q) -> bool {  // token + literal length at ip
    ensure(ia0 + ip + 32);
    if (ip >= cl) return false;
    q.token = in_u8(ip++);
    uint32_t lit = q.token >> 4;
    if (lit == 15) {
      uint32_t b;
      do {
        if (ip >= cl) return false;
        ensure(ia0 + ip + 1);
        b = in_u8(ip++);
        lit += b;
      } while (b == 255);
    }
    if (lit > cl - ip) return false;
    q.lit = lit;
    q.lit_src = ip;
    q.ipx = ip + lit;
    q.last = q.ipx == cl;  // the last sequence carries literals only
    q.tail = q.pre = false;
    return true;
  };
  auto tail = [&](Seq& q) -> bool {  // offset + match length after the literals
    uint32_t ip = q.ipx;
    if (cl - ip < 2) return false;
    ensure(ia0 + ip + 2);
    q.moff = in_u8(ip) | (in_u8(ip + 1) << 8);
    ip += 2;
    if (q.moff == 0) return false;
    uint32_t ml = q.token & 15;
    if (ml == 15) {
      uint32_t b;
      do {
        if (ip >= cl) return false;
        ensure(ia0 + ip + 1);
        b = in_u8(ip++);
        ml += b;
      } while (b == 255);
    }
    q.ml = ml + 4;
    q.ipx = ip;
    q.tail = true;
    return true;
  };
  // Append k <= 16 bytes (v, little-endian) at output position op: the bytes are shifted into the 8-byte word
  // containing op (its bytes below op are kept from the ring's copy of that word) and whole 8-byte words are
  // stored into the ring (no byte stores); bytes past op + k in the last word are scratch, overwritten by later
  // appends before any read (they alias ring bytes more than OR - 24 behind: flushed, and no near match reads them).
  uint64_t acc = 0;  // the ring word holding output bytes [(ga0 + op) & ~7, ga0 + op)
  auto put16 = [&](uint32_t op, const uint32_t (&v)[4], uint32_t k) {
    const uintptr_t ga = ga0 + op;
    const uint32_t fill = uint32_t(ga & 7u), sh = 8u * fill;
    const uint64_t v01 = (uint64_t(v[1]) << 32) | v[0], v23 = (uint64_t(v[3]) << 32) | v[2];
    const uint64_t keep = fill ? (acc & ((1ull << sh) - 1ull)) : 0ull;
    const uint64_t w0 = keep | (v01 << sh);
    const uint64_t w1 = (fill ? (v01 >> (64u - sh)) : 0ull) | (v23 << sh);
    const uint64_t w2 = fill ? (v23 >> (64u - sh)) : 0ull;
    uint64_t* rw8 = reinterpret_cast<uint64_t*>(oring);
    const uint32_t q = uint32_t(ga >> 3), words = (fill + k + 7u) >> 3;  // words touched: 1..3
    rw8[q & (OR / 8 - 1)] = w0;
    if (words > 1) rw8[(q + 1) & (OR / 8 - 1)] = w1;
    if (words > 2) rw8[(q + 2) & (OR / 8 - 1)] = w2;
    const uint32_t last = (fill + k) >> 3;  // index of the word holding the new end position
    acc = last == 0 ? w0 : last == 1 ? w1 : w2;
    if ((ga & (FB - 1)) + k >= FB) flush(ga & ~uintptr_t(FB - 1));
  };
  // the 8-byte words holding source bytes [src, src + k) (k <= 16): only those are loaded, so a short match does not
  // pull in the next 32 / 64-byte DRAM fetch unit (96 % of the l_comment matches are 4-12 bytes, > 96 bytes back)
  auto far_load = [&](uintptr_t src, uint32_t k, uint2& x0, uint2& x1, uint2& x2) {
    const uintptr_t a8 = src & ~uintptr_t(7);
    const uint32_t e = uint32_t(src & 7u) + k;
    x0 = ld_v2_far(reinterpret_cast<const void*>(a8));
    x1 = e > 8 ? ld_v2_far(reinterpret_cast<const void*>(a8 + 8)) : make_uint2(0u, 0u);
    x2 = e > 16 ? ld_v2_far(reinterpret_cast<const void*>(a8 + 16)) : make_uint2(0u, 0u);
  };
  auto far_words = [&](uintptr_t src, const uint2& x0, const uint2& x1, const uint2& x2, uint32_t (&v)[4]) {
    const bool hi = (src & 4u) != 0;
    const uint32_t sh = uint32_t(src & 3u) * 8u;
    const uint32_t w0 = hi ? x0.y : x0.x, w1 = hi ? x1.x : x0.y, w2 = hi ? x1.y : x1.x, w3 = hi ? x2.x : x1.y,
                   w4 = hi ? x2.y : x2.x;
    v[0] = __funnelshift_r(w0, w1, sh);
    v[1] = __funnelshift_r(w1, w2, sh);
    v[2] = __funnelshift_r(w2, w3, sh);
    v[3] = __funnelshift_r(w3, w4, sh);
  };

  uint32_t op = 0;
  Seq T;
  if (!head(0, T)) bad = true;
  while (!bad) {
    // ---- T's literals, 16 bytes per step from the input ring
    if (T.lit > dl - op) { bad = true; break; }
    for (uint32_t done = 0; done < T.lit;) {
      const uint32_t k = min(16u, T.lit - done);
      ensure(ia0 + T.lit_src + done + 16);
      uint32_t v[4];
      ring16(irw, kLzRing, ia0 + T.lit_src + done, v);
      put16(op, v, k);
      op += k;
      done += k;
    }
    if (T.last) break;
    if (!T.tail && !tail(T)) { bad = true; break; }
    if (T.moff > op || T.ml > dl - op) { bad = true; break; }
    // ---- look ahead: the next sequence's header (short literal runs only, so its literal bytes stay in the
    // input ring) and, for a far match whose first 16 source bytes are already flushed, its source loads --
    // in flight while T's match completes
    Seq N;
    if (!head(T.ipx, N)) { bad = true; break; }
    if (!N.last && N.lit <= 16 && (N.token & 15) != 15) {
      if (!tail(N)) { bad = true; break; }
      const uint32_t opm = op + T.ml + N.lit;  // N's match position
      const uintptr_t flushed = (ga0 + op) & ~uintptr_t(FB - 1);
      const uint32_t kN = min(min(16u, N.ml), N.moff);  // N's first match step
      if (N.moff > kLzNear && N.moff <= opm && ga0 + opm - N.moff + kN <= flushed) {
        far_load(ga0 + opm - N.moff, kN, N.x0, N.x1, N.x2);
        N.pre = true;
      }
    }
    // ---- T's match, up to 16 bytes (at most `moff`) per step
    for (uint32_t done = 0; done < T.ml;) {
      const uint32_t k = min(min(16u, T.ml - done), T.moff);
      const uintptr_t src = ga0 + op - T.moff;
      uint32_t v[4];
      if (T.moff <= kLzNear) {
        ring16(orw, OR, src, v);
      } else if (done == 0 && T.pre) {
        far_words(src, T.x0, T.x1, T.x2, v);
      } else {
        uint2 x0, x1, x2;
        far_load(src, k, x0, x1, x2);
        far_words(src, x0, x1, x2, v);
      }
      put16(op, v, k);
      op += k;
      done += k;
    }
    T = N;
  }
  if (!bad && op != dl) bad = true;
  if (bad) {
    atomicOr(B.err + D.err_idx, 0x4u);
    return;
  }
  if (ge & (FB - 1)) flush(ge & ~uintptr_t(FB - 1));  // the partial last block
}

// ------------------------------------------------------------------------------------------ split parse / copy
// The thread kernel's sub-chunk chain costs ~270 instructions per LZ4 sequence because one thread both parses
// and copies.  This schedule splits the two (knob lz4_split): a warp owns G sub-chunks; per
// round each owner lane (lane < G) parses the next kSplitR sequences of its sub-chunk -- only the header chain
// (token, length extensions, offset), ~20 instructions per sequence -- into a shared record table
// {output position, literal source, literal length, match offset}; then the whole warp copies the G x kSplitR
// sequences 32 at a time, one sequence per lane: all literals first (compressed input -> output), then the
// matches in dependency order (a match whose source overlaps the output of a lower lane's match in the same
// sub-chunk waits for it; sources further back were written in earlier steps).  Output goes straight to
// global memory with aligned word stores (byte stores at a sequence's unaligned edges: lanes write disjoint
// byte ranges); match sources are read back through the SM's L1 after __syncwarp.  G is chosen per launch so
// that the launch has about one wave of warps (few sub-chunks per launch: 2 per warp; many: 32).
constexpr uint32_t kSplitWarps = 4;  // warps per CTA (G = 32: 35 KB of record tables per CTA, 5 CTAs per SM)

// 16 bytes at shared address a (any alignment; the 4 bytes after a + 16 must be readable)
__device__ __forceinline__ void load16s(const uint8_t* a, uint32_t (&v)[4]) {
  const uintptr_t p = reinterpret_cast<uintptr_t>(a);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(p & ~uintptr_t(3));
  const uint32_t sh = uint32_t(p & 3u) * 8u;
  const uint32_t w0 = w[0], w1 = w[1], w2 = w[2], w3 = w[3], w4 = w[4];
  v[0] = __funnelshift_r(w0, w1, sh);
  v[1] = __funnelshift_r(w1, w2, sh);
  v[2] = __funnelshift_r(w2, w3, sh);
  v[3] = __funnelshift_r(w3, w4, sh);
}

// k <= 16 bytes of v to dst: whole aligned words with one 4-byte store, the edge words byte by byte (the
// neighbouring bytes belong to other lanes' sequences)
__device__ __forceinline__ void store16(uint8_t* dst, const uint32_t (&v)[4], uint32_t k) {
  const uintptr_t p = reinterpret_cast<uintptr_t>(dst);
  const int a = int(p & 3u);
  uint32_t* base = reinterpret_cast<uint32_t*>(p & ~uintptr_t(3));
  const uint32_t sh = 8u * uint32_t(a);
  uint32_t u[5];
  u[0] = v[0] << sh;
  u[1] = __funnelshift_l(v[0], v[1], sh);
  u[2] = __funnelshift_l(v[1], v[2], sh);
  u[3] = __funnelshift_l(v[2], v[3], sh);
  u[4] = sh ? (v[3] >> (32u - sh)) : 0u;
#pragma unroll
  for (int i = 0; i < 5; i++) {
    const int lo = 4 * i - a;  // data byte index of the word's first byte
    if (lo >= int(k) || lo + 4 <= 0) continue;
    if (lo >= 0 && lo + 4 <= int(k)) {
      base[i] = u[i];
    } else {
#pragma unroll
      for (int b = 0; b < 4; b++)
        if (lo + b >= 0 && lo + b < int(k)) reinterpret_cast<uint8_t*>(base + i)[b] = uint8_t(u[i] >> (8 * b));
    }
  }
}

template <uint32_t G, uint32_t R, uint32_t F>
__global__ void __launch_bounds__(kSplitWarps * 32, 5) lz4_split_kernel(const __grid_constant__ Lz4Batch B) {
  static_assert(G >= 1 && G <= 8 && (G * R) % 32 == 0, "G sub-chunks per warp, R records each per round");
  static_assert(F % 16 == 0 && (G * F / 16) % 32 == 0, "F refill bytes per sub-chunk: whole 16-byte blocks per lane");
  constexpr uint32_t kRing = 2 * F;           // header ring per sub-chunk (bytes)
  constexpr uint32_t kBlk = G * F / 16 / 32;  // refill blocks per lane per round
  __shared__ __align__(16) uint4 rec_s[kSplitWarps][G][R + 1];
  __shared__ __align__(16) uint8_t ring_s[kSplitWarps][G][kRing];
  __shared__ uint32_t cnt_s[kSplitWarps][G];
  __shared__ __align__(16) uint32_t scr_s[kSplitWarps * 32][8];  // a lane's replicated short match period
  constexpr uint32_t kStg = R >= 32 ? 2048 : 1024;               // staging bytes per step segment
  __shared__ __align__(16) uint8_t stg_s[kSplitWarps][32 / R][kStg + 48];  // 16 guard bytes before, 32 after
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t gs = (blockIdx.x * kSplitWarps + wib) * G + lane;  // owner lanes: lane < G
  const bool live = lane < G && gs < B.total_subs;
  const Lz4Desc& D = B.d[find_desc_lz4(B, live ? gs : B.total_subs - 1)];
  const uint32_t s = gs - D.sub0;
  const uint32_t* tab = reinterpret_cast<const uint32_t*>(D.table);
  uint64_t off = 0;
  if (live && D.uniform) off = uint64_t(s) * D.uniform;
  {
    // non-uniform sub-chunks: the sum of the preceding sub-chunks' lengths, the warp cooperating per owner
    const uint32_t act = __ballot_sync(FULL, live && !D.uniform);
    for (uint32_t L = 0; L < G; L++) {
      if (!(act >> L & 1u)) continue;
      const uint32_t sL = __shfl_sync(FULL, s, L);
      const uint64_t tL = __shfl_sync(FULL, reinterpret_cast<uint64_t>(tab), L);
      uint64_t acc = 0;
      for (uint32_t k = lane; k < sL; k += 32) acc += __ldg(reinterpret_cast<const uint32_t*>(tL) + 3 * k + 2);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
      if (lane == L) off = acc;
    }
  }
  uint32_t co = 0, cl = 0, dl = 0;
  bool bad = false;
  if (live) {
    co = __ldg(tab + 3 * s); cl = __ldg(tab + 3 * s + 1); dl = __ldg(tab + 3 * s + 2);
    bad = uint64_t(co) + cl > D.payload_bytes || off + dl > D.n || (s + 1 == D.n_sub && off + dl != D.n);
  }
  const uint8_t* const in = live ? D.payload + co : D.payload;
  uint8_t* const out = live ? D.out + off : D.out;
  bool done = !live || bad;
  uint4* const rec = rec_s[wib][lane < G ? lane : 0];
  uint8_t* const scr = reinterpret_cast<uint8_t*>(scr_s[threadIdx.x]);
  // The parse reads header bytes (tokens, length extensions, offsets) from a per-sub-chunk shared ring of
  // kRing bytes that the whole warp refills F bytes at a time: the refill loads of round r are issued right
  // after its parse and stored into the ring after its copy phase, so their latency hides behind the copies.
  // Positions u are relative to `abase` (the 16-aligned address at or below the sub-chunk's first byte):
  // the ring holds [fu - kRing, fu) (fu: the loaded frontier, a multiple of 16); blocks at or past the
  // payload's padded end are never loaded.  Literal bytes are not read by the parse.
  const uintptr_t abase = reinterpret_cast<uintptr_t>(in) & ~uintptr_t(15);
  const uint32_t d0 = uint32_t(reinterpret_cast<uintptr_t>(in) & 15u);
  const uintptr_t istop = (reinterpret_cast<uintptr_t>(D.payload) + D.payload_bytes + 31) & ~uintptr_t(15);
  uint8_t* const ring = ring_s[wib][lane < G ? lane : 0];
  uint32_t u = d0, ue = d0 + cl;  // parse position, end of the sub-chunk's input
  uint32_t fu = 0;                // frontier (owner lanes)
  uint32_t op = 0;
  // refill request of each owner: the F bytes at [rq, rq + F) (rq = ~0u: none); the warp loads them
  auto refill_issue = [&](uint32_t rq_own, uint4 (&blk)[kBlk]) {
#pragma unroll
    for (uint32_t i = 0; i < kBlk; i++) {
      const uint32_t g = (i * 32 + lane) / (F / 16), bo = (i * 32 + lane) % (F / 16);
      const uint32_t rq = __shfl_sync(FULL, rq_own, g);
      const uint64_t ab = __shfl_sync(FULL, uint64_t(abase), g);
      const uint64_t stop = __shfl_sync(FULL, uint64_t(istop), g);  // sub-chunk g's payload (its own chunk's)
      const uintptr_t a = uintptr_t(ab) + rq + 16u * bo;
      blk[i] = make_uint4(0u, 0u, 0u, 0u);
      if (rq != ~0u && a + 16 <= stop) blk[i] = __ldg(reinterpret_cast<const uint4*>(a));
    }
  };
  auto refill_store = [&](uint32_t rq_own, const uint4 (&blk)[kBlk]) {
#pragma unroll
    for (uint32_t i = 0; i < kBlk; i++) {
      const uint32_t g = (i * 32 + lane) / (F / 16), bo = (i * 32 + lane) % (F / 16);
      const uint32_t rq = __shfl_sync(FULL, rq_own, g);
      if (rq != ~0u)
        *reinterpret_cast<uint4*>(&ring_s[wib][g][(rq + 16u * bo) & (kRing - 1)]) = blk[i];
    }
  };
  {  // prologue: the first kRing bytes
    uint4 blk[kBlk];
    refill_issue(done ? ~0u : 0u, blk);
    refill_store(done ? ~0u : 0u, blk);
    refill_issue(done ? ~0u : F, blk);
    refill_store(done ? ~0u : F, blk);
    fu = kRing;
    __syncwarp();
  }
  // header byte at position v >= u: from the ring below the frontier, else (a header past a long literal run,
  // rare) straight from global memory
  auto rb = [&](uint32_t v) -> uint32_t {
    return v < fu ? uint32_t(ring[v & (kRing - 1)]) : uint32_t(__ldg(reinterpret_cast<const uint8_t*>(abase + v)));
  };
  for (;;) {
    // ---- parse: up to R sequence headers per owner lane
    uint32_t n = 0;
    if (!done) {
      for (; n < R; n++) {
        // fast path: no length extension, not the last sequence, header bytes inside the ring (the common
        // case: ~25 instructions, one load latency on the chain); everything else takes the general path
        if (u + 17 <= fu && u + 3 <= ue) {
          const uint32_t tok = ring[u & (kRing - 1)];
          const uint32_t lit = tok >> 4, mlc = tok & 15u, v = u + 1 + lit;
          if (lit < 15 && mlc < 15 && v + 2 <= ue) {
            const uint32_t moff = uint32_t(ring[v & (kRing - 1)]) | (uint32_t(ring[(v + 1) & (kRing - 1)]) << 8);
            const uint32_t ml = mlc + 4;
            const bool b = moff == 0 || moff > op + lit || lit + ml > dl - op;
            rec[n] = make_uint4(op, u + 1 - d0, lit, moff);
            op += lit + ml;
            u = v + 2;
            if (b) { bad = true; break; }
            continue;
          }
        }
        if (u >= ue) { bad = true; break; }
        const uint32_t tok = rb(u);
        uint32_t lit = tok >> 4, ml = tok & 15u, v = u + 1;
        if (lit == 15) {
          uint32_t b;
          do {
            if (v >= ue) { bad = true; break; }
            b = rb(v++);
            lit += b;
          } while (b == 255);
          if (bad) break;
        }
        if (lit > ue - v) { bad = true; break; }
        const uint32_t lsrc = v - d0;
        v += lit;
        if (v == ue) {  // the last sequence: literals only
          if (lit > dl - op) { bad = true; break; }
          rec[n] = make_uint4(op, lsrc, lit, 0u);
          op += lit;
          n++;
          u = v;
          done = true;
          if (op != dl) bad = true;
          break;
        }
        if (ue - v < 2) { bad = true; break; }
        const uint32_t moff = rb(v) | (rb(v + 1) << 8);
        v += 2;
        if (ml == 15) {
          uint32_t b;
          do {
            if (v >= ue) { bad = true; break; }
            b = rb(v++);
            ml += b;
          } while (b == 255);
          if (bad) break;
        }
        ml += 4;
        if (lit > dl - op || moff == 0 || moff > op + lit || ml > dl - op - lit) { bad = true; break; }
        rec[n] = make_uint4(op, lsrc, lit, moff);
        op += lit + ml;
        u = v;
      }
      if (bad) { n = 0; done = true; }
      rec[n].x = op;  // the end of the last record
    }
    if (lane < G) cnt_s[wib][lane] = n;
    // refill request: keep at least F bytes ahead of u; a jump past the frontier (a long literal run)
    // restarts the ring at u
    uint32_t rq = ~0u;
    if (!done) {
      if (u + 16 > fu) {
        fu = (u & ~15u);
        rq = fu;
        fu += F;
      } else if (fu - u < F) {
        rq = fu;
        fu += F;
      }
    }
    uint4 blk[kBlk];
    refill_issue(rq, blk);
    __syncwarp();
    if (__ballot_sync(FULL, n > 0 || rq != ~0u) == 0) break;
    // ---- copy: the round's records, 32 at a time (lane -> record flat % R of sub-chunk flat / R).  A step covers
    // all of a sub-chunk's records of the round, i.e. one contiguous output range [S0, S1); when it fits the
    // segment's shared staging buffer, literals and matches are written there (match sources inside the range
    // are read back from shared memory: dependent matches wait ~30 cycles, not an L2 round trip) and the range
    // is flushed to global memory with aligned 16-byte stores; sources before S0 come from global memory.
#pragma unroll 1
    for (uint32_t st = 0; st < G * R / 32; st++) {
      const uint32_t flat = st * 32 + lane, sc = flat / R, k = flat % R;
      const uint8_t* const inj =
          reinterpret_cast<const uint8_t*>(__shfl_sync(FULL, reinterpret_cast<uint64_t>(in), sc));
      uint8_t* const outj = reinterpret_cast<uint8_t*>(__shfl_sync(FULL, reinterpret_cast<uint64_t>(out), sc));
      const uint32_t nsc = cnt_s[wib][sc];
      const bool act = k < nsc;
      uint4 r = make_uint4(0u, 0u, 0u, 0u);
      uint32_t ml = 0;
      if (act) {
        r = rec_s[wib][sc][k];
        ml = rec_s[wib][sc][k + 1].x - r.x - r.z;
      }
      const uint32_t S0 = rec_s[wib][sc][0].x, S1 = rec_s[wib][sc][nsc].x;
      const uintptr_t A0 = reinterpret_cast<uintptr_t>(outj) + S0, A1 = reinterpret_cast<uintptr_t>(outj) + S1;
      const uintptr_t Ab = A0 & ~uintptr_t(15);
      const bool staged = nsc > 0 && A1 - Ab <= kStg;
      uint8_t* const stg = stg_s[wib][lane / R] + 16;
      // destination / source byte at output position x (relative to the sub-chunk)
      auto dstp = [&](uint32_t x) -> uint8_t* {
        return staged ? stg + (reinterpret_cast<uintptr_t>(outj) + x - Ab) : outj + x;
      };
      // kk <= 16 source bytes at output position x: global below S0, staged at or above it
      auto src16 = [&](uint32_t x, uint32_t kk, uint32_t (&v)[4]) {
        if (!staged || x + kk <= S0) {
          load16<false>(outj + x, kk, v);
        } else if (x >= S0) {
          load16s(stg + (reinterpret_cast<uintptr_t>(outj) + x - Ab), v);
        } else {  // straddles S0: the first S0 - x bytes from global memory, the rest staged
          uint32_t g[4], h[4];
          load16<false>(outj + x, S0 - x, g);
          load16s(stg + (A0 - Ab) - (S0 - x), h);  // staged bytes below A0 are never read: merged away
          const uint32_t c = S0 - x;
#pragma unroll
          for (int i = 0; i < 4; i++) {
            const uint32_t lo = 4u * i;
            const uint32_t m = c >= lo + 4 ? 0xFFFFFFFFu : c <= lo ? 0u : (1u << (8u * (c - lo))) - 1u;
            v[i] = (g[i] & m) | (h[i] & ~m);
          }
        }
      };
      // literals (independent of every other write)
      for (uint32_t t = 0; t < r.z; t += 16) {
        const uint32_t kk = min(16u, r.z - t);
        uint32_t v[4];
        load16<true>(inj + r.y + t, kk, v);
        store16(dstp(r.x + t), v, kk);
      }
      __syncwarp();
      // matches, in dependency order within a sub-chunk's lanes
      const uint32_t mpos = r.x + r.z, src = mpos - r.w, se = src + min(ml, r.w);
      const uint32_t segmask = R >= 32 ? FULL : (((1u << R) - 1u) << (lane & ~(R - 1u)));
      bool pend = act && ml > 0;
      uint32_t pm = __ballot_sync(FULL, pend);
      while (pm) {
        const uint32_t mine = pm & segmask;
        const uint32_t lp = mine ? uint32_t(__ffs(mine) - 1) : lane;
        const uint32_t mp_lp = __shfl_sync(FULL, mpos, lp);
        const bool ready = pend && (lp == lane || mp_lp >= se);
        if (ready) {
          if (r.w >= 16 || ml <= r.w) {
            for (uint32_t t = 0; t < ml; t += 16) {
              const uint32_t kk = min(16u, ml - t);
              uint32_t v[4];
              src16(src + t, kk, v);
              store16(dstp(mpos + t), v, kk);
            }
          } else {  // period r.w < 16 shorter than the match: replicate it into 32 scratch bytes
            uint32_t v[4];
            src16(src, r.w, v);
            reinterpret_cast<uint4*>(scr)[0] = make_uint4(v[0], v[1], v[2], v[3]);
            for (uint32_t i = r.w; i < 32; i++) scr[i] = scr[i - r.w];
            const uint32_t* sw = reinterpret_cast<const uint32_t*>(scr);
            const uint32_t s16 = 16u % r.w;
            uint32_t ph = 0;
            for (uint32_t t = 0; t < ml; t += 16) {
              const uint32_t kk = min(16u, ml - t), q = ph >> 2, sh = (ph & 3u) * 8u;
              const uint32_t w0 = sw[q], w1 = sw[q + 1], w2 = sw[q + 2], w3 = sw[q + 3], w4 = sw[min(q + 4, 7u)];
              uint32_t x[4] = {__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh), __funnelshift_r(w2, w3, sh),
                               __funnelshift_r(w3, w4, sh)};
              store16(dstp(mpos + t), x, kk);
              ph += s16;
              if (ph >= r.w) ph -= r.w;
            }
          }
        }
        __syncwarp();
        pend = pend && !ready;
        pm = __ballot_sync(FULL, pend);
      }
      // flush the staged range: whole 16-byte blocks with one vector store, the two edge blocks byte by byte
      if (staged) {
        const uint32_t nb = uint32_t((A1 - Ab + 15) / 16);
        for (uint32_t bi = lane % R; bi < nb; bi += R) {
          const uintptr_t Bk = Ab + 16u * bi;
          const uint8_t* sb = stg + 16u * bi;
          if (Bk >= A0 && Bk + 16 <= A1) {
            const uint4 q = *reinterpret_cast<const uint4*>(sb);
            st_v4_u32(reinterpret_cast<void*>(Bk), q.x, q.y, q.z, q.w);
          } else {
            for (uint32_t j = 0; j < 16; j++)
              if (Bk + j >= A0 && Bk + j < A1) reinterpret_cast<uint8_t*>(Bk)[j] = sb[j];
          }
        }
      }
      __syncwarp();
    }
    refill_store(rq, blk);
    __syncwarp();  // the record table is rewritten next round; the ring refill is visible to the parse
  }
  if (live && bad) atomicOr(B.err + D.err_idx, 0x4u);
}


// ------------------------------------------------------------------------------------------ speculative parse
// Warp per sub-chunk with the header chain parsed in parallel (knob lz4_spec).  A sub-chunk's
// sequences form a chain p -> next(p) through the compressed bytes (next = p + 1 + literal-length extension +
// literals + 2 + match-length extension), so the N.P. decode time is (sequences) x (latency per header).
// Here the compressed stream is cut into 32 word-aligned segments; lane j walks the chain SPECULATIVELY from its
// segment's first byte, marking every position it visits in a shared bitmask.  Chains from a wrong start merge
// with the true one after a few headers (next() is a function, so once two chains share a position they agree),
// so a fix-up pass re-walks each segment from its true entry (the exit of the previous segment's true chain)
// only until it meets a marked position; the few wrong marks before that point are cleared and the true ones set.
// Iterated until no segment's exit changes (lane 0's chain is exact, so this ends after at most 32 rounds; in
// practice 1-2).  The bitmask then holds exactly the true header positions; the copy phase takes them 32 at a time
// in stream order (one sequence per lane: header parse, a warp scan of the output lengths, literals, then matches
// in dependency order as in lz4_split_kernel) into a shared-memory image of the sub-chunk's output, so every
// match source is a shared-memory read, and finished 16-byte blocks leave with one vector store each.
// Sub-chunks of at most kSpecOut decompressed bytes (the launcher falls back to the other schedules otherwise);
// compressed bytes are staged in shared memory when they fit kSpecIn, else read through L1.
constexpr uint32_t kSpecWarps = 4;
constexpr uint32_t kSpecOut = 16384;
constexpr uint32_t kSpecIn = 8192;
constexpr uint32_t kSpecMaxCl = 17408;  // >= the LZ4 bound of kSpecOut bytes
struct SpecSmem {
  uint8_t out[kSpecOut + 16 + 48];   // output image at alignment offset (out & 15), 16-byte blocks
  uint8_t in[kSpecIn + 48];          // compressed bytes at alignment offset (in & 15)
  uint32_t bits[kSpecMaxCl / 32];    // header positions
};
static_assert(sizeof(SpecSmem) % 16 == 0, "per-warp shared layout keeps 16-byte alignment");
constexpr uint32_t kSpecSmem = kSpecWarps * sizeof(SpecSmem);

// position of the r-th (0-based) set bit of x (r < popc(x))
__device__ __forceinline__ uint32_t select_bit(uint32_t x, uint32_t r) {
  uint32_t pos = 0, c;
  c = __popc(x & 0xFFFFu); if (r >= c) { r -= c; pos += 16; x >>= 16; }
  c = __popc(x & 0xFFu);   if (r >= c) { r -= c; pos += 8;  x >>= 8; }
  c = __popc(x & 0xFu);    if (r >= c) { r -= c; pos += 4;  x >>= 4; }
  c = __popc(x & 0x3u);    if (r >= c) { r -= c; pos += 2;  x >>= 2; }
  c = x & 1u;              if (r >= c) { pos += 1; }
  return pos;
}

__global__ void __launch_bounds__(kSpecWarps * 32, 2) lz4_spec_kernel(const __grid_constant__ Lz4Batch B) {
  extern __shared__ __align__(16) uint8_t spec_smem[];
  SpecSmem& S = reinterpret_cast<SpecSmem*>(spec_smem)[threadIdx.x >> 5];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * kSpecWarps;
  for (uint32_t gs = blockIdx.x * kSpecWarps + (threadIdx.x >> 5); gs < B.total_subs; gs += nwarps) {
    const Lz4Desc& D = B.d[find_desc_lz4(B, gs)];
    const uint32_t s = gs - D.sub0;
    const uint32_t* tab = reinterpret_cast<const uint32_t*>(D.table);
    uint64_t off = 0;
    if (D.uniform) {
      off = uint64_t(s) * D.uniform;
    } else {
      for (uint32_t k = lane; k < s; k += 32) off += __ldg(tab + 3 * k + 2);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) off += __shfl_xor_sync(FULL, off, o);
    }
    const uint32_t co = __ldg(tab + 3 * s), cl = __ldg(tab + 3 * s + 1), dl = __ldg(tab + 3 * s + 2);
    if (uint64_t(co) + cl > D.payload_bytes || off + dl > D.n || (s + 1 == D.n_sub && off + dl != D.n) ||
        dl > kSpecOut || cl == 0 || cl > kSpecMaxCl) {
      if (lane == 0) atomicOr(B.err + D.err_idx, 0x4u);
      continue;
    }
    const uint8_t* const in = D.payload + co;
    uint8_t* const out = D.out + off;
    const uint32_t ai = uint32_t(reinterpret_cast<uintptr_t>(in) & 15u);
    const uint32_t ao = uint32_t(reinterpret_cast<uintptr_t>(out) & 15u);
    const bool sin = ai + cl <= kSpecIn;
    const uint32_t nwords = (cl + 31) / 32;
    // ---- stage the compressed bytes (16-byte blocks below the payload's padded end) and clear the bitmask
    if (sin) {
      const uintptr_t ab = reinterpret_cast<uintptr_t>(in) - ai;
      const uintptr_t istop = (reinterpret_cast<uintptr_t>(D.payload) + D.payload_bytes + 31) & ~uintptr_t(15);
      for (uint32_t i = lane; 16 * i < ai + cl; i += 32) {
        const uintptr_t a = ab + 16u * i;
        const uint4 v = a + 16 <= istop ? __ldg(reinterpret_cast<const uint4*>(a)) : make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(S.in + 16 * i) = v;
      }
    }
    for (uint32_t i = lane; i < nwords; i += 32) S.bits[i] = 0u;
    const uint32_t sim = smem_addr(S.out), sinb = smem_addr(S.in) + ai;  // image block 0, input byte 0
    for (uint32_t i = lane; 16 * i < ao + dl; i += 32) sts_v4(sim + 16 * i, make_uint4(0u, 0u, 0u, 0u));
    __syncwarp();
    auto ib = [&](uint32_t p) -> uint32_t { return sin ? lds_u8(sinb + p) : uint32_t(__ldg(in + p)); };
    // next header position after a header at p < cl (cl: the chain ends with a literal-only sequence; cl + 1:
    // the header runs past the end)
    auto nxt = [&](uint32_t p) -> uint32_t {
      const uint32_t t = ib(p);
      uint32_t q = p + 1, lit = t >> 4;
      if (lit == 15) {
        uint32_t b;
        do {
          if (q >= cl) return cl + 1;
          b = ib(q++);
          lit += b;
        } while (b == 255);
      }
      if (lit > cl - q) return cl + 1;
      q += lit;
      if (q == cl) return cl;
      if (cl - q < 2) return cl + 1;
      q += 2;
      if ((t & 15u) == 15u) {
        uint32_t b;
        do {
          if (q >= cl) return cl + 1;
          b = ib(q++);
        } while (b == 255);
      }
      return q;
    };
    auto marked = [&](uint32_t p) -> bool { return (S.bits[p >> 5] >> (p & 31u)) & 1u; };
    // ---- speculative walks: lane j over segment [s0, e)
    const uint32_t L = 32u * ((nwords + 31) / 32);
    const uint32_t s0 = lane * L, e = min(s0 + L, cl);
    const bool seg = s0 < cl;
    uint32_t ex = s0;
    if (seg) {
      uint32_t p = s0, acc = 0;
      while (p < e) {
        acc |= 1u << (p & 31u);
        const uint32_t q = nxt(p);
        if (q >= e || (q >> 5) != (p >> 5)) { S.bits[p >> 5] = acc; acc = 0; }
        p = q;
      }
      ex = p;
    }
    __syncwarp();
    // ---- fix-up: entry = the previous segment's true exit; walk to the first marked position (the merge)
    uint32_t E = ex, entry = s0, mpos = s0, tprev = s0;
    bool walked = false;
    for (int it = 0; it < 33; it++) {
      const uint32_t up = __shfl_up_sync(FULL, E, 1);
      const uint32_t t = lane == 0 ? 0u : up;
      bool changed = false;
      if (seg && (!walked || t != tprev)) {
        uint32_t p = t;
        while (p < e && !marked(p)) p = nxt(p);
        const uint32_t nE = p < e ? ex : p;
        entry = t;
        mpos = p < e ? p : e;
        changed = nE != E;
        E = nE;
        tprev = t;
        walked = true;
      }
      if (!__any_sync(FULL, changed)) break;
    }
    // ---- the bitmask becomes the true chain: clear [s0, mpos), set the re-walked headers [entry, mpos)
    if (seg && mpos != s0) {
      const uint32_t wlo = s0 >> 5, wm = mpos >> 5;
      for (uint32_t w = wlo; w < wm; w++) S.bits[w] = 0u;
      if (mpos < e) S.bits[wm] &= ~((1u << (mpos & 31u)) - 1u);
      else if (e & 31u) S.bits[wm] = 0u;  // no merge, segment ends inside a word (e == cl): that word is ours
      for (uint32_t p = entry; p < mpos; p = nxt(p)) S.bits[p >> 5] |= 1u << (p & 31u);
    }
    __syncwarp();
    // ---- copy: headers 32 at a time in stream order into the shared output image
    const uint32_t img = sim + ao;  // shared address of output byte 0
    const uintptr_t obase = reinterpret_cast<uintptr_t>(out) - ao;
    auto flush = [&](uint32_t b) {  // image block b -> global (bytes of [ao, ao + dl) only)
      const uintptr_t g = obase + 16u * b;
      const uint4 q = lds_v4(sim + 16u * b);
      if (16u * b >= ao && 16u * b + 16u <= ao + dl) {
        st_v4_u32(reinterpret_cast<void*>(g), q.x, q.y, q.z, q.w);
      } else {
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
        for (uint32_t j = 0; j < 16; j++)
          if (16u * b + j >= ao && 16u * b + j < ao + dl) reinterpret_cast<uint8_t*>(g)[j] = uint8_t(w[j >> 2] >> (8 * (j & 3)));
      }
    };
    uint32_t P = 0, op0 = 0, fb = 0;
    bool bad = false, ended = false;
    for (;;) {
      const uint32_t w0 = P >> 5, wi = w0 + lane;
      uint32_t word = wi < nwords ? S.bits[wi] : 0u;
      if (lane == 0) word &= ~0u << (P & 31u);
      const uint32_t c = __popc(word);
      uint32_t C = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(FULL, C, o);
        if (lane >= uint32_t(o)) C += v;
      }
      const uint32_t total = __shfl_sync(FULL, C, 31);
      if (total == 0) {
        if (w0 + 32 >= nwords) break;
        P = 32u * (w0 + 32);
        continue;
      }
      if (ended) { bad = true; break; }  // headers after the literal-only last sequence
      const uint32_t n = min(total, 32u);
      // lane k < n takes the k-th header: the word i with C[i-1] <= k < C[i]
      uint32_t i = 0;
#pragma unroll
      for (uint32_t b = 16; b > 0; b >>= 1) {
        const uint32_t Ci = __shfl_sync(FULL, C, i + b - 1);
        if (Ci <= lane) i += b;
      }
      i = min(i, 31u);
      const uint32_t wd = __shfl_sync(FULL, word, i), below = __shfl_sync(FULL, C - c, i);
      const bool act = lane < n;
      const uint32_t hp = 32u * (w0 + i) + select_bit(wd, act ? lane - below : 0u);
      P = __shfl_sync(FULL, hp, n - 1) + 1;
      // header
      uint32_t lit = 0, ml = 0, moff = 0, lsrc = 0;
      bool b = false, last = false;
      if (act) {
        const uint32_t t = ib(hp);
        uint32_t q = hp + 1;
        lit = t >> 4;
        if (lit == 15) {
          uint32_t x;
          do {
            if (q >= cl) { b = true; break; }
            x = ib(q++);
            lit += x;
          } while (x == 255);
        }
        if (!b && lit > cl - q) b = true;
        if (!b) {
          lsrc = q;
          q += lit;
          if (q == cl) {
            last = true;
          } else if (cl - q < 2) {
            b = true;
          } else {
            moff = ib(q) | (ib(q + 1) << 8);
            q += 2;
            ml = t & 15u;
            if (ml == 15) {
              uint32_t x;
              do {
                if (q >= cl) { b = true; break; }
                x = ib(q++);
                ml += x;
              } while (x == 255);
            }
            ml += 4;
          }
        }
      }
      // output positions: exclusive scan of the sequences' lengths
      const uint32_t len = b ? 0u : lit + ml;
      uint32_t incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(FULL, incl, o);
        if (lane >= uint32_t(o)) incl += v;
      }
      const uint32_t x = op0 + incl - len;
      if (act && !b) {
        if (uint64_t(x) + lit + ml > dl) b = true;
        if (!last && (moff == 0 || moff > x + lit)) b = true;
        if (last && lane != n - 1) b = true;
      }
      if (__any_sync(FULL, b)) { bad = true; break; }
      ended = __any_sync(FULL, act && last);
      op0 += __shfl_sync(FULL, incl, 31);
      // literals
      if (act) {
        for (uint32_t t = 0; t < lit; t += 16) {
          const uint32_t kk = min(16u, lit - t);
          uint32_t v[4];
          if (sin) sload16(sinb + lsrc + t, v);
          else load16<true>(in + lsrc + t, kk, v);
          sstore16(img + x + t, v, kk);
        }
      }
      __syncwarp();
      // matches in dependency order: ready when the source lies below the lowest pending match
      const uint32_t mp = x + lit, src = mp - moff, se = src + min(ml, moff);
      bool pend = act && ml > 0;
      uint32_t pm = __ballot_sync(FULL, pend);
      while (pm) {
        const uint32_t lp = uint32_t(__ffs(pm) - 1);
        const uint32_t mp_lp = __shfl_sync(FULL, mp, lp);
        const bool ready = pend && (lp == lane || mp_lp >= se);
        if (ready) {
          if (moff >= 16 || ml <= moff) {
            for (uint32_t t = 0; t < ml; t += 16) {
              uint32_t v[4];
              sload16(img + src + t, v);
              sstore16(img + mp + t, v, min(16u, ml - t));
            }
          } else {  // short period: copy from a distance d (a multiple of moff) that grows as the run is written
            uint32_t d = moff;
            for (uint32_t t = 0; t < ml;) {
              const uint32_t kk = min(min(16u, ml - t), d);
              uint32_t v[4];
              sload16(img + mp + t - d, v);
              sstore16(img + mp + t, v, kk);
              t += kk;
              while (d <= t) d += moff;
            }
          }
        }
        __syncwarp();
        pend = pend && !ready;
        pm = __ballot_sync(FULL, pend);
      }
      // finished 16-byte blocks of the image leave with one vector store each
      const uint32_t fe = (ao + op0) >> 4;
      for (uint32_t bk = fb + lane; bk < fe; bk += 32) flush(bk);
      fb = fe;
    }
    if (!bad && (!ended || op0 != dl)) bad = true;
    if (!bad) {
      const uint32_t fe = (ao + dl + 15) >> 4;
      for (uint32_t bk = fb + lane; bk < fe; bk += 32) flush(bk);
    } else if (lane == 0) {
      atomicOr(B.err + D.err_idx, 0x4u);
    }
    __syncwarp();
  }
}

}  // namespace

cudaError_t launch_lz4(const Lz4Batch& b, uint32_t max_sub, uint32_t max_csub, cudaStream_t s) {
  if (!b.total_subs) return cudaSuccess;
  // lz4_spec: the speculative-parse warp-per-sub-chunk kernel (every sub-chunk must fit its shared-memory output
  // image; persistent warps, sub-chunks strided over them).  1 (default) = for launches of at most two of its
  // waves, where its short per-sub-chunk chain wins (one 16 KiB sub-chunk: 0.19 ms vs 0.45 split / 1.41 thread);
  // bigger launches are throughput-bound and it issues ~40 % more instructions per sequence at 8 warps per SM
  // (config 3's l_comment: 13.0 ms vs 5.45 ms for the thread kernel); 2 = always, 0 = never.
  const int spec = tune_get(TUNE_LZ4_SPEC);
  if (spec && max_sub <= kSpecOut && max_csub <= kSpecMaxCl) {
    static int occ[kMaxDevices] = {};
    const int dev = current_device();
    if (!occ[dev]) {
      cudaFuncSetAttribute(lz4_spec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSpecSmem));
      cudaFuncSetAttribute(lz4_spec_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[dev], lz4_spec_kernel, kSpecWarps * 32, kSpecSmem);
      if (occ[dev] < 1) occ[dev] = 1;
    }
    const uint32_t slots = uint32_t(device_sms() * occ[dev]) * kSpecWarps;
    if (spec == 2 || b.total_subs <= 2 * slots) {
      const uint32_t need = (b.total_subs + kSpecWarps - 1) / kSpecWarps;
      const uint32_t grid = std::min<uint32_t>(need, slots / kSpecWarps);
      lz4_spec_kernel<<<grid, kSpecWarps * 32, kSpecSmem, s>>>(b);
      return cudaGetLastError();
    }
  }
  // H8 schedule (NEXT-3 knobs): lz4_split = 1 (default) takes the split parse/copy kernel for latency-bound
  // launches -- up to ~4 sub-chunks per resident warp slot, G = the smallest sub-chunks per warp that fits one
  // wave -- and the lz4_lanes schedule for bigger, throughput-bound ones, where the thread kernel issues fewer
  // instructions per sequence (measured: one 7 K-sub-chunk chunk 1.12 vs 3.85 ms; 112 K sub-chunks 9.1 vs 5.4
  // ms); lz4_split_g > 0 forces the split kernel with that G.
  if (tune_get(TUNE_LZ4_SPLIT)) {
    static int occ[kMaxDevices] = {};
    const int dev = current_device();
    if (!occ[dev]) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[dev], lz4_split_kernel<2, 16, 256>, kSplitWarps * 32, 0);
      if (occ[dev] < 1) occ[dev] = 1;
    }
    const uint32_t wave = uint32_t(device_sms()) * uint32_t(occ[dev]) * kSplitWarps;
    uint32_t g = uint32_t(tune_get(TUNE_LZ4_SPLIT_G));
    if (!g) {
      g = 1;
      while (g < 4 && uint64_t(g) * wave < b.total_subs) g *= 2;
      if (uint64_t(g) * wave < b.total_subs) g = 0;
    }
    if (g) {
      const uint32_t per_cta = kSplitWarps * g, grid = (b.total_subs + per_cta - 1) / per_cta;
      switch (g) {
        case 1: lz4_split_kernel<1, 32, 512><<<grid, kSplitWarps * 32, 0, s>>>(b); break;
        case 2: lz4_split_kernel<2, 16, 256><<<grid, kSplitWarps * 32, 0, s>>>(b); break;
        case 4: lz4_split_kernel<4, 16, 256><<<grid, kSplitWarps * 32, 0, s>>>(b); break;
        default: lz4_split_kernel<8, 16, 256><<<grid, kSplitWarps * 32, 0, s>>>(b); break;
      }
      return cudaGetLastError();
    }
  }
  // lanes per sub-chunk (knob lz4_lanes, env CDM_LZ4_G): 1 = the paper's thread per chunk (P:329,
  // lz4_thread_kernel), 2/4/8/16 = lane groups, 32 = one warp per sub-chunk
  const int G = tune_get(TUNE_LZ4_LANES);
  if (G == 1) {
    const uint32_t grid = (b.total_subs + kWarpsPerCta * 32 - 1) / (kWarpsPerCta * 32);
    // 128-byte output rings flushed in 32-byte (whole-sector) blocks: config 3's l_comment 5.36 -> 4.87 ms vs
    // 64-byte rings / 16-byte blocks (more matches served from the ring: offsets <= 96 instead of <= 48)
    lz4_thread_kernel<128, 32><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
    return cudaGetLastError();
  }
  if (G != 32) {
    const uint32_t per_cta = kWarpsPerCta * 32 / G;
    const uint32_t grid = (b.total_subs + per_cta - 1) / per_cta;
    if (G == 4) lz4_group_kernel<4, 1><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
    else if (G == 2) lz4_group_kernel<2, 1><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
    else if (G == 16) lz4_group_kernel<16, 1><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
    else lz4_group_kernel<8, 1><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
    return cudaGetLastError();
  }
  const uint32_t grid = (b.total_subs + kWarpsPerCta - 1) / kWarpsPerCta;
  lz4_kernel<<<grid, kWarpsPerCta * 32, 0, s>>>(b);
  return cudaGetLastError();
}

}  // namespace cdm
