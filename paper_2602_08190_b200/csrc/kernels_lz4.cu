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

// ------------------------------------------------------------------------------------------ smem decoder
// Sub-chunks of <= kLz4SmemMax decompressed bytes are decoded into a per-warp shared-memory window: match
// sources are then shared-memory reads instead of L2 round trips.  Each sequence is parsed from one
// coalesced 32-byte window of the compressed stream held across the lanes (token, literals, offset
// fetched with shuffles); long literal runs / extension bytes fall back to broadcast loads.  The finished
// window is copied out with 16-byte stores: it is placed at byte offset (dst & 15) inside its buffer so
// shared and global addresses share their alignment.
constexpr uint32_t kLz4SmemMax = 32768;

__device__ __forceinline__ uint32_t ldb(const uint8_t* __restrict__ p) { return __ldg(p); }

// A two-window reader over the compressed stream held across the warp's lanes: bytes [pos, pos+64) live in
// (cur, nxt), one byte per lane each, and the window after them is already in flight (pre), so the next
// sequence's bytes are usually a shuffle away.
struct Lz4Reader {
  const uint8_t* __restrict__ in;
  uint32_t cl, pos;
  uint32_t cur, nxt, pre;
  __device__ __forceinline__ uint32_t load(uint32_t q, uint32_t lane) const {
    return (q + lane < cl) ? uint32_t(__ldg(in + q + lane)) : 0u;
  }
  __device__ __forceinline__ void init(const uint8_t* p, uint32_t n, uint32_t lane) {
    in = p; cl = n; pos = 0;
    cur = load(0, lane); nxt = load(32, lane); pre = load(64, lane);
  }
  // make q < pos + 32 (q's byte and the 32 after it are resident)
  __device__ __forceinline__ void advance(uint32_t q, uint32_t lane) {
    while (q >= pos + 32) {
      cur = nxt; nxt = pre; pos += 32;
      pre = load(pos + 64, lane);
    }
  }
  // byte at q (uniform across lanes), q in [pos, pos + 64)
  __device__ __forceinline__ uint32_t at(uint32_t q) const {
    const uint32_t d = q - pos;
    const uint32_t a = __shfl_sync(FULL, cur, d & 31), b = __shfl_sync(FULL, nxt, d & 31);
    return d < 32 ? a : b;
  }
  // per-lane byte at q + lane (q + 31 < pos + 64)
  __device__ __forceinline__ uint32_t lane_at(uint32_t q, uint32_t lane) const {
    const uint32_t d = q + lane - pos;
    const uint32_t a = __shfl_sync(FULL, cur, d & 31), b = __shfl_sync(FULL, nxt, d & 31);
    return d < 32 ? a : b;
  }
};

__global__ void lz4_smem_kernel(const __grid_constant__ Lz4Batch B, uint32_t cap) {
  extern __shared__ __align__(16) uint8_t lzbuf[];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const uint32_t gs = blockIdx.x * wpc + wib;
  if (gs >= B.total_subs) return;
  const Lz4Desc& D = B.d[find_desc_lz4(B, gs)];
  const uint32_t s = gs - D.sub0;
  const uint32_t* tab = reinterpret_cast<const uint32_t*>(D.table);
  uint64_t off = 0;
  if (D.uniform) {
    off = uint64_t(s) * D.uniform;  // host-verified uniform sub-chunk sizes
  } else {
    for (uint32_t k = lane; k < s; k += 32) off += __ldg(tab + 3 * k + 2);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) off += __shfl_xor_sync(FULL, off, o);
  }
  const uint32_t co = __ldg(tab + 3 * s), cl = __ldg(tab + 3 * s + 1), dl = __ldg(tab + 3 * s + 2);
  bool bad = uint64_t(co) + cl > D.payload_bytes || off + dl > D.n || dl > cap;
  if (s + 1 == D.n_sub && off + dl != D.n) bad = true;
  if (bad) {
    if (lane == 0) atomicOr(B.err + D.err_idx, 0x4u);
    return;
  }
  uint8_t* gdst = D.out + off;
  const uint32_t mis = uint32_t(reinterpret_cast<uintptr_t>(gdst) & 15);
  uint8_t* win = lzbuf + wib * (cap + 16) + mis;
  Lz4Reader R;
  R.init(D.payload + co, cl, lane);
  uint32_t ip = 0, op = 0;
  for (;;) {
    if (ip >= cl) { bad = true; break; }
    R.advance(ip, lane);
    const uint32_t token = R.at(ip);
    uint32_t lit = token >> 4;
    ip++;
    if (lit == 15) {
      uint32_t b;
      do {
        if (ip >= cl) { bad = true; break; }
        R.advance(ip, lane);
        b = R.at(ip++);
        lit += b;
      } while (b == 255);
      if (bad) break;
    }
    if (lit > cl - ip || lit > dl - op) { bad = true; break; }
    // literals: 32 per step, from the reader's windows
    for (uint32_t k = 0; k < lit; k += 32) {
      R.advance(ip + k, lane);
      const uint32_t v = R.lane_at(ip + k, lane);
      if (k + lane < lit) win[op + k + lane] = uint8_t(v);
    }
    ip += lit;
    op += lit;
    if (ip == cl) break;  // the last sequence carries literals only
    if (cl - ip < 2) { bad = true; break; }
    R.advance(ip, lane);
    const uint32_t moff = R.at(ip) | (R.at(ip + 1) << 8);
    ip += 2;
    if (moff == 0 || moff > op) { bad = true; break; }
    uint32_t ml = token & 15;
    if (ml == 15) {
      uint32_t b;
      do {
        if (ip >= cl) { bad = true; break; }
        R.advance(ip, lane);
        b = R.at(ip++);
        ml += b;
      } while (b == 255);
      if (bad) break;
    }
    ml += 4;
    if (ml > dl - op) { bad = true; break; }
    __syncwarp();  // literal bytes written by other lanes are visible to the match copy
    if (moff >= 32 || moff >= ml) {
      for (uint32_t base = 0; base < ml; base += 32) {
        const uint32_t k = base + lane;
        if (k < ml) win[op + k] = win[op - moff + k];
        __syncwarp();
      }
    } else {  // period moff < 32 and overlapping: out[op+k] = out[op - moff + (k mod moff)]
      uint32_t m = lane % moff;
      const uint32_t step = 32 % moff;
      for (uint32_t base = 0; base < ml; base += 32) {
        const uint32_t k = base + lane;
        if (k < ml) win[op + k] = win[op - moff + m];
        m += step;
        if (m >= moff) m -= moff;
      }
      __syncwarp();
    }
    op += ml;
  }
  if (!bad && op != dl) bad = true;
  if (bad) {
    if (lane == 0) atomicOr(B.err + D.err_idx, 0x4u);
    return;
  }
  __syncwarp();
  // copy-out: unaligned head bytes, 16-byte body, tail bytes
  const uint32_t head = min(dl, (16u - mis) & 15u);
  if (lane < head) gdst[lane] = win[lane];
  const uint32_t body = (dl - head) & ~15u;
  for (uint32_t o = head + lane * 16; o < head + body; o += 32 * 16) {
    const uint4 v = *reinterpret_cast<const uint4*>(win + o);
    st_v4_u32(gdst + o, v.x, v.y, v.z, v.w);
  }
  const uint32_t t = head + body + lane;
  if (t < dl) gdst[t] = win[t];
}

}  // namespace

cudaError_t launch_lz4(const Lz4Batch& b, uint32_t max_sub, cudaStream_t s) {
  if (!b.total_subs) return cudaSuccess;
  // The shared-memory variant is opt-in (CDM_LZ4_SMEM=1): measured on config 3 (16 KiB sub-chunks) it is
  // 2.5x slower than the global-memory kernel (12 vs 64 resident warps per SM; both are issue-bound).
  static const bool use_smem = std::getenv("CDM_LZ4_SMEM") != nullptr;
  if (max_sub <= kLz4SmemMax && use_smem) {
    // warps per CTA such that 3 CTAs fit an SM's shared memory
    const uint32_t cap = (max_sub + 15) & ~15u;
    uint32_t wpc = 8;
    while (wpc > 1 && 3ull * wpc * (cap + 16) > 220 * 1024) wpc >>= 1;
    const uint32_t smem = wpc * (cap + 16);
    static uint32_t configured[kMaxDevices] = {};
    uint32_t& conf = configured[current_device()];
    if (smem > 48 * 1024 && smem > conf) {
      cudaFuncSetAttribute(lz4_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      conf = smem;
    }
    const uint32_t grid = (b.total_subs + wpc - 1) / wpc;
    lz4_smem_kernel<<<grid, wpc * 32, smem, s>>>(b, cap);
    return cudaGetLastError();
  }
  // lane groups of G lanes per sub-chunk (default 4: 8 sub-chunks per warp; G = 1 is the paper's thread per
  // chunk); G = 32 is one warp per
  // sub-chunk (tuning knob TUNE_LZ4_LANES; env CDM_LZ4_G / CDM_LZ4_WARP)
  const int G = tune_get(TUNE_LZ4_LANES);
  if (G != 32) {
    const uint32_t per_cta = kWarpsPerCta * 32 / G;
    const uint32_t grid = (b.total_subs + per_cta - 1) / per_cta;
    // window bytes per lane: 1 (default) or 4 (CDM_LZ4_WIN=4: a 16-byte window per 4-lane group -- measured
    // 10.0 vs 9.5 ms on config 3's l_comment: the sequence chain is not bound by its compressed-byte loads)
    static const bool win1 = !(std::getenv("CDM_LZ4_WIN") && std::getenv("CDM_LZ4_WIN")[0] == '4');
    if (win1) {
      if (G == 4) lz4_group_kernel<4, 1><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
      else if (G == 1) lz4_group_kernel<1, 1><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
      else if (G == 2) lz4_group_kernel<2, 1><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
      else if (G == 16) lz4_group_kernel<16, 1><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
      else lz4_group_kernel<8, 1><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
    } else {
      if (G == 4) lz4_group_kernel<4, 4><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
      else if (G == 1) lz4_group_kernel<1, 4><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
      else if (G == 2) lz4_group_kernel<2, 4><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
      else if (G == 16) lz4_group_kernel<16, 4><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
      else lz4_group_kernel<8, 4><<<grid, kWarpsPerCta * 32, 0, s>>>(b);
    }
    return cudaGetLastError();
  }
  const uint32_t grid = (b.total_subs + kWarpsPerCta - 1) / kWarpsPerCta;
  lz4_kernel<<<grid, kWarpsPerCta * 32, 0, s>>>(b);
  return cudaGetLastError();
}

}  // namespace cdm
