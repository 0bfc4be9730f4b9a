// kernels_fpc.cu -- H5 for CHAR(n) rows: the fused Dict|BitPack decode of fixed-width text columns
// (PAPER.md:237-240 Fully-Parallel dictionary example; reading R14: CHAR(n) = space-padded n-byte rows).
//
//   out[i*E .. i*E+E) = dict[(FOR + bits[i*w, i*w+w)) * E .. +E)
//
// E-byte rows (E not 4 or 8) do not map onto whole words per row, so the byte assembly is organised around
// row groups that do: a thread owns G = P/E consecutive rows whose P bytes are P/4 whole 32-bit words, P a
// multiple of lcm(4, E) near 60 B with an odd word count (E = 25: 4 rows = 25 words; E = 10 and 3: 6 / 20
// rows = 15 words; E = 1, 2: P = 16).  With E a template parameter every row's byte position inside the
// group is a compile-time constant, so a row costs one field extraction from the group's 64-bit index
// window, ceil((E+3)/4)+1 dictionary word loads (read at the row's byte alignment with one funnel shift per
// word; E <= 2: one byte / halfword gather) and one OR per word into registers -- no data-dependent loops.
// The words of a warp's 32 groups are transposed through shared memory (odd word strides: conflict-free) so
// the warp writes its contiguous 32*P-byte region with 16-byte stores, 512 contiguous bytes per store
// instruction.  Small dictionaries (the TPC-H flags, modes, priorities: <= 100 B) are read from shared
// memory, large ones (o_clerk: ~1.5 MB per chunk) through the read-only path.  Persistent CTAs walk
// contiguous ranges of (tile, pass) units of 256*G rows.  Widths without an instantiation use fp_kernel's generic byte path.
#include <cstdlib>

#include "device_util.cuh"
#include "kernels.h"

namespace cdm {
namespace {

using namespace dev;

constexpr int lcm4(int e) { return e % 4 == 0 ? e : (e % 2 == 0 ? 2 * e : 4 * e); }

// P = bytes per thread group: a multiple of lcm(4, E) of ~60 bytes with an odd word count (conflict-free
// shared-memory transposition: lanes write at word stride NW); E <= 2: P = 16 (adjacent 16-byte stores)
constexpr int char_p(int e) {
  return e <= 2 ? 16 : lcm4(e) >= 48 ? lcm4(e) : lcm4(e) * ((60 / lcm4(e)) | 1);
}

template <int E>
struct CharShape {
  static constexpr int P = char_p(E);          // bytes per thread group
  static constexpr int G = P / E;              // rows per thread group
  static constexpr int NW = P / 4;             // words per thread group
  static constexpr bool DIRECT = P == 16;      // lanes' groups are adjacent 16-byte stores
  static constexpr int RP = kThreads * G;      // rows per CTA pass (a work unit; a tile's last unit may be short)
  static constexpr int UPT = (kFpTile + RP - 1) / RP;  // units per tile
  static_assert(P % E == 0 && P % 4 == 0 && (DIRECT || NW % 2 == 1), "row group shape");
};

constexpr uint32_t kCharDictSmem = 16384;  // dictionaries up to this many bytes are staged in shared memory

__device__ __forceinline__ int find_desc_fpc(const FpBatch& B, uint32_t tile) {
  int lo = 0, hi = int(B.n) - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (B.d[mid].tile0 <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ uint4 lds128(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_addr(p)));
  return v;
}

// Pre-shifted dictionaries (PRE): for the few-entry dictionaries of the TPC-H CHAR(n) columns (modes, priorities,
// instructions: 4-7 entries) the shared copy holds every entry at each of the 4 byte alignments a row can start
// at inside its group, zero-padded to PB = 16 / 32 bytes: table[s][idx] = the entry's bytes at byte offset s.
// A row then costs one or two 16-byte shared loads and an OR per word (no funnel shifts, no edge masks).
template <int E>
struct PreShape {
  static constexpr int PB = E + 3 <= 16 ? 16 : 32;      // padded bytes per shifted entry
  static constexpr int MAXE = kCharDictSmem / (4 * PB);  // entries that fit the shared table
};

// DSM: every dictionary of the launch fits kCharDictSmem and is read from shared memory; PRE (implies DSM):
// every dictionary has at most PreShape<E>::MAXE entries and is read from the pre-shifted table
template <int E, bool DSM, bool PRE>
__global__ void __launch_bounds__(kThreads) fpc_kernel(const __grid_constant__ FpBatch B, uint32_t total_units) {
  using S = CharShape<E>;
  constexpr int NW = S::NW, G = S::G;
  constexpr int PB = PreShape<E>::PB;
  // shared: [DSM: 4 guard words + dictionary words + 4 guard words] [!DIRECT: 8 warps x 32 groups x NW words]
  extern __shared__ __align__(16) uint32_t sm[];
  constexpr uint32_t kDictWords = DSM ? kCharDictSmem / 4 + 8 : 0;
  uint32_t* const dict_s = sm;
  uint32_t* const stage = sm + kDictWords;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int staged_di = -1;

  // a contiguous range of units per CTA: the chunk (and its staged dictionary) changes rarely
  const uint32_t upc = (total_units + gridDim.x - 1) / gridDim.x;
  const uint32_t u_end = min(total_units, (blockIdx.x + 1) * upc);
  int dcur = -1;  // the CTA's units increase: the descriptor moves forward from one search
  for (uint32_t u = blockIdx.x * upc; u < u_end; u++) {
    const uint32_t tile = u / S::UPT, pass = u % S::UPT;
    if (dcur < 0) dcur = find_desc_fpc(B, tile);
    while (dcur + 1 < int(B.n) && B.d[dcur + 1].tile0 <= tile) dcur++;
    const int di = dcur;
    const FpDesc& D = B.d[di];
    const uint32_t lt = tile - D.tile0;
    const uint64_t tile_start = uint64_t(lt) * kFpTile;
    const uint32_t valid = uint32_t(min(uint64_t(kFpTile), uint64_t(D.n) - tile_start));
    const uint32_t r0 = pass * S::RP;  // the unit's first row in the tile
    if (r0 >= valid) continue;         // CTA-uniform
    const uint32_t w = D.w, entries = D.entries;
    const uint64_t base = D.base;
    const uint64_t lim = base < entries ? entries - base : 0ull;  // field f is a valid index iff f < lim
    const uint32_t base32 = uint32_t(base);
    const uint32_t m32 = w >= 32 ? 0xFFFFFFFFu : (1u << w) - 1u;
    if (DSM && di != staged_di) {  // CTA-uniform: stage this chunk's dictionary (guard words stay zero)
      __syncthreads();             // nobody still reads the previous dictionary
      if (PRE) {  // table word (s, idx, m): bytes 4m..4m+3 of entry idx placed at byte offset s
        const uint32_t per_s = entries * (PB / 4), nwords = 4 * per_s;
        for (uint32_t q = tid; q < nwords; q += kThreads) {
          const uint32_t sft = q / per_s, r = q % per_s, idx = r / (PB / 4), m = r % (PB / 4);
          uint32_t x = 0;
#pragma unroll
          for (int b = 0; b < 4; b++) {
            const int src = int(4 * m + b) - int(sft);
            if (src >= 0 && src < E) x |= uint32_t(__ldg(D.dict + size_t(idx) * E + src)) << (8 * b);
          }
          dict_s[q] = x;
        }
      } else {
        const uint32_t nwords = (entries * uint32_t(E) + 3) / 4;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(D.dict);
        for (uint32_t q = tid; q < nwords + 8; q += kThreads)
          dict_s[q] = (q >= 4 && q - 4 < nwords) ? __ldg(src + (q - 4)) : 0u;
      }
      __syncthreads();
      staged_di = di;
    }
    const uint32_t* wd = reinterpret_cast<const uint32_t*>(D.packed + uint64_t(lt) * (kFpTile / 8) * w);
    const uint32_t* dg = reinterpret_cast<const uint32_t*>(D.dict);
    auto dword = [&](int64_t q) -> uint32_t {  // dictionary word q (q >= -1; guard/slack words beyond)
      return DSM ? dict_s[q + 4] : __ldg(dg + q);
    };

    const uint32_t g0 = r0 + tid * G;  // this thread's first row (tile-local)
    // the group's G fields: one 64-bit window when G*w <= 64 (w <= 32: a valid index has < 2^32 entries)
    const bool win = uint32_t(G) * w <= 64u;
    uint64_t wv = 0;
    if (win && g0 < valid) {  // (a group past the tile's rows reads nothing: its rows are never stored)
      const uint32_t b = g0 * w, q = b >> 5, sh = b & 31;
      const uint32_t a0 = __ldg(wd + q), a1 = __ldg(wd + q + 1), a2 = __ldg(wd + q + 2);
      wv = (uint64_t(__funnelshift_r(a1, a2, sh)) << 32) | __funnelshift_r(a0, a1, sh);
    }
    uint32_t word[NW];
#pragma unroll
    for (int m = 0; m < NW; m++) word[m] = 0u;
    bool bad = false;
#pragma unroll
    for (int j = 0; j < G; j++) {
      const uint32_t r = g0 + j;
      uint64_t f;
      if (win) {
        f = uint32_t(wv >> (j * w)) & m32;
      } else if (r >= valid) {
        f = 0;
      } else if (w <= 32) {
        const uint32_t b = r * w;
        f = __funnelshift_r(__ldg(wd + (b >> 5)), __ldg(wd + (b >> 5) + 1), b & 31) & m32;
      } else {
        f = extract_bits_global(wd, uint64_t(r) * w, w);
      }
      const bool ok = f < lim;
      bad |= !ok && r < valid;
      const uint32_t idx = ok ? base32 + uint32_t(f) : 0u;
      if (E <= 2) {  // whole entries into one word: a byte / halfword gather and a shift
        uint32_t x;
        if (E == 1) x = DSM ? reinterpret_cast<const uint8_t*>(dict_s + 4)[idx] : __ldg(D.dict + idx);
        else x = DSM ? reinterpret_cast<const uint16_t*>(dict_s + 4)[idx]
                     : __ldg(reinterpret_cast<const uint16_t*>(D.dict) + idx);
        word[(j * E) >> 2] |= x << (8 * ((j * E) & 3));
        continue;
      }
      // row j occupies group bytes [j*E, j*E + E): words q0..q1, starting at byte s of word q0
      const int s = (j * E) & 3, q0 = (j * E) >> 2, q1 = (j * E + E - 1) >> 2;
      if (PRE) {  // the entry pre-shifted to byte s: whole words, zero outside the row
        const uint32_t* t = dict_s + (uint32_t(s) * entries + idx) * (PB / 4);
#pragma unroll
        for (int h = 0; h < PB / 16; h++) {
          if (4 * h > q1 - q0) break;
          const uint4 x = lds128(t + 4 * h);
          const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int m = 0; m < 4; m++)
            if (4 * h + m <= q1 - q0) word[q0 + 4 * h + m] |= xw[m];
        }
        continue;
      }
      const int64_t a = int64_t(idx) * E - s;  // dictionary byte that lands on group byte 4*q0
      const int64_t aw = a >> 2;                // >= -1 (guard word)
      const uint32_t sh = uint32_t(a) & 3u;
      // large dictionaries (read through L1: the row kernel is L1-wavefront bound there): the words aw .. aw +
      // q1 - q0 + 1 arrive as whole 16-byte chunks (one L1 wavefront per chunk instead of per word); word aw + m
      // is W[r0 + m], picked with selects.  Chunks are 16-byte aligned inside the dictionary stream's padding.
      constexpr int NCHM = ((E + 2) / 4 + 4) / 4 + 1;
      uint32_t W[4 * NCHM];
      const uint32_t r0 = uint32_t(aw & 3);
      if (!DSM) {
        const uint4* dg4 = reinterpret_cast<const uint4*>(D.dict) + (aw >> 2);
        const uint32_t nch = (r0 + uint32_t(q1 - q0) + 1) / 4 + 1;
#pragma unroll
        for (int c = 0; c < NCHM; c++) {
          const uint4 x = uint32_t(c) < nch ? __ldg(dg4 + c) : make_uint4(0u, 0u, 0u, 0u);
          W[4 * c] = x.x; W[4 * c + 1] = x.y; W[4 * c + 2] = x.z; W[4 * c + 3] = x.w;
        }
      }
      auto rword = [&](int m) -> uint32_t {  // dictionary word aw + m
        if (DSM) return dword(aw + m);
        return r0 == 0 ? W[m] : r0 == 1 ? W[m + 1] : r0 == 2 ? W[m + 2] : W[m + 3];
      };
      uint32_t prev = rword(0);
#pragma unroll
      for (int m = 0; m <= q1 - q0; m++) {
        const uint32_t nxt = rword(m + 1);
        uint32_t x = __funnelshift_r(prev, nxt, 8 * sh);
        prev = nxt;
        if (m == 0 && s) x &= 0xFFFFFFFFu << (8 * s);
        const int e = j * E + E - 4 * (q0 + m);  // row bytes left from this word on
        if (e < 4) x &= (1u << (8 * e)) - 1u;
        word[q0 + m] |= x;
      }
    }
    if (bad) atomicOr(B.err + D.err_idx, 0x1u);

    uint8_t* const obase = static_cast<uint8_t*>(D.out) + tile_start * E;
    const uint32_t limit = valid * E;  // tile payload bytes
    if (S::DIRECT) {
      const uint32_t p0 = g0 * E;
      if (p0 + 16 <= limit) {
        st_v4_u32(obase + p0, word[0], word[1 % NW], word[2 % NW], word[3 % NW]);
      } else if (p0 < limit) {
#pragma unroll
        for (uint32_t b = 0; b < 16; b++)
          if (p0 + b < limit) obase[p0 + b] = uint8_t(word[(b >> 2) % NW] >> (8 * (b & 3)));
      }
    } else {
      uint32_t* const ws = stage + warp * (32 * NW);
      __syncwarp();  // the warp's previous copy-out has read the stage
#pragma unroll
      for (int m = 0; m < NW; m++) ws[lane * NW + m] = word[m];
      __syncwarp();
      const uint32_t rb = (r0 + warp * 32 * G) * E;  // the warp's region in the tile's payload
      if (rb < limit) {
        const uint32_t rl = min(uint32_t(32 * S::P), limit - rb);
#pragma unroll 4
        for (uint32_t c = lane; c < uint32_t(2 * S::P); c += 32) {
          const uint32_t off = c * 16;
          if (off + 16 <= rl) {
            const uint4 v = lds128(ws + off / 4);
            st_v4_u32(obase + rb + off, v.x, v.y, v.z, v.w);
          } else if (off < rl) {
            const uint8_t* sb = reinterpret_cast<const uint8_t*>(ws) + off;
            for (uint32_t b = 0; off + b < rl; b++) obase[rb + off + b] = sb[b];
          }
        }
      }
    }
  }
}

template <int E>
cudaError_t launch_fpc_e(const FpBatch& b, cudaStream_t s) {
  using S = CharShape<E>;
  bool dsm = true, pre = E > 2;
  for (uint32_t i = 0; i < b.n; i++) {
    dsm = dsm && uint64_t(b.d[i].entries) * E <= kCharDictSmem;
    pre = pre && b.d[i].entries <= uint32_t(PreShape<E>::MAXE);
  }
  static const bool no_pre = std::getenv("CDM_FPC_PRE") && std::getenv("CDM_FPC_PRE")[0] == '0';
  pre = pre && !no_pre;
  const uint32_t smem = (dsm ? (kCharDictSmem + 32) : 0) + (S::DIRECT ? 0 : 8 * 32 * S::NW * 4);
  auto kern = pre ? fpc_kernel<E, true, true> : dsm ? fpc_kernel<E, true, false> : fpc_kernel<E, false, false>;
  static bool configured[kMaxDevices][3] = {};
  bool& conf = configured[current_device()][pre ? 2 : dsm];
  if (!conf) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    conf = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const uint32_t units = b.total_tiles * S::UPT;
  uint32_t grid = uint32_t(device_sms() * per_sm);
  if (grid > units) grid = units;
  kern<<<grid, kThreads, smem, s>>>(b, units);
  return cudaGetLastError();
}

}  // namespace

bool fpc_supported(uint32_t E) { return E == 1 || E == 2 || E == 10 || E == 15 || E == 25; }

cudaError_t launch_fpc(const FpBatch& b, uint32_t E, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  switch (E) {
    case 1: return launch_fpc_e<1>(b, s);
    case 2: return launch_fpc_e<2>(b, s);
    case 10: return launch_fpc_e<10>(b, s);
    case 15: return launch_fpc_e<15>(b, s);
    case 25: return launch_fpc_e<25>(b, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cdm
