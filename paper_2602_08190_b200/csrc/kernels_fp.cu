// kernels_fp.cu -- H5: element-parallel ("Fully-Parallel") fused decode.
//
//   out[i] = MAP( FOR + bits[i*w, i*w+w) )           MAP in { cast, dict[.], (double)(.)/10^d }
//
// The paper fuses consecutive Fully-Parallel kernels (bit-unpack + dictionary / Float2Int,
// PAPER.md:277, Eq. 2) so the plain-size intermediate never touches HBM.  B200 shape
// (DESIGN.md "H5"): persistent CTAs (grid = SMs x resident CTAs) walk 4096-value tiles; the tile's
// packed bytes (512*w B, 16-aligned by construction) are staged into shared memory by the TMA engine
// (cp.async.bulk + mbarrier), double-buffered so tile k+1 streams in while tile k is unpacked; each
// thread unpacks 4 consecutive values per group with funnel shifts and writes them with one 16-byte
// store (int32 / f32) or two (int64 / f64), so a warp writes 512 or 1024 contiguous bytes per group.
#include <cstdlib>

#include "device_util.cuh"
#include "kernels.h"

namespace cdm {
namespace {

using namespace dev;

__constant__ double kPow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                  1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};

__device__ __forceinline__ int find_desc_fp(const FpBatch& B, uint32_t tile) {
  int lo = 0, hi = int(B.n) - 1;
  while (lo < hi) {  // last desc with tile0 <= tile
    const int mid = (lo + hi + 1) >> 1;
    if (B.d[mid].tile0 <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ uint32_t stage_bytes(const FpDesc& D, uint32_t lt) {
  const uint64_t stream_bytes = ((uint64_t(D.n) * D.w + 7) / 8 + 15) & ~15ull;  // padded extent
  const uint64_t start = uint64_t(lt) * (kFpTile / 8) * D.w;
  const uint64_t want = uint64_t(kFpTile / 8) * D.w;
  const uint64_t have = stream_bytes > start ? stream_bytes - start : 0;
  return uint32_t(want < have ? want : have);
}

constexpr uint32_t kDictSmemBytes = 8192;  // dictionaries up to this size are gathered from shared memory

// Dictionaries up to kDictSmemBytes are gathered from shared memory (copied there when the tile's chunk
// changes), larger ones through the read-only L1 path; the tile's packed bytes are staged in shared memory by
// the TMA engine, double-buffered across the tiles of a persistent CTA.
__global__ void __launch_bounds__(kThreads, 4) fp_kernel(const __grid_constant__ FpBatch B, uint32_t stage_bytes_alloc) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ __align__(16) uint64_t dict_s[kDictSmemBytes / 8];
  int staged_di = -1;
  const uint32_t tid = threadIdx.x;
  // stage_bytes_alloc: set by the host from the batch's largest w; dynamic smem = 2 stages

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  uint32_t tile = blockIdx.x;
  // a CTA's tiles increase, so the descriptor of the current / next tile only moves forward from one search
  int dcur = tile < B.total_tiles ? find_desc_fp(B, tile) : 0, dnext = dcur;
  auto advance = [&](int d, uint32_t t) {
    while (d + 1 < int(B.n) && B.d[d + 1].tile0 <= t) d++;
    return d;
  };
  // prologue: stage the first tile
  if (tid == 0 && tile < B.total_tiles) {
    const int di = dcur;
    const FpDesc& D = B.d[di];
    const uint32_t lt = tile - D.tile0;
    const uint32_t nb = stage_bytes(D, lt);
    mbar_arrive_expect_tx(&bar[0], nb);
    if (nb) tma_load_1d(smem, D.packed + uint64_t(lt) * (kFpTile / 8) * D.w, nb, &bar[0]);
  }
  for (uint32_t it = 0; tile < B.total_tiles; it++, tile += gridDim.x) {
    const uint32_t s = it & 1;
    const uint32_t next = tile + gridDim.x;
    if (tid == 0 && next < B.total_tiles) {  // stage s^1 was released by the __syncthreads ending it-1
      dnext = advance(dnext, next);
      const int dn = dnext;
      const FpDesc& Dn = B.d[dn];
      const uint32_t ltn = next - Dn.tile0;
      const uint32_t nb = stage_bytes(Dn, ltn);
      fence_proxy_async();  // generic reads of stage s^1 (iteration it-1) precede the TMA refill
      mbar_arrive_expect_tx(&bar[s ^ 1], nb);
      if (nb) tma_load_1d(smem + (s ^ 1) * stage_bytes_alloc, Dn.packed + uint64_t(ltn) * (kFpTile / 8) * Dn.w, nb,
                          &bar[s ^ 1]);
    }
    dcur = advance(dcur, tile);
    const int di = dcur;
    const FpDesc& D = B.d[di];
    // descriptor fields in registers (param-space reads with a dynamic index cost a load per use)
    const uint32_t lt = tile - D.tile0;
    const uint32_t w = D.w, mode = D.mode, ob = D.out_bytes, entries = D.entries;
    const uint64_t base = D.base;
    const uint8_t* const dict8 = D.dict;
    uint8_t* const out8 = reinterpret_cast<uint8_t*>(D.out);
    mbar_wait(&bar[s], (it >> 1) & 1);
    const uint32_t* wd = reinterpret_cast<const uint32_t*>(smem + s * stage_bytes_alloc);
    const uint64_t tile_start = uint64_t(lt) * kFpTile;
    const uint32_t valid = uint32_t(min(uint64_t(kFpTile), uint64_t(D.n) - tile_start));
    bool bad_index = false;
    const bool pair_map = B.pair_map;
    const bool bytes_path = mode == FP_DICT && ob != 4 && ob != 8;  // CHAR(n) rows
    const bool dsm = mode == FP_DICT && !bytes_path && entries * ob <= kDictSmemBytes;
    const bool dsmb = bytes_path && uint64_t(entries) * ob + 8 <= kDictSmemBytes;
    if ((dsm || dsmb) && di != staged_di) {  // uniform: every thread passed the barrier ending the previous tile
      const uint4* src = reinterpret_cast<const uint4*>(dict8);
      for (uint32_t q = tid; q < (entries * ob + 15) / 16; q += kThreads) reinterpret_cast<uint4*>(dict_s)[q] = __ldg(src + q);
      __syncthreads();
      staged_di = di;
    }
    // width class: the 4 consecutive fields of a thread lie in one 32-bit window (w <= 8) or one 64-bit
    // window (w <= 16); wider fields are extracted one by one
    const uint32_t cls = w <= 8 ? 0u : w <= 16 ? 1u : w <= 32 ? 2u : 3u;
    const uint32_t m32 = w >= 32 ? 0xFFFFFFFFu : (1u << w) - 1u;
    // dictionary index limits: field f is valid iff f < lim (base >= entries: none is)
    const uint64_t lim = base < entries ? entries - base : 0ull;
    const uint32_t base32 = uint32_t(base);

#pragma unroll 1
    for (uint32_t k = 0; k < kFpTile / 1024 && !bytes_path; k++) {
      if (ob == 8 && pair_map) {
        // 8-byte rows: lane l of warp u takes the pairs (pa, pa+1) and (pa+64, pa+65), pa = 128u + 2l, so each
        // 16-byte store instruction of a warp covers 512 contiguous bytes (whole sectors)
        if (k * 1024 >= valid) break;
        const uint32_t pa = k * 1024 + (tid >> 5) * 128 + 2 * (tid & 31);
        const uint32_t q[4] = {pa, pa + 1, pa + 64, pa + 65};
        uint64_t v[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint32_t bj = q[j] * w;
          v[j] = w <= 32 ? base + (__funnelshift_r(wd[bj >> 5], wd[(bj >> 5) + 1], bj & 31) & m32)
                         : base + extract_bits(wd, uint64_t(q[j]) * w, w);
        }
        uint64_t r[4];
        if (mode == FP_INT) {
#pragma unroll
          for (int j = 0; j < 4; j++) r[j] = v[j];
        } else if (mode == FP_DICT) {
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const uint64_t f = v[j] - base;
            const bool ok = f < lim;
            bad_index |= !ok && q[j] < valid;
            const uint32_t idx = ok ? base32 + uint32_t(f) : 0u;
            r[j] = dsm ? dict_s[idx] : __ldg(reinterpret_cast<const uint64_t*>(dict8) + idx);
          }
        } else {
          const double p = kPow10[D.d];
#pragma unroll
          for (int j = 0; j < 4; j++) r[j] = __double_as_longlong(double(int64_t(v[j])) / p);
        }
        uint64_t* o = reinterpret_cast<uint64_t*>(out8) + tile_start;
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const uint32_t e = q[2 * h];
          if (e + 1 < valid) st_v2_u64(o + e, r[2 * h], r[2 * h + 1]);
          else if (e < valid) o[e] = r[2 * h];
        }
        continue;
      }
      const uint32_t i0 = k * 1024 + tid * 4;  // 4 consecutive values
      if (i0 >= valid) break;
      uint64_t v[4];
      const uint32_t b0 = i0 * w, wi = b0 >> 5, sh = b0 & 31;
      if (cls == 0) {
        const uint32_t x = __funnelshift_r(wd[wi], wd[wi + 1], sh);
#pragma unroll
        for (int j = 0; j < 4; j++) v[j] = base + ((x >> (j * w)) & m32);
      } else if (cls == 1) {
        const uint32_t a0 = wd[wi], a1 = wd[wi + 1], a2 = wd[wi + 2];
        const uint64_t x = (uint64_t(__funnelshift_r(a1, a2, sh)) << 32) | __funnelshift_r(a0, a1, sh);
#pragma unroll
        for (int j = 0; j < 4; j++) v[j] = base + (uint32_t(x >> (j * w)) & m32);
      } else if (cls == 2) {
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint32_t bj = b0 + j * w;
          v[j] = base + (__funnelshift_r(wd[bj >> 5], wd[(bj >> 5) + 1], bj & 31) & m32);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; j++) v[j] = base + extract_bits(wd, uint64_t(i0 + j) * w, w);
      }
      const uint64_t gi = tile_start + i0;
      const bool full = i0 + 4 <= valid;
      if (mode == FP_INT) {
        if (ob == 4) {
          uint32_t* o = reinterpret_cast<uint32_t*>(out8) + gi;
          if (full) st_v4_u32(o, uint32_t(v[0]), uint32_t(v[1]), uint32_t(v[2]), uint32_t(v[3]));
          else _Pragma("unroll") for (uint32_t j = 0; j < 4; j++) if (i0 + j < valid) o[j] = uint32_t(v[j]);
        } else if (ob == 8) {
          uint64_t* o = reinterpret_cast<uint64_t*>(out8) + gi;
          if (full) { st_v2_u64(o, v[0], v[1]); st_v2_u64(o + 2, v[2], v[3]); }
          else _Pragma("unroll") for (uint32_t j = 0; j < 4; j++) if (i0 + j < valid) o[j] = v[j];
        } else if (ob == 2) {
          uint16_t* o = reinterpret_cast<uint16_t*>(out8) + gi;
          _Pragma("unroll") for (uint32_t j = 0; j < 4; j++) if (i0 + j < valid) o[j] = uint16_t(v[j]);
        } else {
          uint8_t* o = out8 + gi;
          if (full) *reinterpret_cast<uint32_t*>(o) = (v[0] & 0xFF) | ((v[1] & 0xFF) << 8) | ((v[2] & 0xFF) << 16) | ((v[3] & 0xFF) << 24);
          else _Pragma("unroll") for (uint32_t j = 0; j < 4; j++) if (i0 + j < valid) o[j] = uint8_t(v[j]);
        }
      } else if (mode == FP_DICT) {
        // index = base + field, valid iff field < lim = entries - base (all 32-bit: w <= 32 here, and a
        // dictionary has < 2^32 entries); an invalid index raises the error bit and reads entry 0
        uint32_t idx[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint64_t f = v[j] - base;
          const bool ok = f < lim;
          // fields past the tile's last row decode stale staging bytes: never an error, never stored
          bad_index |= !ok && i0 + j < valid;
          idx[j] = ok ? base32 + uint32_t(f) : 0u;
        }
        if (dsm && ob == 8) {
          uint64_t* o = reinterpret_cast<uint64_t*>(out8) + gi;
          if (full) {
            st_v2_u64(o, dict_s[idx[0]], dict_s[idx[1]]);
            st_v2_u64(o + 2, dict_s[idx[2]], dict_s[idx[3]]);
          } else _Pragma("unroll") for (uint32_t j = 0; j < 4; j++) if (i0 + j < valid) o[j] = dict_s[idx[j]];
        } else if (dsm) {
          const uint32_t* d32 = reinterpret_cast<const uint32_t*>(dict_s);
          uint32_t* o = reinterpret_cast<uint32_t*>(out8) + gi;
          if (full) st_v4_u32(o, d32[idx[0]], d32[idx[1]], d32[idx[2]], d32[idx[3]]);
          else _Pragma("unroll") for (uint32_t j = 0; j < 4; j++) if (i0 + j < valid) o[j] = d32[idx[j]];
        } else if (ob == 8) {
          const uint64_t* dict = reinterpret_cast<const uint64_t*>(dict8);
          uint64_t* o = reinterpret_cast<uint64_t*>(out8) + gi;
          if (full) {
            st_v2_u64(o, __ldg(dict + idx[0]), __ldg(dict + idx[1]));
            st_v2_u64(o + 2, __ldg(dict + idx[2]), __ldg(dict + idx[3]));
          } else _Pragma("unroll") for (uint32_t j = 0; j < 4; j++) if (i0 + j < valid) o[j] = __ldg(dict + idx[j]);
        } else if (ob == 4) {
          const uint32_t* dict = reinterpret_cast<const uint32_t*>(dict8);
          uint32_t* o = reinterpret_cast<uint32_t*>(out8) + gi;
          if (full) st_v4_u32(o, __ldg(dict + idx[0]), __ldg(dict + idx[1]), __ldg(dict + idx[2]), __ldg(dict + idx[3]));
          else _Pragma("unroll") for (uint32_t j = 0; j < 4; j++) if (i0 + j < valid) o[j] = __ldg(dict + idx[j]);
        }
      } else {  // FP_F2I: one IEEE division per element (no reciprocal: bit-exact, R13)
        const double p = kPow10[D.d];
        double f[4];
#pragma unroll
        for (int j = 0; j < 4; j++) f[j] = double(int64_t(v[j])) / p;
        uint64_t* o = reinterpret_cast<uint64_t*>(out8) + gi;
        if (full) {
          st_v2_u64(o, __double_as_longlong(f[0]), __double_as_longlong(f[1]));
          st_v2_u64(o + 2, __double_as_longlong(f[2]), __double_as_longlong(f[3]));
        } else _Pragma("unroll") for (uint32_t j = 0; j < 4; j++) if (i0 + j < valid) o[j] = __double_as_longlong(f[j]);
      }
    }
    if (bytes_path) {
      // FP_DICT with E-byte rows (CHAR(n), E not 4/8): the tile's output (valid*E bytes, 16-aligned since
      // 4096*E is a multiple of 16) is produced as 16-byte chunks of four 32-bit words; each word is
      // assembled from <= 4 pieces, a piece = the bytes of one row's entry starting at column col read with
      // one unaligned 4-byte funnel read from the dictionary (shared memory when it fits, else L1/L2); a
      // row's index is extracted only when the row changes.
      const uint32_t E = ob;
      const uint32_t total = valid * E;
      uint8_t* obase = out8 + tile_start * E;
      auto fetch = [&](uint32_t row) -> uint32_t {
        const uint64_t f = w ? extract_bits(wd, uint64_t(row) * w, w) : 0ull;
        if (f >= lim) { bad_index = true; return 0u; }
        return base32 + uint32_t(f);
      };
      const uint32_t* dws = reinterpret_cast<const uint32_t*>(dict_s);
      const uint32_t* dwg = reinterpret_cast<const uint32_t*>(dict8);
      auto rd4 = [&](uint32_t off) -> uint32_t {  // dictionary bytes [off, off + 4), any alignment
        const uint32_t q = off >> 2, sh = (off & 3) * 8;
        const uint32_t lo = dsmb ? dws[q] : __ldg(dwg + q), hi = dsmb ? dws[q + 1] : __ldg(dwg + q + 1);
        return __funnelshift_r(lo, hi, sh);
      };
      for (uint32_t c = tid; c * 16 < total; c += kThreads) {
        const uint32_t p0 = c * 16;
        uint32_t row = p0 / E, col = p0 - row * E;
        uint32_t idx = fetch(row);
        uint32_t word[4];
#pragma unroll
        for (uint32_t j = 0; j < 4; j++) {
          uint32_t acc = 0, filled = 0;
          while (filled < 4 && p0 + 4 * j + filled < total) {
            const uint32_t take = min(4u - filled, E - col);
            const uint32_t v = rd4(idx * E + col);
            const uint32_t m = take >= 4 ? 0xFFFFFFFFu : (1u << (8 * take)) - 1u;
            acc |= (v & m) << (8 * filled);
            filled += take;
            col += take;
            if (col == E) {
              col = 0;
              row++;
              if (row < valid) idx = fetch(row);
            }
          }
          word[j] = acc;
        }
        if (p0 + 16 <= total) {
          st_v4_u32(obase + p0, word[0], word[1], word[2], word[3]);
        } else {
#pragma unroll
          for (uint32_t b = 0; b < 16; b++)
            if (p0 + b < total) obase[p0 + b] = uint8_t(word[b >> 2] >> (8 * (b & 3)));
        }
      }
    }
    if (bad_index) atomicOr(B.err + D.err_idx, 0x1u);
    __syncthreads();  // everyone is done with stage s before it is refilled
  }
}

}  // namespace

namespace {
int g_tune[kTuneKnobs];
bool g_tune_init = false;
void tune_init() {
  if (g_tune_init) return;
  g_tune[TUNE_FP_CTAS_PER_SM] = std::getenv("CDM_FP_CTAS_PER_SM") ? std::atoi(std::getenv("CDM_FP_CTAS_PER_SM")) : 0;
  g_tune[TUNE_LZ4_LANES] = std::getenv("CDM_LZ4_G") ? std::atoi(std::getenv("CDM_LZ4_G")) : 1;
  g_tune[TUNE_SCAN_MODE] = std::getenv("CDM_SCAN_MODE") ? std::atoi(std::getenv("CDM_SCAN_MODE")) : 2;
  g_tune[TUNE_GP_CTAS_PER_SM] = 0;
  g_tune[TUNE_LZ4_SPLIT] = std::getenv("CDM_LZ4_SPLIT") ? std::atoi(std::getenv("CDM_LZ4_SPLIT")) : 1;
  g_tune[TUNE_LZ4_SPLIT_G] = std::getenv("CDM_LZ4_SPLIT_G") ? std::atoi(std::getenv("CDM_LZ4_SPLIT_G")) : 0;
  g_tune[TUNE_LZ4_SPEC] = std::getenv("CDM_LZ4_SPEC") ? std::atoi(std::getenv("CDM_LZ4_SPEC")) : 1;
  g_tune_init = true;
}
}  // namespace

int tune_get(int knob) {
  tune_init();
  return knob >= 0 && knob < kTuneKnobs ? g_tune[knob] : 0;
}

void tune_set(int knob, int value) {
  tune_init();
  if (knob >= 0 && knob < kTuneKnobs) g_tune[knob] = value;
}

int device_sms() {
  static int sms[kMaxDevices] = {};
  const int dev = current_device();
  if (!sms[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev] = v > 0 ? v : 148;
  }
  return sms[dev];
}

cudaError_t launch_fp(const FpBatch& b, uint32_t max_w, cudaStream_t s) {
  if (!b.total_tiles) return cudaSuccess;
  {  // CHAR(n) dictionary rows of one width: the row-group kernel
    bool chr = b.n > 0;
    const uint32_t E = b.n ? b.d[0].out_bytes : 0;
    for (uint32_t i = 0; i < b.n && chr; i++) chr = b.d[i].mode == FP_DICT && b.d[i].out_bytes == E;
    static const bool generic = std::getenv("CDM_FPC") && std::getenv("CDM_FPC")[0] == '0';
    if (chr && E != 4 && E != 8 && fpc_supported(E) && !generic) return launch_fpc(b, E, s);
  }
  const uint32_t stage = ((kFpTile / 8) * (max_w ? max_w : 1) + 16 + 127) & ~127u;  // + slack words for extraction
  const uint32_t smem = 2 * stage;
  auto kern = fp_kernel;
  static uint32_t configured[kMaxDevices] = {};
  uint32_t& conf = configured[current_device()];
  if (smem > 40 * 1024 && smem > conf) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    conf = smem;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  // persistent CTAs per SM: 2 for short batches (each CTA still walks ~5 tiles with its TMA double buffer
  // full, and SM slots stay free for a concurrent RLE chain: config 2), up to 4 for long ones (more tiles in
  // flight per SM: E2 widths at 268 MB, +20 %); the tuning knob (env CDM_FP_CTAS_PER_SM) overrides
  const int cap_env = tune_get(TUNE_FP_CTAS_PER_SM);
  const uint32_t tiles_per_sm = b.total_tiles / uint32_t(device_sms());
  const int cap = cap_env > 0 ? cap_env : tiles_per_sm >= 32 ? 4 : tiles_per_sm >= 20 ? 3 : 2;
  if (cap < per_sm) per_sm = cap;
  uint32_t grid = uint32_t(device_sms() * per_sm);
  // CDM_FP_GRID=tiles: one CTA per tile (no persistence), so CTAs of a concurrent higher-priority family
  // are scheduled as soon as any FP CTA retires
  static const bool per_tile = std::getenv("CDM_FP_GRID") && std::getenv("CDM_FP_GRID")[0] == 't';
  if (per_tile || grid > b.total_tiles) grid = b.total_tiles;
  // default: 4 consecutive values per thread (8-byte rows: two 16-byte stores 32 bytes apart per lane);
  // CDM_FP_PAIR=1: pair-interleaved lanes (whole-sector store instructions) -- measured: E7 l_quantity
  // 0.127 -> 0.104 ms but l_extendedprice 0.118 -> 0.125 ms and config 2 2695 -> 2601 GB/s, so off
  static const bool pair = std::getenv("CDM_FP_PAIR") && std::getenv("CDM_FP_PAIR")[0] == '1';
  if (b.pair_map != uint32_t(pair)) {
    FpBatch c = b;
    c.pair_map = pair;
    kern<<<grid, kThreads, smem, s>>>(c, stage);
  } else {
    kern<<<grid, kThreads, smem, s>>>(b, stage);
  }
  return cudaGetLastError();
}

}  // namespace cdm
