// kernels.h -- device descriptors + host launch wrappers of the sm_100a decode kernels.
//
// Every kernel decodes a BATCH of chunks that share a kernel family in one launch: descriptors are
// passed by value as __grid_constant__ parameters (no descriptor upload), tiles of all chunks are
// enumerated globally (desc.tile0 = first global tile of the chunk).
#pragma once
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

namespace cdm {

constexpr int kMaxBatch = 32;      // descriptors per launch (more chunks -> more launches)
constexpr int kFpTile = 8192;      // H5 values per tile = 256 threads x 32
constexpr int kScanTile = 4096;    // H6 values per tile = 256 threads x 16
constexpr int kRleTile = 1024;     // H7 runs per tile = 256 threads x 4
constexpr uint32_t kRleSegRows = 32768;  // rle_kernel: output rows per run-start bitmap segment
constexpr uint32_t kRleBigLimit = 1u << 18;  // a tile with more output rows is expanded by rle_big (a CTA
                                              // expands up to 8 bitmap segments itself)
constexpr uint32_t kRleBigPiece = 8192;       // rows per rle_big work item
constexpr int kThreads = 256;

// ---------------------------------------------------------------- H5: element-parallel fused decode
enum FpMode : uint8_t { FP_INT = 0, FP_DICT = 1, FP_F2I = 2 };

struct FpDesc {
  const uint8_t* packed;  // bit-packed stream (16-aligned, padded)
  const uint8_t* dict;    // FP_DICT: dictionary, entries * out_bytes bytes
  void* out;              // decoded output, n * out_bytes
  uint64_t base;          // FOR base
  uint32_t n;             // elements
  uint32_t entries;       // FP_DICT entries
  uint32_t tile0;         // first global tile
  uint32_t err_idx;       // index of this chunk's error word
  uint16_t w;             // bit width 0..64
  uint16_t out_bytes;     // output element bytes
  uint8_t mode;           // FpMode
  uint8_t d;              // FP_F2I decimal exponent
  uint8_t pad[6];
};

// FP launches take up to kMaxFpBatch chunks (a 16 KB __grid_constant__ parameter): fewer persistent launches, fewer
// drain tails between them
constexpr int kMaxFpBatch = 256;
struct FpBatch {
  uint32_t n;
  uint32_t total_tiles;
  uint32_t pair_map;      // 8-byte rows: pair-interleaved lane mapping (set by launch_fp)
  uint32_t* err;          // per-chunk error words
  FpDesc d[kMaxFpBatch];
};
static_assert(sizeof(FpBatch) <= 32000, "kernel parameter limit");

// ---------------------------------------------------------------- H6: scan-dependent delta / offsets
enum ScanMode : uint8_t { SCAN_DELTA = 0, SCAN_OFFSETS = 1 };

struct ScanDesc {
  const uint8_t* packed;  // bit-packed deltas (or lengths)
  void* out;              // DELTA: n values; OFFSETS: n+1 int32
  uint64_t for_base;      // FOR base of the packed stream
  uint64_t base;          // DELTA: base value; OFFSETS: expected total (payload bytes)
  uint32_t n;
  uint32_t tile0;
  uint32_t ntiles;
  uint32_t err_idx;
  uint16_t w;
  uint8_t out_bytes;      // DELTA: 4 or 8; OFFSETS: 4
  uint8_t mode;           // ScanMode
  uint32_t entries;       // DELTA with dict: dictionary entries
  const uint64_t* dict;   // DELTA over Dict|BitPack (Table 2 PS_SUPPKEY): delta_i = dict[FOR + bits_i], else null
};

struct ScanBatch {
  uint32_t n;
  uint32_t total_tiles;
  uint64_t* trace;               // CDM_TRACE: per-tile globaltimer stamps [tile][8], else null
  uint32_t* err;
  unsigned long long* ticket;  // look-back mode: epoch|ticket counter
  uint4* lb;                   // look-back mode: [total_tiles][3] records: flag word, AGG values, INC values
  uint64_t* tsum;              // reduce-then-scan mode: [total_tiles] tile sums (scan_sums_kernel)
  ScanDesc d[kMaxBatch];
};

// ---------------------------------------------------------------- H7: scan-dependent RLE expansion
enum RleValueMode : uint8_t {
  V_BP = 0,      // values = FOR + bits
  V_DICT = 1,    // values = dict[FOR + bits]
  V_F2I = 2,     // values = (double)(FOR + bits) / 10^d
  V_DRLE = 3,    // (host plan only) values = Delta|RLE|[BitPack,BitPack]: decoded by a level-0 V_LINEAR
                 // job into an L2-resident run-value array, then expanded as V_RAW
  V_LINEAR = 4,  // root Delta|RLE|[BitPack,BitPack]: run j is an arithmetic run (start, slope dv_j)
  V_RAW = 5      // values = a plain u64 array (the level-0 output)
};

struct RleDesc {
  const uint8_t* cnt_packed;
  const uint8_t* val_packed;  // V_BP/V_DICT/V_F2I: packed values or indices; V_LINEAR: packed dv;
                              // V_RAW: u64 run values (32-byte aligned)
  const uint8_t* dict;
  void* out;
  const uint64_t* tsum;       // [ntiles][2] per tile {sum of counts, sum of dv*count} (rle_sums)
  uint64_t cnt_base;
  uint64_t val_base;
  uint64_t delta_base;        // V_LINEAR: Delta base
  uint64_t stride;            // strided (DeltaStride): row j of run g = value_g + j * stride
  uint32_t n;                 // output rows
  uint32_t nruns;
  uint32_t tile0;
  uint32_t ntiles;
  uint32_t entries;
  uint32_t err_idx;
  uint16_t cnt_w;
  uint16_t val_w;
  uint8_t vmode;
  uint8_t out_bytes;          // 4 or 8
  uint8_t d;
  uint8_t strided;
};

struct RleBig {  // queue of oversize tiles, expanded by rle_big
  unsigned long long* counter;   // (entries << 44) | pieces
  uint32_t* done;                // rle_big completion counter (resets the queue)
  struct Entry {
    void* out;                   // chunk output base
    uint32_t O;                  // tile output offset in the chunk
    uint32_t T;                  // tile output rows
    uint32_t nr;                 // runs in tile
    uint32_t slot;               // scratch slot
    uint64_t piece0;             // first piece index
    uint32_t out_bytes;
    uint32_t linear;
  }* entries;
  uint32_t* soffs;               // [slots][kRleTile + 1]
  uint64_t* vals;                // [slots][kRleTile]
  uint64_t* slopes;              // [slots][kRleTile]
  uint32_t max_slots;
};

struct RleBatch {
  uint32_t n;
  uint32_t total_tiles;
  uint32_t any_linear;           // some descriptor is V_LINEAR (the kernel variant with a slope table)
  uint64_t* trace;               // CDM_TRACE: per-tile globaltimer stamps [tile][8], else null
  uint32_t* err;
  uint32_t big_enabled;          // 0: rle_big is not launched -> oversize tiles are expanded in place
  uint32_t short_runs;           // <= 16 rows per run on average: the 5-CTAs/SM variant (non-arithmetic)
  RleBig big;
  RleDesc d[kMaxBatch];
};

// rle_sums: per-tile sums of the RLE family, fully parallel (no look-back, no scan): one warp per 1024-run
// tile, tsum[t] = {sum of counts, sum of dv*count (root Delta|RLE)}.  Each rle_kernel CTA reduces the sums
// of the tiles before its own (a few KB from L2) into its output offset.
struct SumsChunk {
  const uint8_t* cnt_packed;   // counts
  const uint8_t* dv_packed;    // V_LINEAR: dv (slopes)
  uint64_t cnt_base, dv_base;
  uint64_t* tsum;              // [tiles][2] count, w
  uint32_t nruns, rows;
  uint32_t tiles;
  uint32_t unit0;              // first global unit (rle_sums CTA) of this chunk
  uint32_t units;
  uint32_t err_idx;
  uint16_t cnt_w, dv_w;
  uint8_t linear;
  uint8_t pad[3];
};

struct SumsBatch {
  uint32_t n;
  uint32_t total_units;
  uint64_t* trace;
  uint32_t* err;
  SumsChunk d[kMaxBatch];
};

// ---------------------------------------------------------------- H8: chunk-sequential LZ4
struct Lz4Desc {
  const uint8_t* payload;  // concatenated LZ4 blocks
  const uint8_t* table;    // n_sub x {u32 comp_off, u32 comp_len, u32 decomp_len}
  uint8_t* out;
  uint64_t payload_bytes;  // compressed payload bytes
  uint64_t n;              // decompressed bytes expected
  uint32_t n_sub;
  uint32_t sub0;           // first global sub-chunk index
  uint32_t err_idx;
  uint32_t uniform;        // > 0: every sub-chunk but the last decompresses to exactly this many bytes
};

// LZ4 launches take up to kMaxLz4Batch chunks (a 14 KB __grid_constant__ parameter): the thread kernel's CTAs
// retire in waves of one sub-chunk chain each, so fewer, larger launches leave fewer partly idle drain waves
constexpr int kMaxLz4Batch = 256;
struct Lz4Batch {
  uint32_t n;
  uint32_t total_subs;
  uint32_t* err;
  Lz4Desc d[kMaxLz4Batch];
};
static_assert(sizeof(Lz4Batch) <= 32000, "kernel parameter limit");

// ---------------------------------------------------------------- NEXT-1: chunk-sequential range ANS
struct AnsDesc {
  const uint16_t* words;   // 16-bit renormalisation words of all ANS chunks, each chunk's in decode order
  const uint8_t* table;    // 256 x u16 frequencies, then per chunk {u32 first word, u32 words, u32 state}
  uint8_t* out;            // decoded bytes
  uint64_t n;              // decoded bytes
  uint64_t n_words;
  uint32_t nchunks;
  uint32_t chunk;          // bytes per ANS chunk (multiple of 16)
  uint32_t tile0;          // first global tile (kThreads chunks per tile; kThreads/32 when il = 32)
  uint32_t err_idx;
  uint32_t tl;             // table log (8..12)
  uint32_t il;             // interleaved states per chunk: 1 (thread per chunk) or 32 (warp per chunk)
};

constexpr int kMaxAnsBatch = 256;  // column chunks per ANS launch (a 16 KB grid-constant parameter)
struct AnsBatch {  // one batch holds chunks of one interleave (il) only
  uint32_t n;
  uint32_t total_tiles;
  uint32_t cpw;      // il = 32: chunks per warp (a CTA's slot table serves kThreads/32 * cpw chunks)
  uint32_t* err;
  AnsDesc d[kMaxAnsBatch];
};
static_assert(sizeof(AnsBatch) <= 32000, "kernel parameter limit");

// ---------------------------------------------------------------- NEXT-2: String-dictionary expansion
// PAPER.md:498 ("each unique word serve as a group in [the Group-Parallel pattern] and expands according to the
// lookup dictionary"): token ids -> token bytes at positions = exclusive scan of the tokens' lengths.
constexpr int kSdTile = 2048;         // tokens per tile = 256 threads x 8
constexpr int kSdStage = 24576;       // staged output bytes per tile (larger tiles store directly)
constexpr int kSdDictSmem = 49152;    // dictionaries up to this size are copied into shared memory
struct SdDesc {
  const uint8_t* ids_packed;   // w-bit token ids, LSB-first (a chunk stream or the ANS output in the arena)
  const uint8_t* dict;         // u32 offsets[entries + 1] (validated on the host), then the token bytes
  uint8_t* out;                // decoded bytes (the Str payload)
  uint64_t* tsum;              // [ntiles] token bytes per tile (sd_sums); exclusive prefix after sd_scan
  uint64_t id_base;            // FOR base of the ids
  uint32_t ntok;
  uint32_t n_out;              // bytes the tokens must total
  uint32_t entries;
  uint32_t tile0;
  uint32_t ntiles;
  uint32_t err_idx;
  uint32_t w;
  uint32_t cta0;               // first sd_expand CTA (kSdCtaTiles tiles per CTA)
};

constexpr int kSdCtaTiles = 4;        // sd_expand: tiles per CTA (the dictionary is copied once per CTA)

constexpr int kMaxSdBatch = 256;  // column chunks per String-dictionary launch (an 18 KB grid-constant parameter)
struct SdBatch {
  uint32_t n;
  uint32_t total_tiles;
  uint32_t total_ctas;         // sd_expand grid
  uint32_t dict_smem;          // largest dictionary stream rounded to 16 B + 16 if all fit kSdDictSmem, else 0 (L1)
  uint32_t* err;
  SdDesc d[kMaxSdBatch];
};
static_assert(sizeof(SdBatch) <= 32000, "kernel parameter limit");

// ---------------------------------------------------------------- launchers (return cudaGetLastError)
cudaError_t launch_fp(const FpBatch& b, uint32_t max_w, cudaStream_t s);
// CHAR(n) rows (FP_DICT, every descriptor of the batch with out_bytes == E): the row-group kernel
// (kernels_fpc.cu) for the widths fpc_supported() names; launch_fp routes such batches there
bool fpc_supported(uint32_t E);
cudaError_t launch_fpc(const FpBatch& b, uint32_t E, cudaStream_t s);
cudaError_t launch_scan(const ScanBatch& b, cudaStream_t s);
cudaError_t launch_rle_sums(const SumsBatch& b, cudaStream_t s);
cudaError_t launch_rle(const RleBatch& b, cudaStream_t s);
cudaError_t launch_rle_big(const RleBatch& b, cudaStream_t s);
// max_sub / max_csub: the largest decompressed / compressed sub-chunk of the batch (host-read, selects the schedule)
cudaError_t launch_lz4(const Lz4Batch& b, uint32_t max_sub, uint32_t max_csub, cudaStream_t s);
cudaError_t launch_ans(const AnsBatch& b, bool interleaved, cudaStream_t s);
// String-dictionary: tile sums -> per-descriptor exclusive scan of the sums -> expansion
cudaError_t launch_strdict(const SdBatch& b, cudaStream_t s);
// engine bookkeeping: zero a 16-byte-aligned scratch prefix; move error words into mapped pinned memory
// (copy, then zero them for the next launch)
cudaError_t launch_zero(void* p, size_t bytes, cudaStream_t s);
cudaError_t launch_harvest(uint32_t* err, uint32_t* host_mapped, uint32_t n, cudaStream_t s);
int device_sms();
// per-device launch state (function attributes, occupancy) is cached per device ordinal: an engine on a
// second device of the process configures its own context
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d >= 0 && d < kMaxDevices ? d : 0;
}
// H9 positional checksum of a device buffer, ADDED into *dev_out (zero it first)
cudaError_t launch_checksum(const void* p, uint64_t bytes, uint64_t chunk_id, uint64_t* dev_out, cudaStream_t s);

// NEXT-3: launch parameters the offline tuner explores (Table 3's per-pattern spaces).
// Process-wide; read by the launchers at enqueue time (a captured graph keeps the values it was built with).
enum TuneKnob : int {
  TUNE_FP_CTAS_PER_SM = 0,  // F.P. "L": persistent fp_kernel CTAs per SM (0 = adaptive 2/3/4)
  TUNE_LZ4_LANES = 1,       // N.P. "C": lanes per LZ4 sub-chunk: 1 (thread per sub-chunk), 2..16 (lane groups), 32
  TUNE_SCAN_MODE = 2,       // H6 schedule: 0 reduce-then-scan, 1 decoupled look-back, 2 warp tiles (3 passes, default)
  TUNE_GP_CTAS_PER_SM = 3,  // G.P. "L": resident rle_kernel CTAs per SM (0 = the kernel's occupancy), 1..8
  TUNE_LZ4_SPLIT = 4,       // H8 schedule: 1 = split parse (owner lane) / copy (whole warp), 0 = TUNE_LZ4_LANES
  TUNE_LZ4_SPLIT_G = 5,     // split schedule: sub-chunks per warp, 0 = per launch size, else 1/2/4/8
  TUNE_LZ4_SPEC = 6,        // H8 schedule: speculative parallel parse, warp per sub-chunk (<= 16 KiB): 0 never, 1 small launches, 2 always
  kTuneKnobs
};
int tune_get(int knob);
void tune_set(int knob, int value);

}  // namespace cdm
