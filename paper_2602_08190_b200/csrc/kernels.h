// kernels.h -- device descriptors + host launch wrappers of the sm_100a decode kernels.
//
// Every kernel decodes a BATCH of chunks that share a kernel family in one launch: descriptors are
// passed by value as __grid_constant__ parameters (no descriptor upload), tiles of all chunks are
// enumerated globally (desc.tile0 = first global tile of the chunk).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cdm {

constexpr int kMaxBatch = 32;      // descriptors per launch (more chunks -> more launches)
constexpr int kFpTile = 4096;      // H5 values per tile = 256 threads x 16
constexpr int kScanTile = 4096;    // H6 values per tile = 256 threads x 16
constexpr int kRleTile = 1024;     // H7 runs per tile = 256 threads x 4
constexpr int kPrepOuterTile = 8 * 2048;  // rle_prep OUTER: 8 warps x 2048 runs (two rle tiles each)
constexpr int kPrepInnerTile = 8 * 1024;  // rle_prep INNER: 8 warps x 1024 inner runs
constexpr int kRleOutBytes = 44 * 1024;    // rle_kernel: a tile's output is staged in shared memory (dynamic)
constexpr int kRleWindow = 384;    // DRLE inner-run window staged per outer tile (larger: global search)
constexpr uint32_t kRleBigLimit = 1u << 15;  // a tile with more output rows is expanded by rle_big
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

struct FpBatch {
  uint32_t n;
  uint32_t total_tiles;
  uint32_t* err;          // per-chunk error words
  FpDesc d[kMaxBatch];
};

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
  uint8_t pad[4];
};

struct ScanBatch {
  uint32_t n;
  uint32_t total_tiles;
  uint64_t* trace;               // CDM_TRACE: per-tile globaltimer stamps [tile][8], else null
  uint32_t* err;
  unsigned long long* ticket;  // epoch|ticket counter
  uint4* lb;                   // [total_tiles] 16-byte look-back words
  ScanDesc d[kMaxBatch];
};

// ---------------------------------------------------------------- H7: scan-dependent RLE expansion
enum RleValueMode : uint8_t {
  V_BP = 0,      // values = FOR + bits
  V_DICT = 1,    // values = dict[FOR + bits]
  V_F2I = 2,     // values = (double)(FOR + bits) / 10^d
  V_DRLE = 3,    // values = Delta|RLE|[BitPack,BitPack] closed form from the inner pre-pass
  V_LINEAR = 4   // root Delta|RLE|[BitPack,BitPack]: run j is an arithmetic run (start, slope dv_j)
};

struct RleDesc {
  const uint8_t* cnt_packed;
  const uint8_t* val_packed;  // V_BP/V_DICT/V_F2I: packed values or indices; V_LINEAR: packed dv
  const uint8_t* dict;
  void* out;
  const uint32_t* S;          // V_DRLE inner run table (from rle_prep)
  const uint64_t* Q;
  const uint64_t* DV;
  const uint32_t* tstart;
  const uint4* prefix;        // per outer tile exclusive prefix {flag, count, w} (from rle_prep)
  uint64_t cnt_base;
  uint64_t val_base;
  uint64_t delta_base;        // V_LINEAR: Delta base
  uint32_t n;                 // output rows
  uint32_t nruns;
  uint32_t tile0;
  uint32_t ntiles;
  uint32_t entries;
  uint32_t n_inner;
  uint32_t err_idx;
  uint16_t cnt_w;
  uint16_t val_w;
  uint8_t vmode;
  uint8_t out_bytes;          // 4 or 8
  uint8_t d;
  uint8_t pad[5];
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
  uint64_t* trace;               // CDM_TRACE: per-tile globaltimer stamps [tile][8], else null
  uint32_t* err;
  uint32_t big_enabled;          // 0: rle_big is not launched -> oversize tiles are expanded in place
  uint32_t debug;                // CDM_DEBUG_RLE bits (experiments only): 1 = skip output stores
  RleBig big;
  RleDesc d[kMaxBatch];
};

// rle_prep: every look-back of the RLE family in ONE launch, over tiny per-tile aggregates only.
//  PREP_OUTER: per outer tile of kRleTile runs, sum of counts (and of dv*count for arithmetic runs) ->
//              exclusive prefix per tile, so rle_kernel never waits on a predecessor.
//  PREP_INNER: Delta|RLE value lineage (V_DRLE): per inner run j, S_j (first outer run), Q_j (base +
//              sum_{k<j} dv_k dc_k), DV_j, and tstart[t] (inner run holding outer run t*kRleTile;
//              tstart[outer_tiles] = n_inner - 1 closes the last window).
enum PrepKind : uint8_t { PREP_OUTER = 0, PREP_INNER = 1 };

struct PrepDesc {
  const uint8_t* a_packed;    // OUTER: counts;  INNER: dc
  const uint8_t* b_packed;    // OUTER(linear): dv; INNER: dv
  uint4* prefix;              // OUTER: [ntiles] exclusive prefixes
  uint32_t* S;                // INNER outputs
  uint64_t* Q;
  uint64_t* DV;
  uint32_t* tstart;
  uint64_t a_base;
  uint64_t b_base;
  uint64_t base;              // INNER: Delta base
  uint32_t n_items;           // OUTER: runs; INNER: inner runs
  uint32_t total;             // OUTER: rows (sum of counts); INNER: outer runs (sum of dc)
  uint32_t tile0;
  uint32_t ntiles;
  uint32_t outer_tiles;       // INNER: ceil(outer runs / kRleTile); OUTER: ceil(runs / kRleTile)
  uint32_t err_idx;
  uint16_t a_w;
  uint16_t b_w;
  uint8_t kind;               // PrepKind
  uint8_t linear;             // OUTER: also accumulate dv*count
  uint8_t pad[6];
};

struct PrepBatch {
  uint32_t n;
  uint32_t total_tiles;
  uint64_t* trace;
  uint32_t* err;
  unsigned long long* ticket;
  uint4* lb;
  PrepDesc d[kMaxBatch];
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

struct Lz4Batch {
  uint32_t n;
  uint32_t total_subs;
  uint32_t* err;
  Lz4Desc d[kMaxBatch];
};

// ---------------------------------------------------------------- launchers (return cudaGetLastError)
cudaError_t launch_fp(const FpBatch& b, uint32_t max_w, cudaStream_t s);
cudaError_t launch_scan(const ScanBatch& b, cudaStream_t s);
cudaError_t launch_rle_prep(const PrepBatch& b, cudaStream_t s);
cudaError_t launch_rle(const RleBatch& b, cudaStream_t s);
cudaError_t launch_rle_big(const RleBatch& b, cudaStream_t s);
cudaError_t launch_lz4(const Lz4Batch& b, uint32_t max_sub, cudaStream_t s);
int device_sms();

}  // namespace cdm
