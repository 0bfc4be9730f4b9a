/*
 * cdm.h -- C-ABI of libcdm, the B200 (sm_100a) decode hot path of "a Compiler-based Framework to
 * Unleash Compressed Data Movement for Modern GPUs" (arxiv 2602.08190).
 *
 * The paper's problem statement (Sec. 3 Design): columns are compressed on the CPU
 * with nested lightweight codecs and stored in CPU memory; the framework "facilitates the efficient
 * movement of compressed data across the PCIe interconnect, followed by an ultra-fast, device-specific
 * decompression phase", with "optimized overlap between PCIe data transfers and on-device
 * decompression".  The three calls of that statement are:
 *   describe a column's encoding cascade   -> cdm_cascade_create   (Table 2 notation)
 *   submit compressed chunks from pinned host memory -> cdm_submit / cdm_submit_batch
 *                                             (Pipelining Layer, Johnson order)
 *   receive decoded device buffers          -> cdm_wait / cdm_synchronize (caller-owned device memory)
 * plus a device-resident batch API (cdm_batch_*) that decodes chunks already in HBM, used to measure
 * the kernels alone.
 *
 * Conventions.
 *  - All pointers are plain host or device pointers; sizes are bytes unless stated.  No torch types.
 *  - Every call returns cdm_status; nothing throws or aborts across the ABI.  Argument errors are
 *    reported synchronously; data errors found on the device (dictionary index out of range, run
 *    lengths not summing to the row count, LZ4 offsets/lengths out of bounds) are reported by
 *    cdm_wait / cdm_batch_results as CDM_E_CORRUPT with cdm_result.error_bits set.  Kernels never
 *    read or write out of bounds, even on corrupt input.
 *  - Ordering: the engine's copy/decode streams are non-blocking with respect to the legacy default stream.
 *    Writes the caller makes to dev_out / dev_offsets / dev_chunk (e.g. torch fills on the default stream)
 *    must be complete, or ordered before the launch stream passed in, when a job is submitted or launched;
 *    results are ready after cdm_wait / cdm_batch_results / cdm_pipeline_results or cdm_ticket_event.
 *  - cdm_last_error() returns a thread-local human-readable detail of the last failing call.
 *  - Chunks are CDM1 containers: self-contained row groups of
 *    < 2^31 rows, little-endian, 16-byte aligned zero-padded streams.
 *  - Threading: one engine per (process, device).  cdm_submit, cdm_submit_batch, cdm_wait, cdm_ticket_event
 *    and cdm_synchronize are thread-safe on one engine (serialised by an engine mutex; a wait blocks with the
 *    mutex released).  Batches and pipelines are single-threaded objects.  Cascades are immutable and may be
 *    shared by engines and threads.
 */
#ifndef CDM_H
#define CDM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define CDM_API __attribute__((visibility("default")))
#else
#define CDM_API
#endif

typedef enum {
  CDM_OK = 0,
  CDM_E_INVALID_ARG = 1,  /* null/misaligned pointer, bad size, bad option */
  CDM_E_PARSE = 2,        /* cascade text does not parse / arity error (Table 2 grammar) */
  CDM_E_UNSUPPORTED = 3,  /* a valid cascade with no fused device plan, or dtype mismatch */
  CDM_E_CORRUPT = 4,      /* bad magic/version/bounds (host check) or device-detected data error */
  CDM_E_CAPACITY = 5,     /* output buffer or staging slot too small */
  CDM_E_CUDA = 6,         /* a CUDA runtime call failed (detail in cdm_last_error) */
  CDM_E_OOM = 7,          /* device or pinned allocation failed */
  CDM_E_BUSY = 8          /* unknown / already-consumed ticket */
} cdm_status;

/* Decoded element types (SURVEY Sec. 8d "Decoded types"). */
typedef enum {
  CDM_I32 = 0,      /* int32 (identifiers, date32 days since 1970-01-01) */
  CDM_I64 = 1,      /* int64 (order keys) */
  CDM_F64 = 2,      /* IEEE float64 (decimals) */
  CDM_FIXED = 3,    /* fixed-width byte rows, width bytes each (CHAR(n)) */
  CDM_VARBYTES = 4  /* variable-length bytes + int32 offsets[rows+1] (VARCHAR) */
} cdm_dtype;

/* Device error bits (cdm_result.error_bits). */
#define CDM_ERR_DICT_INDEX 0x1u   /* a dictionary index >= number of entries */
#define CDM_ERR_RUN_SUM 0x2u      /* RLE counts do not sum to the node's element count */
#define CDM_ERR_LZ4 0x4u          /* malformed LZ4 block: offset 0 / before start, over-run, truncation */
#define CDM_ERR_LENGTHS 0x8u      /* VARBYTES lengths do not sum to the payload size */
#define CDM_ERR_WIDTH 0x10u       /* a bit width unusable for the stream it packs */
#define CDM_ERR_ANS 0x20u         /* an ANS chunk does not end at the initial state with every word read */

typedef struct cdm_engine cdm_engine;
typedef struct cdm_cascade cdm_cascade;
typedef struct cdm_batch cdm_batch;
typedef struct cdm_pipeline cdm_pipeline;

typedef struct {
  uint32_t n_slots;       /* device staging ring depth, >= 2 (default 4) */
  uint64_t slot_bytes;    /* bytes per staging slot; a chunk must fit one slot (default 64 MiB) */
  void *copy_stream;      /* cudaStream_t for H2D copies, or NULL: the engine creates one */
  void *decode_stream;    /* cudaStream_t for decode kernels: every group decodes in order on it; NULL: the
                             engine gives each staging slot its own decode stream, so groups held by
                             different slots decode concurrently (the default) */
  double pcie_gbps;       /* H2D link estimate for Johnson costs t_i (default 55 GB/s) */
  double decode_gbps;     /* element-parallel decode rate for Johnson costs d_i (default 5000 GB/s); the
                             other kernel families are costed at fixed fractions of it measured on B200
                             (scan 1/2, RLE 1/8, LZ4 1/40, raw copy 1) */
  uint32_t order_policy;  /* 0 = submission order, 1 = Johnson's rule */
  uint32_t flags;         /* CDM_ENGINE_* */
} cdm_engine_opts;

/* cdm_engine_opts.flags: compute the H9 positional checksum of every chunk decoded through cdm_submit* on the
 * device, after its decode (cdm_result.checksum): h = sum over the 8-byte words k of the zero-padded payload of
 * splitmix64(chunk_id ^ k ^ word_k) mod 2^64, plus the same over the offsets under chunk_id ^ 2^63. */
#define CDM_ENGINE_CHECKSUM 0x1u

typedef struct {
  uint64_t rows;              /* rows decoded */
  uint64_t payload_bytes;     /* decoded payload bytes written to dev_out */
  uint64_t offsets_bytes;     /* decoded offsets bytes written to dev_offsets (VARBYTES) */
  uint64_t compressed_bytes;  /* bytes of the chunk (what crossed PCIe) */
  uint64_t chunk_id;          /* from the chunk header */
  uint32_t error_bits;        /* CDM_ERR_* found on the device, 0 if clean */
  uint32_t status;            /* cdm_status of this chunk */
  uint64_t checksum;          /* H9 checksum of the decoded chunk (engines created with CDM_ENGINE_CHECKSUM), else 0 */
} cdm_result;

typedef struct {
  const cdm_cascade *cascade;  /* compiled cascade the chunk was encoded with */
  const void *host_chunk;      /* CDM1 chunk in host memory (pinned for cdm_submit*); headers are read here */
  const void *dev_chunk;       /* the same bytes already resident in device memory (cdm_batch_*), else NULL */
  size_t chunk_bytes;          /* chunk size in bytes (>= header total) */
  void *dev_out;               /* device output, >= payload bytes; 16-byte aligned */
  size_t dev_out_bytes;
  void *dev_offsets;           /* VARBYTES: device int32[rows+1]; else NULL */
  size_t dev_offsets_bytes;
} cdm_job;

CDM_API const char *cdm_status_str(cdm_status s);
CDM_API const char *cdm_last_error(void);
CDM_API const char *cdm_version(void);

/* ---- cascades (Nesting Layer; fusion rules PAPER.md:277-278) ----
 * spec: Table 2 notation, e.g. "Dict|BitPack", "RLE|[Delta|RLE|[BitPack,BitPack],BitPack]",
 * "Str|[LZ4,BitPack]" (case-insensitive, "Bit-packing"/"Dictionary encoding" accepted).
 * The cascade is compiled into a fused plan of at most three kernel launches per chunk; a cascade
 * that parses but has no fused device plan returns CDM_E_UNSUPPORTED.  width: row bytes for
 * CDM_FIXED, ignored otherwise. */
CDM_API cdm_status cdm_cascade_create(const char *spec, cdm_dtype dtype, uint32_t width, cdm_cascade **out);
CDM_API cdm_status cdm_cascade_destroy(cdm_cascade *c);
/* canonical text (e.g. "DICT|[RAW,BITPACK|RAW]") + " => " + the fused plan, into buf (NUL-terminated) */
CDM_API cdm_status cdm_cascade_describe(const cdm_cascade *c, char *buf, size_t cap);

/* Host-only parse + validation of a chunk header (no device work). */
CDM_API cdm_status cdm_chunk_info(const void *host_chunk, size_t bytes, cdm_result *out);
/* Host-only: validate a chunk against a cascade exactly as cdm_submit / cdm_batch_create will (header,
 * node tree == cascade, stream bounds, per-codec sizes); no device memory is touched. */
CDM_API cdm_status cdm_chunk_check(const cdm_cascade *c, const void *host_chunk, size_t bytes);

/* ---- engine: staging ring + copy/decode streams (Pipelining Layer) ---- */
CDM_API cdm_status cdm_engine_create(int device, const cdm_engine_opts *opts, cdm_engine **out);
CDM_API cdm_status cdm_engine_destroy(cdm_engine *e);  /* waits for in-flight work */

/* Asynchronously copy one chunk H2D into a staging slot (copy stream) and decode it (decode stream)
 * after the copy's event.  host_chunk must stay valid and unmodified until the ticket completes. */
CDM_API cdm_status cdm_submit(cdm_engine *e, const cdm_job *job, uint64_t *ticket);
/* Submit n jobs; with order_policy = 1 they are issued in Johnson order (tickets[i] is job i's). */
CDM_API cdm_status cdm_submit_batch(cdm_engine *e, const cdm_job *jobs, size_t n, uint64_t *tickets);
/* Block until the ticket's decode finished; fills *out.  CDM_E_CORRUPT if error_bits != 0. */
CDM_API cdm_status cdm_wait(cdm_engine *e, uint64_t ticket, cdm_result *out);
/* A CUDA event (cudaEvent_t, owned by the engine) that completes when the ticket's decode (and its checksum)
 * has finished, so a consumer stream can cudaStreamWaitEvent on it without a host synchronisation
 * (SURVEY Sec. 8b).  Valid until the ticket is consumed by cdm_wait; for a ticket whose group was already
 * harvested it is an event that has completed.  Errors: CDM_E_INVALID_ARG, CDM_E_BUSY (unknown ticket). */
CDM_API cdm_status cdm_ticket_event(cdm_engine *e, uint64_t ticket, void **cuda_event);
/* NEXT-4 multi-link ingestion (Vortex): route the H2D copies of cdm_submit* over the PCIe links of
 * `devices` (round-robin per group): each group is copied into a staging buffer on that device and then peer-copied
 * over NVLink into the engine device's staging slot, so one consumer GPU can draw on several hosts links.  A listed
 * device equal to the engine's takes the same two-hop path (H2D, then a device-to-device copy).  n = 0 restores
 * direct copies.  Drains in-flight work first; allocates slot_bytes on each listed device.
 * Errors: CDM_E_INVALID_ARG (null / device out of range), CDM_E_OOM, CDM_E_CUDA. */
CDM_API cdm_status cdm_engine_set_ingest(cdm_engine *e, const int *devices, size_t n);
/* Kernels the engine has enqueued through cdm_submit* so far (fused decode kernels, scratch zeroing, error
 * harvest, checksums): the launch count of a measured region is the difference of two reads. */
CDM_API cdm_status cdm_engine_launches(cdm_engine *e, uint64_t *n);
/* Wait for everything submitted so far (results stay retrievable with cdm_wait). */
CDM_API cdm_status cdm_synchronize(cdm_engine *e);
/* H3 as a pure host function: Johnson's rule over jobs with transfer costs t[i] and
 * decode costs d[i]; writes the issue order (a permutation of 0..n-1) to order[].  Jobs with t <= d come
 * first by ascending t, the rest by descending d, ties by index.  O(n log n). */
CDM_API cdm_status cdm_johnson_order(const double *t, const double *d, size_t n, size_t *order);

/* ---- device-resident batches: chunks already in HBM (job.dev_chunk), decoded by grouped launches ----
 * create: parses/validates headers on the host and sizes scratch (no device work is enqueued);
 * launch: enqueues the fused decode of every job on `stream` (cudaStream_t, NULL = engine decode
 *         stream); capturable into a CUDA graph; returns the number of kernel launches in *n_launches;
 * results: synchronises `stream` and reads the per-chunk device error words, then clears them: error
 *          bits accumulate (OR) over all launches since the previous cdm_batch_results. */
CDM_API cdm_status cdm_batch_create(cdm_engine *e, const cdm_job *jobs, size_t n, cdm_batch **out);
CDM_API cdm_status cdm_batch_launch(cdm_batch *b, void *stream, uint32_t *n_launches);
CDM_API cdm_status cdm_batch_results(cdm_batch *b, void *stream, cdm_result *results);
CDM_API cdm_status cdm_batch_destroy(cdm_batch *b);
/* Graph mode (enable != 0): the first cdm_batch_launch on a stream captures the whole enqueue into a CUDA
 * graph, later launches on that stream replay it with one cudaGraphLaunch (re-captured when the stream or
 * the timing setting changes; the jobs' buffers must stay where they were).  Removes the host launch
 * overhead of the ~10 kernel launches + fork/join events per decode. */
CDM_API cdm_status cdm_batch_set_graph(cdm_batch *b, int enable);

/* ---- pipelines: a fixed job set from PINNED host memory, captured once into a CUDA graph ----
 * The H4 schedule of cdm_submit_batch (Johnson order, groups, H2D copies overlapped with the fused
 * decodes of earlier groups) recorded as one graph: every launch re-copies each job's
 * host_chunk (which must be pinned and may change contents, not size or structure, between launches)
 * and decodes it into the job's dev_out / dev_offsets.  Staging and scratch are owned by the pipeline.
 * create: binds/validates every job on the host, allocates, captures and instantiates (no device work);
 *         CDM_E_CAPACITY if one chunk exceeds the engine's slot_bytes;
 * launch: one cudaGraphLaunch on `stream` (cudaStream_t, NULL = engine decode stream): the copies and
 *         decodes are ordered after the stream's prior work and the stream waits for them;
 * results: synchronises that stream and fills results[i] for job i from the error words the graph
 *         wrote to mapped pinned memory; CDM_E_CORRUPT if any job has error bits. */
CDM_API cdm_status cdm_pipeline_create(cdm_engine *e, const cdm_job *jobs, size_t n, cdm_pipeline **out);
CDM_API cdm_status cdm_pipeline_launch(cdm_pipeline *p, void *stream);
CDM_API cdm_status cdm_pipeline_results(cdm_pipeline *p, cdm_result *results);
CDM_API cdm_status cdm_pipeline_destroy(cdm_pipeline *p);
/* What one cdm_pipeline_launch enqueues: kernel launches (every decode kernel + the error harvest), groups
 * (staging regions / multi-chunk batches) and H2D copies (runs of host-contiguous chunks). */
CDM_API cdm_status cdm_pipeline_info(const cdm_pipeline *p, uint32_t *n_launches, uint32_t *n_groups,
                                     uint32_t *n_copies);

/* ---- pinned host memory: page-lock (cudaHostRegister) a caller-owned host range in place, so chunks that
 * live in it can be submitted (the paper pins all host buffers).  p/bytes: the range (page
 * aligned for best results); unregister before freeing it.  Errors: CDM_E_INVALID_ARG, CDM_E_CUDA. */
CDM_API cdm_status cdm_host_register(void *p, size_t bytes);
CDM_API cdm_status cdm_host_unregister(void *p);
/* Allocate / free page-locked host memory for a column store (cudaHostAlloc; exactly `bytes`, no rounding).
 * Errors: CDM_E_INVALID_ARG, CDM_E_OOM. */
CDM_API cdm_status cdm_host_alloc(size_t bytes, void **out);
CDM_API cdm_status cdm_host_free(void *p);

/* ---- instrumentation ---- */
/* Record CUDA events around each kernel family (enable = 1) or around each kernel launch (enable = 2,
 * which runs the families one after another and serialises programmatically dependent launches, so each
 * launch is timed alone) issued by cdm_batch_launch; 0 = off; every
 * call resets the accumulators.  After cdm_batch_results (or cdm_batch_collect_timing in graph mode):
 * cdm_batch_kernel_ms() -> per-family milliseconds and launches: index 0 FP (H5), 1 delta/offset scan (H6),
 *   2 RLE (H7), 3 LZ4 (H8), 4 raw copies;
 * cdm_batch_kernel_times() -> per-kernel milliseconds and launches (mode 2): index 0 fp_kernel (numeric rows),
 *   1 scan_kernel, 2 rle_sums_kernel, 3 rle_kernel level 0 (value lineage), 4 rle_kernel, 5 rle_big_kernel,
 *   6 lz4 kernel, 7 device copies, 8 ANS kernel, 9 String-dictionary (sd_sums + sd_scan + sd_expand),
 *   10 fp_kernel on FIXED (CHAR(n)) rows (arrays of CDM_KERNEL_KINDS);
 * cdm_batch_kernel_bytes() -> per kernel kind, the ALGORITHMIC bytes one launch of the batch moves (Eq. 1,
 *   the compressed bytes the kind must read + the decoded bytes it must write, summed over
 *   the batch's jobs; a job's whole RLE chain -- counts, values, output -- is booked on index 4). */
#define CDM_KERNEL_KINDS 11
CDM_API cdm_status cdm_batch_set_timing(cdm_batch *b, int enable);
CDM_API cdm_status cdm_batch_kernel_ms(cdm_batch *b, double *ms5, uint64_t *launches5);
CDM_API cdm_status cdm_batch_kernel_times(cdm_batch *b, double *ms, uint64_t *launches);
CDM_API cdm_status cdm_batch_kernel_bytes(cdm_batch *b, uint64_t *bytes);
/* Graph mode + timing: every replay re-records the same events, so call this after each launch (it
 * waits for that replay) to accumulate its per-family times; a replay not collected is not counted. */
CDM_API cdm_status cdm_batch_collect_timing(cdm_batch *b);

/* ---- H9: optional positional checksum of a decoded device buffer:
 *   h = sum_i splitmix64(chunk_id ^ i ^ w_i) mod 2^64 over its little-endian 8-byte words w_i (the last one
 *   zero padded), computed by a kernel on `stream` (a cudaStream_t, NULL = legacy default stream); the call
 *   waits for it and writes h to *out (host).  dev_data: device pointer, 8-byte aligned (16 reads faster).
 *   Errors: CDM_E_INVALID_ARG (null / misaligned), CDM_E_CUDA. */
CDM_API cdm_status cdm_checksum(const void *dev_data, uint64_t bytes, uint64_t chunk_id, void *stream, uint64_t *out);

/* ---- NEXT-3: launch-parameter knobs for the offline tuner ("Native Config", Table 3).
 * Process-wide, read when a batch / pipeline is enqueued or captured (a captured graph keeps its values).
 *   "fp_ctas_per_sm"  F.P. pattern's L: persistent fp_kernel CTAs per SM, 0 = adaptive (2/3/4 by batch
 *                     length), 1..16 (clamped to what fits an SM); env CDM_FP_CTAS_PER_SM sets the start value
 *   "lz4_lanes"       N.P. pattern's C: lanes cooperating on one LZ4 sub-chunk: 1 (default: the paper's thread
 *                     per chunk, lz4_thread_kernel), 2, 4, 8, 16 (lane groups) or 32 (one warp per sub-chunk);
 *                     env CDM_LZ4_G sets the start value
 *   "lz4_split"       H8 schedule: 1 (default) = the split parse/copy kernel for latency-bound LZ4 launches (owner
 *                     lanes parse sequence headers from a shared ring, the whole warp copies literals and matches
 *                     32 sequences at a time) and the lz4_lanes schedule for throughput-bound ones; 0 = always
 *                     lz4_lanes; env CDM_LZ4_SPLIT sets the start value
 *   "lz4_split_g"     sub-chunks per warp of the split kernel: 0 (default) = by launch size (latency-bound launches
 *                     only), 1, 2, 4 or 8 = always the split kernel with that many; env CDM_LZ4_SPLIT_G
 *   "lz4_spec"        H8 schedule: the speculative-parse kernel (a warp per sub-chunk of <= 16 KiB: 32 lanes walk the
 *                     header chain from 32 segment starts, a fix-up re-walks each segment from its true entry to
 *                     the merge point, then 32 sequences per step are copied into a shared-memory output image):
 *                     1 (default) = for launches of at most two of its waves, 2 = always, 0 = never; env CDM_LZ4_SPEC
 *   "gp_ctas_per_sm"  G.P. pattern's L (Table 3 G.P. row): resident rle_kernel CTAs per SM, 0 = the kernel's own
 *                     occupancy (default), 1..8 (enforced by padding the launch's dynamic shared memory)
 *   "scan_mode"       H6 schedule (single-pass look-back vs the 2-pass baseline): 0 =
 *                     reduce-then-scan (tile sums, then a persistent scan), 1 = single-pass decoupled look-back
 *                     (one tile per CTA in ticket order), 2 = warp tiles (default: 512-value warp-tile sums, a
 *                     per-chunk scan of them, then one warp per tile with no CTA barrier); env CDM_SCAN_MODE
 * Errors: CDM_E_INVALID_ARG for an unknown knob, a value outside its set, or a null pointer. */
CDM_API cdm_status cdm_tune_set(const char *knob, int value);
CDM_API cdm_status cdm_tune_get(const char *knob, int *value);

#ifdef __cplusplus
}
#endif
#endif /* CDM_H */
