// runtime.cpp -- libcdm: the C-ABI (include/cdm.h) over the sm_100a decode kernels.
//
//  H1  cascade text -> fused plan                      (plan.h)
//  H2  CDM1 chunk parse/validation + binding to a plan  (format.h)
//  H3  Johnson order of chunk jobs
//  H4  H2D copies into a device staging ring on a copy stream, decode on a decode stream after the
//      copy's event (overlap of PCIe transfers and on-device decompression)
//  H5-H8 grouped kernel launches (kernels_*.cu), H9 per-chunk device error words.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <array>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "cdm.h"
#include "format.h"
#include "kernels.h"
#include "plan.h"

using namespace cdm;

// ============================================================================ errors
static thread_local std::string g_last;
static cdm_status fail(cdm_status s, const std::string& m) {
  g_last = m;
  return s;
}
#define CUDA_TRY(x)                                                                      \
  do {                                                                                   \
    cudaError_t _e = (x);                                                                \
    if (_e != cudaSuccess) return fail(CDM_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e)); \
  } while (0)

extern "C" CDM_API const char* cdm_status_str(cdm_status s) {
  switch (s) {
    case CDM_OK: return "ok";
    case CDM_E_INVALID_ARG: return "invalid argument";
    case CDM_E_PARSE: return "cascade parse error";
    case CDM_E_UNSUPPORTED: return "unsupported";
    case CDM_E_CORRUPT: return "corrupt chunk";
    case CDM_E_CAPACITY: return "capacity";
    case CDM_E_CUDA: return "cuda error";
    case CDM_E_OOM: return "out of memory";
    case CDM_E_BUSY: return "busy / unknown ticket";
  }
  return "unknown";
}
extern "C" CDM_API const char* cdm_last_error(void) { return g_last.c_str(); }
extern "C" CDM_API const char* cdm_version(void) { return "cdm 0.1 (sm_100a)"; }

// ============================================================================ cascades
struct cdm_cascade {
  std::string canonical;
  uint64_t hash = 0;
  uint8_t dtype = 0;
  uint32_t width = 0;
  Plan plan;
};

static uint32_t dtype_width(uint8_t dtype, uint32_t width) {
  switch (dtype) {
    case T_I32: return 4;
    case T_I64: case T_F64: return 8;
    case T_FIXED: return width;
    case T_VARBYTES: return 1;
  }
  return 0;
}

extern "C" CDM_API cdm_status cdm_cascade_create(const char* spec, cdm_dtype dtype, uint32_t width, cdm_cascade** out) {
  if (!spec || !out) return fail(CDM_E_INVALID_ARG, "null argument");
  if (dtype > CDM_VARBYTES) return fail(CDM_E_INVALID_ARG, "bad dtype");
  if (dtype == CDM_FIXED && width == 0) return fail(CDM_E_INVALID_ARG, "FIXED needs width > 0");
  std::string text(spec);
  CascadeParser P(text);
  auto root = P.node();
  if (!root) return fail(CDM_E_PARSE, P.err);
  P.ws();
  if (P.pos != text.size()) return fail(CDM_E_PARSE, "parse error at " + std::to_string(P.pos) + ": trailing input");
  std::string err;
  if (!complete_tree(root.get(), &err)) return fail(CDM_E_PARSE, err);
  auto c = std::make_unique<cdm_cascade>();
  render_tree(root.get(), &c->canonical);
  c->hash = fnv1a64(c->canonical);
  c->dtype = uint8_t(dtype);
  c->width = dtype == CDM_FIXED ? width : dtype_width(uint8_t(dtype), 0);
  if (!compile_plan(root.get(), uint8_t(dtype), &c->plan, &err)) return fail(CDM_E_UNSUPPORTED, c->canonical + ": " + err);
  *out = c.release();
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_cascade_destroy(cdm_cascade* c) {
  delete c;
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_cascade_describe(const cdm_cascade* c, char* buf, size_t cap) {
  if (!c || !buf || !cap) return fail(CDM_E_INVALID_ARG, "null argument");
  std::string s = c->canonical + " => " + c->plan.text;
  if (s.size() + 1 > cap) return fail(CDM_E_CAPACITY, "buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return CDM_OK;
}

// ============================================================================ chunk binding
namespace {

struct BPB {  // a bound BitPack node
  uint64_t off = 0;  // packed stream offset within the chunk
  uint64_t n = 0;
  uint32_t w = 0;
  uint64_t base = 0;
};

// one expansion level of an RLE-family job (deepest first; the last one writes the column)
struct RleLevel {
  BPB cnt, val;           // counts; values (V_BP / V_DICT / V_F2I) or slopes dv (V_LINEAR); V_RAW: unused
  uint8_t vmode = 0;      // RleValueMode; V_RAW = the previous level's array
  bool strided = false;   // DeltaStride node: row j of run g = value_g + j * stride
  uint64_t delta_base = 0, stride = 0;
  uint32_t n = 0, nruns = 0, max_run = 0;
  int val_src = -1;       // V_RAW: the level (index into Bound::lv) whose u64 output holds the run values
  int cnt_src = -1;       // counts lineage (Table 2 PS_PARTKEY): the level whose u32 output holds the counts
  bool as_counts = false; // this level's output is another level's counts (written as u32)
};

struct Bound {
  const cdm_cascade* casc = nullptr;
  PlanKind kind = PlanKind::RawCopy;
  uint8_t fp_mode = 0, vmode = 0;
  uint64_t rows = 0, payload = 0, offsets_bytes = 0, total = 0, chunk_id = 0;
  uint32_t W = 0;
  BPB main;
  std::vector<RleLevel> lv;  // PlanKind::Rle
  uint64_t dict_off = 0;
  uint32_t entries = 0;
  uint8_t d = 0;
  uint64_t delta_base = 0;
  bool lz4 = false;
  uint64_t lz_pay_off = 0, lz_pay_bytes = 0, lz_tab_off = 0, bytes_off = 0, raw_off = 0;
  uint32_t n_sub = 0, lz_sub_bytes = 0, lz_sub_cbytes = 0, lz_uniform = 0;
  bool ans = false;  // NEXT-1: the bytes come from a range-ANS node (Str child or FIXED root)
  uint64_t ans_w_off = 0, ans_w_n = 0, ans_tab_off = 0, ans_n = 0;
  uint32_t ans_nchunks = 0, ans_chunk = 0, ans_tl = 0, ans_il = 1;
  bool strdict = false;  // NEXT-2: the bytes come from a String-dictionary node (ids BitPack'd, maybe |ANS)
  uint64_t sd_dict_off = 0, sd_ids_off = 0, sd_id_base = 0;
  uint32_t sd_entries = 0, sd_ntok = 0, sd_w = 0, sd_dict_bytes = 0;
  const uint8_t* dev_chunk = nullptr;
  void* out = nullptr;
  void* offs = nullptr;
};

struct Tree {
  const Chunk& c;
  std::vector<std::vector<int>> kids;
  std::string err;
  explicit Tree(const Chunk& ch) : c(ch), kids(ch.nodes.size()) {}
  int walk(size_t* idx) {
    if (*idx >= c.nodes.size()) { err = "node table: missing nodes"; return -1; }
    int me = int((*idx)++);
    for (uint32_t k = 0; k < c.nodes[me].nchild; k++) {
      int ch = walk(idx);
      if (ch < 0) return -1;
      kids[me].push_back(ch);
    }
    return me;
  }
  void render(int i, std::string* out) const {
    *out += codec_name(c.nodes[i].codec);
    if (kids[i].empty()) return;
    *out += "|";
    if (kids[i].size() == 1) { render(kids[i][0], out); return; }
    *out += "[";
    for (size_t k = 0; k < kids[i].size(); k++) {
      if (k) *out += ",";
      render(kids[i][k], out);
    }
    *out += "]";
  }
};

std::string raw_stream(const Chunk& c, const Tree& t, int i, uint32_t eb, uint64_t* off, uint64_t* n) {
  const Node& nd = c.nodes[i];
  if (nd.codec != RAW) return "node " + std::to_string(i) + ": expected Raw";
  if (nd.stream >= c.streams.size()) return "node " + std::to_string(i) + ": stream out of range";
  if (nd.elem_bytes == 0 || (eb && nd.elem_bytes != eb)) return "node " + std::to_string(i) + ": raw element bytes";
  const Stream& s = c.streams[nd.stream];
  if (nd.n > s.bytes / nd.elem_bytes || nd.n * nd.elem_bytes != s.bytes)
    return "node " + std::to_string(i) + ": raw stream length mismatch";
  *off = s.offset;
  *n = nd.n;
  (void)t;
  return "";
}

std::string bind_bp(const Chunk& c, const Tree& t, int i, uint64_t n_expect, uint32_t max_w, BPB* b) {
  const Node& nd = c.nodes[i];
  if (nd.codec != BITPACK || t.kids[i].size() != 1) return "node " + std::to_string(i) + ": expected BitPack";
  if (nd.n != n_expect) return "node " + std::to_string(i) + ": BitPack element count mismatch";
  if (nd.w() > max_w) return "node " + std::to_string(i) + ": bit width " + std::to_string(nd.w()) + " too large";
  uint64_t off, bytes;
  std::string e = raw_stream(c, t, t.kids[i][0], 1, &off, &bytes);
  if (!e.empty()) return e;
  if ((nd.n * nd.w() + 7) / 8 > bytes) return "node " + std::to_string(i) + ": packed stream too short";
  b->off = off;
  b->n = nd.n;
  b->w = nd.w();
  b->base = nd.u64_at8();
  return "";
}

cdm_status bind_job(const cdm_job& job, Bound* b) {
  if (!job.cascade || !job.host_chunk) return fail(CDM_E_INVALID_ARG, "job needs a cascade and a host chunk");
  const cdm_cascade* cs = job.cascade;
  Chunk c;
  std::string e = parse_chunk(job.host_chunk, job.chunk_bytes, &c);
  if (!e.empty()) return fail(CDM_E_CORRUPT, e);
  if (c.cascade_hash != cs->hash) return fail(CDM_E_CORRUPT, "chunk was encoded with another cascade (hash mismatch)");
  if (c.dtype != cs->dtype) return fail(CDM_E_CORRUPT, "chunk dtype differs from the cascade's");
  Tree t(c);
  size_t idx = 0;
  if (c.nodes.empty() || t.walk(&idx) != 0 || idx != c.nodes.size()) return fail(CDM_E_CORRUPT, t.err.empty() ? "node table: unused nodes" : t.err);
  for (size_t i = 0; i < c.nodes.size(); i++) {
    static const int arity[11] = {0, 1, 2, 1, 1, 2, 2, 2, 2, 2, 2};
    if (c.nodes[i].codec > STRDICT || t.kids[i].size() != size_t(arity[c.nodes[i].codec]))
      return fail(CDM_E_CORRUPT, "node " + std::to_string(i) + ": bad codec or arity");
  }
  std::string canon;
  t.render(0, &canon);
  if (canon != cs->canonical) return fail(CDM_E_CORRUPT, "chunk tree " + canon + " != cascade " + cs->canonical);
  const uint32_t W = dtype_width(c.dtype, c.width);
  if (c.dtype == T_FIXED && c.width != cs->width) return fail(CDM_E_CORRUPT, "FIXED width differs from the cascade's");
  if (W == 0) return fail(CDM_E_CORRUPT, "zero width");
  b->casc = cs;
  b->kind = cs->plan.kind;
  b->fp_mode = cs->plan.fp_mode;
  b->vmode = cs->plan.vmode;
  b->rows = c.rows;
  b->payload = c.payload_bytes;
  b->offsets_bytes = c.offsets_bytes;
  b->total = c.total_bytes;
  b->chunk_id = c.chunk_id;
  b->W = W;
  const Node& r = c.nodes[0];
  // an ANS root decodes rows * W bytes of a FIXED(W) column
  if (r.n != (b->kind == PlanKind::Ans ? c.rows * W : c.rows)) return fail(CDM_E_CORRUPT, "root element count != rows");
  if (c.dtype != T_VARBYTES && c.payload_bytes != c.rows * W) return fail(CDM_E_CORRUPT, "payload bytes != rows * width");
  auto bad = [&](const std::string& m) { return fail(CDM_E_CORRUPT, m); };
  auto need_w48 = [&]() { return W == 4 || W == 8; };
  // range-ANS node ni: [words (u16), table (256 x u16 freqs + 12 B per chunk)], params {chunks, chunk bytes, tl}
  auto bind_ans = [&](int ni) -> cdm_status {
    const Node& an = c.nodes[ni];
    uint64_t tn;
    if (!(e = raw_stream(c, t, t.kids[ni][0], 2, &b->ans_w_off, &b->ans_w_n)).empty()) return bad(e);
    if (!(e = raw_stream(c, t, t.kids[ni][1], 1, &b->ans_tab_off, &tn)).empty()) return bad(e);
    b->ans = true;
    b->ans_n = an.n;
    b->ans_nchunks = an.u32_at0();
    b->ans_chunk = an.u32_at4();
    b->ans_tl = an.params[8];
    b->ans_il = an.params[9] ? an.params[9] : 1;
    if (b->ans_il != 1 && b->ans_il != 32) return bad("ANS interleave must be 1 or 32");
    if (b->ans_tl < 8 || b->ans_tl > 15) return bad("ANS table log out of range");
    if (b->ans_tl > 12) return fail(CDM_E_UNSUPPORTED, "ANS table log > 12 (device slot table)");
    if (!b->ans_chunk || b->ans_chunk % 16) return bad("ANS chunk size not a positive multiple of 16");
    if (tn != 512 + (8ull + 4ull * b->ans_il) * b->ans_nchunks) return bad("ANS table size");
    const uint64_t cap = uint64_t(b->ans_nchunks) * b->ans_chunk;
    if (cap < an.n || (an.n && cap - b->ans_chunk >= an.n) || (!an.n && b->ans_nchunks)) return bad("ANS chunk count");
    return CDM_OK;
  };

  switch (b->kind) {
    case PlanKind::RawCopy: {
      uint64_t n;
      if (!(e = raw_stream(c, t, 0, W, &b->raw_off, &n)).empty()) return bad(e);
      break;
    }
    case PlanKind::Fp: {
      if (b->fp_mode == FP_INT) {
        if (!(W == 1 || W == 2 || W == 4 || W == 8)) return fail(CDM_E_UNSUPPORTED, "BitPack output width must be 1/2/4/8");
        if (!(e = bind_bp(c, t, 0, c.rows, 64, &b->main)).empty()) return bad(e);
      } else if (b->fp_mode == FP_DICT) {
        int di = t.kids[0][0], ii = t.kids[0][1];
        uint64_t dn;
        if (!(e = raw_stream(c, t, di, W, &b->dict_off, &dn)).empty()) return bad(e);
        b->entries = r.u32_at0();
        if (r.u32_at4() != W || dn != b->entries) return bad("dictionary shape mismatch");
        if (!(e = bind_bp(c, t, ii, c.rows, 64, &b->main)).empty()) return bad(e);
      } else {
        if (c.dtype != T_F64) return fail(CDM_E_UNSUPPORTED, "Float2Int needs F64 output");
        b->d = r.params[0];
        if (b->d > 22) return bad("Float2Int exponent > 22");
        if (!(e = bind_bp(c, t, t.kids[0][0], c.rows, 64, &b->main)).empty()) return bad(e);
      }
      break;
    }
    case PlanKind::Scan: {
      if (!need_w48()) return fail(CDM_E_UNSUPPORTED, "Delta output width must be 4 or 8");
      b->delta_base = r.u64_at8();
      if (b->fp_mode == FP_DICT) {  // Delta|Dict|[Raw entries (8-byte deltas), BitPack indices]
        const int di = t.kids[0][0];
        const Node& dn = c.nodes[di];
        uint64_t n;
        if (dn.n != c.rows) return bad("Dict child count mismatch");
        if (!(e = raw_stream(c, t, t.kids[di][0], 8, &b->dict_off, &n)).empty()) return bad(e);
        b->entries = dn.u32_at0();
        if (dn.u32_at4() != 8 || n != b->entries) return bad("delta dictionary shape mismatch");
        if (!(e = bind_bp(c, t, t.kids[di][1], c.rows, 64, &b->main)).empty()) return bad(e);
        break;
      }
      if (!(e = bind_bp(c, t, t.kids[0][0], c.rows, 64, &b->main)).empty()) return bad(e);
      break;
    }
    case PlanKind::Rle: {
      if (!need_w48()) return fail(CDM_E_UNSUPPORTED, "RLE output width must be 4 or 8");
      // the value lineage, deepest level first (compile_plan fixed the shape; here: counts and streams)
      std::function<std::string(int, uint64_t, bool)> level = [&](int ni, uint64_t rows, bool top) -> std::string {
        const Node& nd = c.nodes[ni];
        RleLevel L;
        L.n = uint32_t(rows);
        std::string er;
        int vi = -1;
        if (nd.codec == DELTA) {  // Delta | RLE | [BitPack dv, BitPack dc]: arithmetic runs
          L.vmode = V_LINEAR;
          L.delta_base = nd.u64_at8();
          const int ri = t.kids[ni][0];
          const Node& rl = c.nodes[ri];
          if (rl.n != rows) return "Delta child count mismatch";
          L.nruns = rl.u32_at0();
          L.max_run = rl.u32_at4();
          if (!(er = bind_bp(c, t, t.kids[ri][0], L.nruns, 64, &L.val)).empty()) return er;
          if (!(er = bind_bp(c, t, t.kids[ri][1], L.nruns, 32, &L.cnt)).empty()) return er;
        } else {  // RLE or DeltaStride: [values, BitPack counts]
          L.nruns = nd.u32_at0();
          L.max_run = nd.u32_at4();
          if (nd.codec == DSTRIDE) { L.strided = true; L.stride = nd.u64_at8(); }
          vi = t.kids[ni][0];
          const int ci = t.kids[ni][1];
          if (c.nodes[ci].codec == RLE || c.nodes[ci].codec == DSTRIDE || c.nodes[ci].codec == DELTA) {
            // the counts are themselves RLE-family coded: a lower level expands them into a u32 array that this
            // level reads as 32-bit packed counts (FOR 0)
            if (c.nodes[ci].n != L.nruns) return "RLE counts count mismatch";
            if (!(er = level(ci, L.nruns, false)).empty()) return er;
            L.cnt_src = int(b->lv.size()) - 1;
            b->lv.back().as_counts = true;
            L.cnt.n = L.nruns; L.cnt.w = 32; L.cnt.base = 0; L.cnt.off = 0;
          } else if (!(er = bind_bp(c, t, ci, L.nruns, 32, &L.cnt)).empty()) {
            return er;
          }
          const Node& v = c.nodes[vi];
          if (v.n != L.nruns) return "RLE values count mismatch";
          if (v.codec == BITPACK) {
            L.vmode = V_BP;
            if (!(er = bind_bp(c, t, vi, L.nruns, 64, &L.val)).empty()) return er;
          } else if (v.codec == DICT && top) {
            uint64_t dn;
            L.vmode = V_DICT;
            if (!(er = raw_stream(c, t, t.kids[vi][0], W, &b->dict_off, &dn)).empty()) return er;
            b->entries = v.u32_at0();
            if (v.u32_at4() != W || dn != b->entries) return "dictionary shape mismatch";
            if (!(er = bind_bp(c, t, t.kids[vi][1], L.nruns, 64, &L.val)).empty()) return er;
          } else if (v.codec == FLOAT2INT && top) {
            if (c.dtype != T_F64) return "!Float2Int needs F64 output";
            L.vmode = V_F2I;
            b->d = v.params[0];
            if (b->d > 22) return "Float2Int exponent > 22";
            if (!(er = bind_bp(c, t, t.kids[vi][0], L.nruns, 64, &L.val)).empty()) return er;
          } else {  // a lower level produces this level's run values
            L.vmode = V_RAW;
            if (!(er = level(vi, L.nruns, false)).empty()) return er;
            L.val_src = int(b->lv.size()) - 1;
          }
        }
        // rows without runs would leave the level's output unwritten with no tile to notice
        if (L.n && !L.nruns) return "RLE has rows but no runs";
        b->lv.push_back(L);
        return "";
      };
      if (!(e = level(0, c.rows, true)).empty()) {
        if (e[0] == '!') return fail(CDM_E_UNSUPPORTED, e.substr(1));
        return bad(e);
      }
      if (b->lv.size() > 4) return bad("RLE lineage of more than 4 levels");
      break;
    }
    case PlanKind::Ans: {
      cdm_status st = bind_ans(0);
      if (st) return st;
      break;
    }
    case PlanKind::Str: {
      if (c.offsets_bytes != 4 * (c.rows + 1)) return bad("offsets bytes != 4 * (rows + 1)");
      if (c.payload_bytes >= (1ull << 31)) return fail(CDM_E_UNSUPPORTED, "VARBYTES payload >= 2^31 per chunk");
      int bi = t.kids[0][0], li = t.kids[0][1];
      if (!(e = bind_bp(c, t, li, c.rows, 64, &b->main)).empty()) return bad(e);
      const Node& bn = c.nodes[bi];
      if (bn.n != c.payload_bytes) return bad("Str bytes count != payload bytes");
      if (bn.codec == ANS) {
        cdm_status st = bind_ans(bi);
        if (st) return st;
      } else if (bn.codec == STRDICT) {  // [Raw dictionary, BitPack ids (|ANS)]
        b->strdict = true;
        uint64_t dn;
        if (!(e = raw_stream(c, t, t.kids[bi][0], 1, &b->sd_dict_off, &dn)).empty()) return bad(e);
        b->sd_entries = bn.u32_at0();
        const uint32_t dbytes = bn.u32_at4();
        if (dn != 4ull * (b->sd_entries + 1ull) + dbytes) return bad("StrDict dictionary stream size");
        if (dn >= (1ull << 31)) return fail(CDM_E_UNSUPPORTED, "StrDict dictionary >= 2 GiB");
        b->sd_dict_bytes = uint32_t(dn);
        // the kernels trust the offsets: 0, non-decreasing, ending at the token bytes (checked here once)
        const uint8_t* dh = static_cast<const uint8_t*>(job.host_chunk) + b->sd_dict_off;
        if (rd32(dh) != 0 || rd32(dh + 4ull * b->sd_entries) != dbytes) return bad("StrDict dictionary offsets");
        for (uint32_t k = 0; k < b->sd_entries; k++)
          if (rd32(dh + 4ull * k) > rd32(dh + 4ull * k + 4)) return bad("StrDict dictionary offsets decrease");
        const int ii = t.kids[bi][1];
        const Node& in = c.nodes[ii];
        if (in.n >= (1ull << 31)) return fail(CDM_E_UNSUPPORTED, "StrDict tokens >= 2^31 per chunk");
        b->sd_ntok = uint32_t(in.n);
        if (c.payload_bytes && !b->sd_ntok) return bad("StrDict without tokens");
        const int pi = t.kids[ii][0];
        if (c.nodes[pi].codec == ANS) {  // BitPack | ANS: the packed id bytes are entropy coded
          b->sd_w = in.w();
          b->sd_id_base = in.u64_at8();
          if (b->sd_w > 32) return bad("StrDict id width > 32");
          if (c.nodes[pi].n < (uint64_t(b->sd_ntok) * b->sd_w + 7) / 8) return bad("StrDict packed ids too short");
          cdm_status st = bind_ans(pi);
          if (st) return st;
        } else {
          BPB ids;
          if (!(e = bind_bp(c, t, ii, in.n, 32, &ids)).empty()) return bad(e);
          b->sd_ids_off = ids.off; b->sd_w = ids.w; b->sd_id_base = ids.base;
        }
      } else if (bn.codec == LZ4) {
        b->lz4 = true;
        uint64_t pn, tn;
        if (!(e = raw_stream(c, t, t.kids[bi][0], 1, &b->lz_pay_off, &pn)).empty()) return bad(e);
        if (!(e = raw_stream(c, t, t.kids[bi][1], 12, &b->lz_tab_off, &tn)).empty()) return bad(e);
        b->lz_pay_bytes = pn;
        b->n_sub = bn.u32_at0();
        // largest decompressed sub-chunk, read from the host copy of the table (selects the kernel variant)
        const uint8_t* tab = static_cast<const uint8_t*>(job.host_chunk) + b->lz_tab_off;
        for (uint32_t k = 0; k < b->n_sub; k++) {
          b->lz_sub_bytes = std::max(b->lz_sub_bytes, rd32(tab + 12ull * k + 8));
          b->lz_sub_cbytes = std::max(b->lz_sub_cbytes, rd32(tab + 12ull * k + 4));
        }
        // uniform sub-chunks (the encoder's layout): sub-chunk s starts at s * size, no prefix needed
        b->lz_uniform = b->n_sub ? rd32(tab + 8) : 0;
        for (uint32_t k = 0; k + 1 < b->n_sub && b->lz_uniform; k++)
          if (rd32(tab + 12ull * k + 8) != b->lz_uniform) b->lz_uniform = 0;
        if (tn != b->n_sub) return bad("LZ4 table entries != n_sub");
        if (c.payload_bytes && !b->n_sub) return bad("LZ4 without sub-chunks");
      } else {
        uint64_t n;
        if (!(e = raw_stream(c, t, bi, 1, &b->bytes_off, &n)).empty()) return bad(e);
      }
      break;
    }
  }
  if (job.dev_out_bytes == SIZE_MAX) return CDM_OK;  // cdm_chunk_check: host validation only
  // output buffers
  if (b->payload && !job.dev_out) return fail(CDM_E_INVALID_ARG, "dev_out is null");
  if (job.dev_out_bytes < b->payload) return fail(CDM_E_CAPACITY, "dev_out smaller than the payload");
  if (reinterpret_cast<uintptr_t>(job.dev_out) % 16) return fail(CDM_E_INVALID_ARG, "dev_out must be 16-byte aligned");
  if (b->kind == PlanKind::Str) {
    if (!job.dev_offsets || job.dev_offsets_bytes < b->offsets_bytes) return fail(CDM_E_CAPACITY, "dev_offsets too small");
  }
  b->out = job.dev_out;
  b->offs = job.dev_offsets;
  b->dev_chunk = static_cast<const uint8_t*>(job.dev_chunk);
  return CDM_OK;
}

uint64_t div_up(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// ============================================================================ scratch layout
struct Alloc {  // bump allocator over one device arena; pass 1 sizes, pass 2 assigns
  uint8_t* base = nullptr;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += count * sizeof(T);
    return p;
  }
};

}  // namespace

// ============================================================================ device batches
enum Family { F_FP = 0, F_SCAN = 1, F_RLE = 2, F_LZ4 = 3, F_COPY = 4 };
// kernel streams: one per family, plus S_ANS for the range-ANS -> String-dictionary chain, which is independent of
// the LZ4 launches (its times and launches are reported under F_LZ4, the chunk-sequential family)
constexpr int S_ANS = 5, kStreams = 6;
constexpr uint64_t kLz4BigSubs = 65536;  // LZ4 sub-chunks per batch from which LZ4 runs in a phase of its own
constexpr int kBigPhaseMode = 2;  // [LZ4, ANS->String-dictionary] then [FP, scan, RLE, copy]

// Stream priority of a kernel family.  CDM_RLE_PRIO=hi: the latency-bound RLE chain (sums -> scan -> expand)
// gets its CTAs scheduled first and the bandwidth-bound families fill the SMs it leaves idle; lo: the
// reverse (short bandwidth-bound kernels of later pipeline groups are never queued behind RLE CTAs).
static int fam_priority(int f, int lo, int hi) {
  static const int mode = [] {
    const char* v = std::getenv("CDM_RLE_PRIO");
    return v && v[0] == 'h' ? 1 : 0;
  }();
  // (giving the LZ4 stream the highest or the lowest priority under the phased schedule measured the same:
  // config 4 SF 100 device-resident 1229-1231 GB/s)
  if (mode == 1) return f == F_RLE ? hi : lo;
  return f == F_RLE ? lo : hi;
}

// kernel kinds of cdm_batch_kernel_times (include/cdm.h)
enum KernelKind { K_FP = 0, K_SCAN, K_RLE_SUMS, K_RLE_L0, K_RLE_L1, K_RLE_BIG, K_LZ4, K_COPY, K_ANS, K_SD, K_FPC,
                  kKernelKinds };

struct cdm_batch {
  cdm_engine* e = nullptr;
  int device = 0;
  std::vector<Bound> jobs;
  std::vector<FpBatch> fp;
  std::vector<uint32_t> fp_maxw;
  std::vector<uint8_t> fp_char;  // 1: the launch decodes FIXED (CHAR(n)) rows (kernel kind K_FPC)
  // algorithmic bytes per kernel kind (Eq. 1: compressed bytes the kind must read + decoded
  // bytes it must write, summed over the batch's jobs); the RLE chain is booked on K_RLE_L1
  uint64_t k_bytes[kKernelKinds] = {};
  std::vector<ScanBatch> scan;
  std::vector<SumsBatch> sums;
  std::vector<RleBatch> rle;
  std::vector<int> sums_phase;  // per sums batch: -1 = before round 0, r = right after round r's expansions
  std::vector<int> rle_round;   // per rle batch: its round
  size_t rle_level0 = 0;  // rle[0, rle_level0) are launches of the value / counts lineages (non-final rounds)
  std::vector<Lz4Batch> lz4;
  std::vector<uint32_t> lz4_max_sub, lz4_max_csub;
  std::vector<AnsBatch> ans;  // runs on the chunk-sequential (LZ4) family stream
  std::vector<SdBatch> sd;    // String-dictionary expansions, after the ANS launches on the same stream
  struct Copy { void* dst; const void* src; size_t bytes; };
  std::vector<Copy> copies;
  std::vector<void*> zero_offsets;  // VARBYTES with rows == 0: offsets[0] = 0
  uint8_t* arena = nullptr;
  size_t arena_bytes = 0, zero_bytes = 0;
  bool own_arena = true;
  uint32_t* err_dev = nullptr;
  uint32_t* err_host = nullptr;
  bool own_err_host = true;
  bool zeroed_by_caller = false;  // the engine zeroes the scratch prefix before waiting for the copy
  // device-resident batches: the error words are cleared by cdm_batch_results (and at creation), not by a
  // kernel in front of every launch -- the epoch-tagged scan words and self-resetting RLE counters in the
  // zeroed region need no per-launch clearing
  bool sticky_errors = false;
  uint32_t* err_external = nullptr;  // pipelines: error words live in one array shared by all groups
  cudaStream_t* fam = nullptr;     // the family streams concurrent kernel families fork onto
  // fork/join events: independent kernel families run concurrently on the engine's family streams
  cudaEvent_t fork = nullptr;
  cudaEvent_t join[kStreams] = {};
  // timing
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  struct Pending { int fam; cudaEvent_t a, b; };
  std::vector<Pending> pending;
  double fam_ms[5] = {0, 0, 0, 0, 0};
  uint64_t fam_launches[5] = {0, 0, 0, 0, 0};
  int timing_mode = 0;  // 1: events around each kernel family; 2: around each kernel launch
  double k_ms[kKernelKinds] = {};
  uint64_t k_n[kKernelKinds] = {};
  // graph mode (cdm_batch_set_graph): the enqueue is captured once per (stream, timing) and replayed
  bool use_graph = false, capturing = false, graph_pending = false, graph_timing = false;
  int graph_mode = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t gstream = nullptr;
  uint32_t graph_nl = 0;
  uint64_t graph_fam_launches[5] = {0, 0, 0, 0, 0};
  std::vector<Pending> graph_events;
  void drop_graph() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    gexec = nullptr;
    graph = nullptr;
  }
  ~cdm_batch() {
    drop_graph();
    if (fork) cudaEventDestroy(fork);
    for (auto ev : join) if (ev) cudaEventDestroy(ev);
    if (own_arena && arena) cudaFree(arena);
    if (own_err_host && err_host) cudaFreeHost(err_host);
    for (auto ev : ev_pool) cudaEventDestroy(ev);
  }
};

namespace {

bool getenv_flag(const char* name) {
  const char* v = std::getenv(name);
  return v && v[0] == '1';
}

// Build all launch descriptors for `jobs` over an arena laid out by `A` (pass 1: A.base == nullptr).
// Returns the arena bytes; `zero_bytes` = prefix of the arena that must start zeroed.
size_t layout_batch(cdm_batch* B, Alloc& A, size_t* zero_bytes) {
  const size_t nj = B->jobs.size();
  B->fp.clear(); B->fp_maxw.clear(); B->fp_char.clear();
  for (auto& kb : B->k_bytes) kb = 0; B->scan.clear(); B->sums.clear(); B->rle.clear(); B->sums_phase.clear(); B->rle_round.clear(); B->lz4.clear(); B->lz4_max_sub.clear(); B->lz4_max_csub.clear();
  B->ans.clear(); B->sd.clear();
  B->copies.clear(); B->zero_offsets.clear();
  // ---- zeroed region: error words, ticket counters, look-back flags/values, rle big counters
  B->err_dev = B->err_external ? B->err_external : A.take<uint32_t>(nj ? nj : 1);
  std::vector<int> fpj, scj, rlj, lzj, anj, sdj;
  for (size_t i = 0; i < nj; i++) {
    const Bound& b = B->jobs[i];
    switch (b.kind) {
      case PlanKind::Fp: if (b.rows) fpj.push_back(int(i)); break;
      case PlanKind::Scan: if (b.rows) scj.push_back(int(i)); break;
      case PlanKind::Rle:
        if (b.rows) rlj.push_back(int(i));
        break;
      case PlanKind::Str:
        if (b.rows) scj.push_back(int(i)); else B->zero_offsets.push_back(b.offs);
        if (b.lz4 && b.payload) lzj.push_back(int(i));
        if (b.ans && b.payload) anj.push_back(int(i));
        if (b.strdict && b.payload) sdj.push_back(int(i));
        if (!b.lz4 && !b.ans && !b.strdict && b.payload) B->copies.push_back({b.out, b.dev_chunk + b.bytes_off, size_t(b.payload)});
        break;
      case PlanKind::Ans:
        if (b.payload) anj.push_back(int(i));
        break;
      case PlanKind::RawCopy:
        if (b.payload) B->copies.push_back({b.out, b.dev_chunk + b.raw_off, size_t(b.payload)});
        break;
    }
  }
  auto groups = [](const std::vector<int>& v, size_t cap = kMaxBatch) {
    std::vector<std::vector<int>> g;
    for (size_t i = 0; i < v.size(); i += cap)
      g.emplace_back(v.begin() + i, v.begin() + std::min(v.size(), i + cap));
    return g;
  };
  // FP: numeric rows and FIXED (CHAR(n)) rows in separate launches (separate kernel kinds)
  std::vector<int> fp_num, fp_chr;
  for (int j : fpj) (B->jobs[j].casc->dtype == T_FIXED ? fp_chr : fp_num).push_back(j);
  // numeric launches: up to kMaxFpBatch chunks of similar bit width (a launch's staging buffers are sized by its
  // widest stream)
  std::stable_sort(fp_num.begin(), fp_num.end(), [&](int a, int c) { return B->jobs[a].main.w < B->jobs[c].main.w; });
  std::vector<std::vector<int>> fp_groups = groups(fp_num, kMaxFpBatch);
  const size_t n_num_groups = fp_groups.size();
  {  // CHAR(n) launches hold one row width each (the row-group kernel is specialised on it) and one dictionary class
     // (the kernel picks its shared-memory variant by the launch's largest dictionary: o_clerk's 1.5 MB ones must
     // not pull the few-entry ones of the same width off the pre-shifted tables)
    auto cls = [&](int j) {
      const Bound& b = B->jobs[j];
      const uint64_t bytes = uint64_t(b.entries) * b.W;
      return bytes > 16384 ? 0 : b.entries > 128 ? 1 : 2;
    };
    auto key = [&](int j) { return std::make_pair(B->jobs[j].W, cls(j)); };
    std::vector<int> by_w(fp_chr);
    std::stable_sort(by_w.begin(), by_w.end(), [&](int a, int c) { return key(a) < key(c); });
    for (size_t i = 0; i < by_w.size();) {
      size_t k = i;
      while (k < by_w.size() && key(by_w[k]) == key(by_w[i])) k++;
      for (auto& g : groups(std::vector<int>(by_w.begin() + i, by_w.begin() + k), kMaxFpBatch)) fp_groups.push_back(g);
      i = k;
    }
  }
  for (size_t gi = 0; gi < fp_groups.size(); gi++) {
    const auto& g = fp_groups[gi];
    B->fp_char.push_back(gi >= n_num_groups);
    FpBatch fb{};
    fb.err = B->err_dev;
    uint32_t tiles = 0, maxw = 0;
    for (int j : g) {
      const Bound& b = B->jobs[j];
      FpDesc& d = fb.d[fb.n++];
      d.packed = b.dev_chunk + b.main.off;
      d.dict = b.fp_mode == FP_DICT ? b.dev_chunk + b.dict_off : nullptr;
      d.out = b.out;
      d.base = b.main.base;
      d.n = uint32_t(b.rows);
      d.entries = b.entries;
      d.tile0 = tiles;
      d.err_idx = uint32_t(j);
      d.w = uint16_t(b.main.w);
      d.out_bytes = uint16_t(b.W);
      d.mode = b.fp_mode;
      d.d = b.d;
      tiles += uint32_t(div_up(b.rows, kFpTile));
      maxw = std::max(maxw, b.main.w);
    }
    fb.total_tiles = tiles;
    B->fp.push_back(fb);
    B->fp_maxw.push_back(maxw);
  }
  // scan (delta + VARBYTES offsets)
  std::vector<uint32_t> scan_tiles;
  for (auto& g : groups(scj)) {
    ScanBatch sb{};
    sb.err = B->err_dev;
    uint32_t tiles = 0;
    for (int j : g) {
      const Bound& b = B->jobs[j];
      ScanDesc& d = sb.d[sb.n++];
      d.packed = b.dev_chunk + b.main.off;
      d.for_base = b.main.base;
      d.n = uint32_t(b.rows);
      d.tile0 = tiles;
      d.ntiles = uint32_t(div_up(b.rows, kScanTile));
      d.err_idx = uint32_t(j);
      d.w = uint16_t(b.main.w);
      if (b.kind == PlanKind::Str) {
        d.out = b.offs; d.base = b.payload; d.out_bytes = 4; d.mode = SCAN_OFFSETS;
      } else {
        d.out = b.out; d.base = b.delta_base; d.out_bytes = uint8_t(b.W); d.mode = SCAN_DELTA;
        if (b.fp_mode == FP_DICT) {
          d.dict = reinterpret_cast<const uint64_t*>(b.dev_chunk + b.dict_off);
          d.entries = b.entries;
        }
      }
      tiles += d.ntiles;
    }
    sb.total_tiles = tiles;
    sb.ticket = A.take<unsigned long long>(1);
    sb.lb = A.take<uint4>(size_t(tiles) * 3);  // per tile: flag word, AGG values, INC values
    B->scan.push_back(sb);
    scan_tiles.push_back(tiles);
  }
  // RLE units: one per expansion level of each RLE job (deepest first).  A non-final level expands into an
  // L2-resident array that a later level of the job reads: its run values (u64, V_RAW; the value lineage of
  // Delta|RLE or DeltaStride nodes) or its run counts (u32, read as 32-bit packed counts; Table 2's PS_PARTKEY).
  // A level's depth is 1 + the deepest level it reads; units run in rounds by depth, aligned at the end (every
  // job's final level in the last round).  Every unit has its own tile sums / prefixes: rle_sums of a level
  // whose counts are packed in the chunk run before round 0, those of a counts-lineage level right after the
  // round that writes its counts.  Each round's expansions follow the previous launch (PDL-chained).
  struct RleUnit { int job; int level; int round; int sums_phase; bool final; };
  std::vector<RleUnit> units;
  std::vector<int> job_unit0(B->jobs.size(), -1);
  int rounds = 0;
  {
    std::vector<std::vector<int>> depth(B->jobs.size());
    for (int j : rlj) {
      const auto& lv = B->jobs[j].lv;
      auto& dp = depth[j];
      dp.assign(lv.size(), 1);
      for (size_t l = 0; l < lv.size(); l++) {
        if (lv[l].val_src >= 0) dp[l] = std::max(dp[l], dp[lv[l].val_src] + 1);
        if (lv[l].cnt_src >= 0) dp[l] = std::max(dp[l], dp[lv[l].cnt_src] + 1);
      }
      rounds = std::max(rounds, dp.back());
    }
    for (int j : rlj) {
      const auto& lv = B->jobs[j].lv;
      const auto& dp = depth[j];
      const int nl = int(lv.size()), shift = rounds - dp.back();
      job_unit0[j] = int(units.size());
      for (int l = 0; l < nl; l++) {
        const int ph = lv[l].cnt_src >= 0 ? shift + dp[lv[l].cnt_src] - 1 : -1;
        units.push_back({j, l, shift + dp[l] - 1, ph, l == nl - 1});
      }
    }
  }
  auto lvl = [&](int u) -> const RleLevel& { return B->jobs[units[u].job].lv[units[u].level]; };
  auto unit_groups = [&](auto key, int k) {  // unit indices with key(u) == k, <= kMaxBatch per group
    std::vector<std::vector<int>> g;
    for (int u = 0; u < int(units.size()); u++) {
      if (key(u) != k) continue;
      if (g.empty() || g.back().size() == size_t(kMaxBatch)) g.emplace_back();
      g.back().push_back(u);
    }
    return g;
  };
  std::vector<std::pair<int, int>> sums_at(units.size()), rle_at(units.size());  // (batch, desc) per unit
  for (int ph = -1; ph < rounds - 1; ph++) {
    for (auto& g : unit_groups([&](int u) { return units[u].sums_phase; }, ph)) {
      SumsBatch sb{};
      sb.err = B->err_dev;
      uint32_t nunits = 0;
      for (int u : g) {
        const Bound& b = B->jobs[units[u].job];
        const RleLevel& L = lvl(u);
        sums_at[u] = {int(B->sums.size()), int(sb.n)};
        SumsChunk& d = sb.d[sb.n++];
        d.cnt_packed = L.cnt_src >= 0 ? nullptr : b.dev_chunk + L.cnt.off;  // lineage counts: assigned below
        d.cnt_base = L.cnt.base; d.cnt_w = uint16_t(L.cnt.w);
        d.linear = L.vmode == V_LINEAR;
        if (d.linear) { d.dv_packed = b.dev_chunk + L.val.off; d.dv_base = L.val.base; d.dv_w = uint16_t(L.val.w); }
        d.nruns = L.nruns;
        d.rows = L.n;
        d.tiles = uint32_t(div_up(d.nruns, kRleTile));
        d.units = uint32_t(div_up(uint64_t(d.tiles) * kRleTile, 8192));  // rle_sums CTA: 8 warps x 1024 runs
        d.unit0 = nunits;
        d.err_idx = uint32_t(units[u].job);
        nunits += d.units;
      }
      sb.total_units = nunits;
      B->sums.push_back(sb);
      B->sums_phase.push_back(ph);
    }
  }
  for (int round = 0; round < rounds; round++) {
    if (round == rounds - 1) B->rle_level0 = B->rle.size();
    for (auto& g : unit_groups([&](int u) { return units[u].round; }, round)) {
      RleBatch rb{};
      rb.err = B->err_dev;
      uint32_t tiles = 0, slots = 0;
      for (int u : g) {
        const Bound& b = B->jobs[units[u].job];
        const RleLevel& L = lvl(u);
        rle_at[u] = {int(B->rle.size()), int(rb.n)};
        RleDesc& d = rb.d[rb.n++];
        d.cnt_packed = L.cnt_src >= 0 ? nullptr : b.dev_chunk + L.cnt.off;  // lineage counts: assigned below
        d.cnt_base = L.cnt.base; d.cnt_w = uint16_t(L.cnt.w);
        d.val_packed = L.vmode == V_RAW ? nullptr : b.dev_chunk + L.val.off;  // V_RAW: assigned below
        d.val_base = L.val.base;
        d.val_w = uint16_t(L.val.w);
        d.dict = L.vmode == V_DICT ? b.dev_chunk + b.dict_off : nullptr;
        d.entries = b.entries;
        d.d = b.d;
        d.vmode = L.vmode;
        d.strided = L.strided;
        d.stride = L.stride;
        d.delta_base = L.delta_base;
        d.out = units[u].final ? b.out : nullptr;  // non-final: the level's array, assigned below
        d.out_bytes = units[u].final ? uint8_t(b.W) : L.as_counts ? uint8_t(4) : uint8_t(8);
        d.n = L.n;
        d.nruns = L.nruns;
        d.tile0 = tiles;
        d.ntiles = uint32_t(div_up(d.nruns, kRleTile));
        d.err_idx = uint32_t(units[u].job);
        if (d.vmode == V_LINEAR || d.strided) rb.any_linear = 1;
        tiles += d.ntiles;
        slots += d.n / kRleBigLimit + 1;
        // the header's max run bounds a tile's output; only then can rle_big be skipped (a lying header
        // only costs speed: oversize tiles are then expanded in place)
        if (uint64_t(kRleTile) * L.max_run > kRleBigLimit) rb.big_enabled = 1;
      }
      rb.total_tiles = tiles;
      {
        uint64_t rows = 0, runs = 0;
        for (int u : g) { rows += lvl(u).n; runs += lvl(u).nruns; }
        rb.short_runs = runs && rows <= 16 * runs;
      }
      rb.big.counter = A.take<unsigned long long>(1);
      rb.big.done = A.take<uint32_t>(1);
      rb.big.max_slots = slots;
      B->rle.push_back(rb);
      B->rle_round.push_back(round);
    }
  }
  *zero_bytes = (A.off + 15) & ~size_t(15);  // launch_zero works in 16-byte words (the next take pads to 256)
  // ---- non-zeroed region: optional per-tile trace (env CDM_TRACE=<csv path>)
  if (std::getenv("CDM_TRACE")) {
    for (auto& sb : B->scan) sb.trace = A.take<uint64_t>(size_t(sb.total_tiles) * 8);
    for (auto& pb : B->sums) pb.trace = A.take<uint64_t>(size_t(pb.total_units) * 8);
    for (auto& rb : B->rle) rb.trace = A.take<uint64_t>(size_t(rb.total_tiles) * 8);
  }
  // ---- non-zeroed region: scan tile sums (reduce-then-scan), RLE tile sums + prefixes, big-tile slots, lineage
  for (size_t i = 0; i < B->scan.size(); i++) B->scan[i].tsum = A.take<uint64_t>(size_t(scan_tiles[i]) * 8);  // 8: warp tiles per tile (scan_mode 2)
  for (size_t u = 0; u < units.size(); u++) {
    SumsChunk& d = B->sums[sums_at[u].first].d[sums_at[u].second];
    d.tsum = A.take<uint64_t>(size_t(d.tiles + d.units) * 2);  // tile sums, then one sum per rle_sums group
    B->rle[rle_at[u].first].d[rle_at[u].second].tsum = d.tsum;
  }
  for (size_t u = 0; u < units.size(); u++) {  // each non-final level's array, wired to the level that reads it
    if (units[u].final) continue;
    uint64_t* V = A.take<uint64_t>(size_t(lvl(int(u)).n) + 4);
    B->rle[rle_at[u].first].d[rle_at[u].second].out = V;
    const auto& lv = B->jobs[units[u].job].lv;
    for (size_t l = 0; l < lv.size(); l++) {
      const int c = job_unit0[units[u].job] + int(l);
      if (lv[l].val_src == units[u].level)
        B->rle[rle_at[c].first].d[rle_at[c].second].val_packed = reinterpret_cast<const uint8_t*>(V);
      if (lv[l].cnt_src == units[u].level) {
        B->rle[rle_at[c].first].d[rle_at[c].second].cnt_packed = reinterpret_cast<const uint8_t*>(V);
        B->sums[sums_at[c].first].d[sums_at[c].second].cnt_packed = reinterpret_cast<const uint8_t*>(V);
      }
    }
  }
  for (auto& rb : B->rle) {
    rb.big.entries = A.take<RleBig::Entry>(rb.big.max_slots);
    rb.big.soffs = A.take<uint32_t>(size_t(rb.big.max_slots) * (kRleTile + 1));
    rb.big.vals = A.take<uint64_t>(size_t(rb.big.max_slots) * kRleTile);
    rb.big.slopes = A.take<uint64_t>(size_t(rb.big.max_slots) * kRleTile);
  }
  std::vector<const uint8_t*> sd_ids(nj, nullptr);
  // ANS: batches of one interleave each; a tile = kThreads chunks (il = 1) or kThreads/32 chunks (il = 32)
  for (int il : {1, 32}) {
    std::vector<int> sel;
    for (int j : anj) if (B->jobs[j].ans_il == uint32_t(il)) sel.push_back(j);
    for (auto& g : groups(sel, kMaxAnsBatch)) {
      AnsBatch ab{};
      ab.err = B->err_dev;
      uint32_t tiles = 0;
      // il = 32: every CTA builds the slot table once for kThreads/32 * cpw chunks; cpw grows with the batch
      // while the grid still fills the GPU (~64 resident warps per SM)
      uint64_t nch = 0;
      for (int j : g) nch += B->jobs[j].ans_nchunks;
      ab.cpw = il == 32 ? uint32_t(std::min<uint64_t>(8, std::max<uint64_t>(1, nch / (uint64_t(device_sms()) * 64)))) : 1;
      const uint32_t per_tile = il == 32 ? uint32_t(kThreads / 32) * ab.cpw : uint32_t(kThreads);
      for (int j : g) {
        const Bound& b = B->jobs[j];
        AnsDesc& d = ab.d[ab.n++];
        d.words = reinterpret_cast<const uint16_t*>(b.dev_chunk + b.ans_w_off);
        d.table = b.dev_chunk + b.ans_tab_off;
        // a String-dictionary job's ANS node decodes its packed ids into the arena
        if (b.strdict) {
          uint8_t* ids = A.take<uint8_t>(size_t(b.ans_n) + 32);
          sd_ids[j] = ids;
          d.out = ids;
        } else {
          d.out = static_cast<uint8_t*>(b.out);
        }
        d.n = b.ans_n;
        d.n_words = b.ans_w_n;
        d.nchunks = b.ans_nchunks;
        d.chunk = b.ans_chunk;
        d.tl = b.ans_tl;
        d.il = b.ans_il;
        d.tile0 = tiles;
        d.err_idx = uint32_t(j);
        tiles += uint32_t(div_up(b.ans_nchunks, per_tile));
      }
      ab.total_tiles = tiles;
      B->ans.push_back(ab);
    }
  }
  // String-dictionary: one tile per kSdTile tokens; the tile sums (then their prefix) live in the arena
  for (auto& g : groups(sdj, kMaxSdBatch)) {
    SdBatch sb{};
    sb.err = B->err_dev;
    uint32_t tiles = 0, dmax = 0, ctas = 0;
    bool fits = true;
    for (int j : g) {
      const Bound& b = B->jobs[j];
      SdDesc& d = sb.d[sb.n++];
      d.ids_packed = b.ans ? sd_ids[j] : b.dev_chunk + b.sd_ids_off;
      d.dict = b.dev_chunk + b.sd_dict_off;
      d.out = static_cast<uint8_t*>(b.out);
      d.id_base = b.sd_id_base;
      d.ntok = b.sd_ntok;
      d.n_out = uint32_t(b.payload);
      d.entries = b.sd_entries;
      d.w = b.sd_w;
      d.tile0 = tiles;
      d.ntiles = uint32_t(div_up(b.sd_ntok, kSdTile));
      d.cta0 = ctas;
      ctas += uint32_t(div_up(d.ntiles, kSdCtaTiles));
      d.tsum = A.take<uint64_t>(d.ntiles + 1);
      d.err_idx = uint32_t(j);
      tiles += d.ntiles;
      const uint32_t db = uint32_t((b.sd_dict_bytes + 15u) & ~15u) + 16u;  // + the word past the last token byte
      dmax = std::max(dmax, db);
      fits = fits && db <= uint32_t(kSdDictSmem);
    }
    sb.total_tiles = tiles;
    sb.total_ctas = ctas;
    sb.dict_smem = fits ? dmax : 0u;  // else the kernels read the dictionaries through L1
    B->sd.push_back(sb);
  }
  // LZ4
  for (auto& g : groups(lzj, kMaxLz4Batch)) {
    Lz4Batch lb{};
    lb.err = B->err_dev;
    uint32_t subs = 0, max_sub = 0, max_csub = 0;
    for (int j : g) {
      const Bound& b = B->jobs[j];
      max_sub = std::max(max_sub, b.lz_sub_bytes);
      max_csub = std::max(max_csub, b.lz_sub_cbytes);
      Lz4Desc& d = lb.d[lb.n++];
      d.payload = b.dev_chunk + b.lz_pay_off;
      d.table = b.dev_chunk + b.lz_tab_off;
      d.out = static_cast<uint8_t*>(b.out);
      d.payload_bytes = b.lz_pay_bytes;
      d.n = b.payload;
      d.n_sub = b.n_sub;
      d.sub0 = subs;
      d.uniform = b.lz_uniform;
      d.err_idx = uint32_t(j);
      subs += b.n_sub;
    }
    lb.total_subs = subs;
    B->lz4.push_back(lb);
    B->lz4_max_sub.push_back(max_sub);
    B->lz4_max_csub.push_back(max_csub);
  }
  for (size_t i = 0; i < nj; i++) {
    const Bound& b = B->jobs[i];
    auto packed = [](const BPB& p) { return (p.n * p.w + 7) / 8; };
    const uint64_t ans_in = b.ans ? 2 * b.ans_w_n + 512 + (8ull + 4ull * b.ans_il) * b.ans_nchunks : 0;
    switch (b.kind) {
      case PlanKind::Fp:
        B->k_bytes[b.casc->dtype == T_FIXED ? K_FPC : K_FP] +=
            packed(b.main) + uint64_t(b.entries) * (b.fp_mode == FP_DICT ? b.W : 0) + b.payload;
        break;
      case PlanKind::Scan: B->k_bytes[K_SCAN] += packed(b.main) + b.payload + (b.fp_mode == FP_DICT ? 8ull * b.entries : 0); break;
      case PlanKind::Rle: {
        uint64_t in = 0;
        for (const RleLevel& L : b.lv) in += (L.cnt_src >= 0 ? 0 : packed(L.cnt)) + (L.vmode == V_RAW ? 0 : packed(L.val));
        if (b.lv.back().vmode == V_DICT) in += uint64_t(b.entries) * b.W;
        B->k_bytes[K_RLE_L1] += in + b.payload;
        break;
      }
      case PlanKind::Ans: B->k_bytes[K_ANS] += ans_in + b.payload; break;
      case PlanKind::RawCopy: B->k_bytes[K_COPY] += 2 * b.payload; break;
      case PlanKind::Str:
        if (b.rows) B->k_bytes[K_SCAN] += packed(b.main) + b.offsets_bytes;
        if (b.lz4) B->k_bytes[K_LZ4] += b.lz_pay_bytes + 12ull * b.n_sub + b.payload;
        else if (b.strdict) {
          const uint64_t ids = b.ans ? b.ans_n : (uint64_t(b.sd_ntok) * b.sd_w + 7) / 8;
          if (b.ans) B->k_bytes[K_ANS] += ans_in + ids;
          B->k_bytes[K_SD] += ids + b.sd_dict_bytes + b.payload;
        } else if (b.ans) B->k_bytes[K_ANS] += ans_in + b.payload;
        else B->k_bytes[K_COPY] += 2 * b.payload;
        break;
    }
  }
  return A.off + 256;
}

cdm_status batch_build(cdm_batch* B, uint8_t* external_arena, size_t external_bytes) {
  Alloc pass1;
  size_t zb = 0;
  size_t bytes = layout_batch(B, pass1, &zb);
  if (external_arena) {
    if (bytes > external_bytes) return fail(CDM_E_CAPACITY, "scratch arena too small");
    B->arena = external_arena;
    B->own_arena = false;
  } else {
    cudaError_t ce = cudaMalloc(&B->arena, bytes);
    if (ce != cudaSuccess) return fail(CDM_E_OOM, std::string("scratch cudaMalloc: ") + cudaGetErrorString(ce));
    CUDA_TRY(cudaMemset(B->arena, 0, zb));
  }
  B->arena_bytes = bytes;
  B->zero_bytes = zb;
  Alloc pass2;
  pass2.base = B->arena;
  layout_batch(B, pass2, &zb);
  return CDM_OK;
}

cudaEvent_t ev_get(cdm_batch* B, size_t k) {
  while (B->ev_pool.size() <= k) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    B->ev_pool.push_back(e);
  }
  return B->ev_pool[k];
}

cdm_status batch_enqueue(cdm_batch* B, cudaStream_t s, uint32_t* nl) {
  uint32_t n = 0;
  size_t evk = B->pending.size() * 2;
  const bool has[kStreams] = {!B->fp.empty(), !B->scan.empty(), !B->rle.empty(), !B->lz4.empty(),
                              !B->copies.empty() || !B->zero_offsets.empty(), !B->ans.empty() || !B->sd.empty()};
  int nfam = 0;
  for (bool h : has) nfam += h;
  // error words, tickets, look-back words and counters start at zero (one tiny kernel, not a memset)
  if (!B->zeroed_by_caller && !B->sticky_errors) CUDA_TRY(launch_zero(B->arena, B->zero_bytes, s));
  // fork: with several families each runs on its own stream (the latency-bound scan/RLE chains overlap
  // the bandwidth-bound FP kernel); a single family stays on `s`
  static const bool serial = std::getenv("CDM_SERIAL") != nullptr;
  // the RLE family always forks: its stream has the lowest priority, so the short bandwidth-bound kernels
  // of later groups (and the engine's bookkeeping kernels) get SMs as soon as an RLE CTA retires
  // per-kernel timing (mode 2) runs the families one after another, so each launch's events time it alone
  const bool fork = (nfam > 1 || has[F_RLE]) && B->fam && !serial && !(B->timing && B->timing_mode == 2);
  if (fork && !B->fork) {
    CUDA_TRY(cudaEventCreateWithFlags(&B->fork, cudaEventDisableTiming));
    for (auto& ev : B->join) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  // phases: the families of one phase run concurrently, phases one after another.  A throughput-bound LZ4
  // launch (>= kLz4BigSubs sub-chunks: its threads hold the SMs for the whole launch and re-read their match
  // windows from DRAM) slows every family running beside it, so big batches give it a phase of its own
  // (config 4, SF 30, device-resident: one phase 854 GB/s, all serial 1090, [LZ4 + ANS/String-dictionary] then
  // [FP, scan, RLE] 1149); small batches keep one phase (SF 1 / 3: one phase 706 / 707 vs serial 542 / 654)
  static const int phase_mode = std::getenv("CDM_PHASES") ? std::atoi(std::getenv("CDM_PHASES")) : -1;
  uint64_t lz4_subs = 0;
  for (const auto& lb : B->lz4) lz4_subs += lb.total_subs;
  int mode = phase_mode >= 0 ? phase_mode : (lz4_subs >= kLz4BigSubs ? kBigPhaseMode : 0);
  int phase[kStreams] = {0, 0, 0, 0, 0, 0};
  switch (mode) {
    case 1: phase[F_LZ4] = 0; phase[F_FP] = phase[F_SCAN] = phase[F_RLE] = phase[F_COPY] = phase[S_ANS] = 1; break;
    case 2: phase[F_LZ4] = phase[S_ANS] = 0; phase[F_FP] = phase[F_SCAN] = phase[F_RLE] = phase[F_COPY] = 1; break;
    case 3: phase[F_FP] = phase[F_SCAN] = phase[F_RLE] = phase[F_COPY] = 0; phase[F_LZ4] = phase[S_ANS] = 1; break;
    case 4: phase[F_FP] = phase[F_SCAN] = phase[F_RLE] = phase[F_COPY] = phase[S_ANS] = 0; phase[F_LZ4] = 1; break;
    default: break;
  }
  for (int ph = 0; ph < 2; ph++) {
  if (fork) CUDA_TRY(cudaEventRecord(B->fork, s));
  for (int fam = 0; fam < kStreams; fam++) {
    if (!has[fam] || phase[fam] != ph) continue;
    const int acct = fam == S_ANS ? F_LZ4 : fam;  // the family the times and launches are reported under
    cudaStream_t fs = fork ? B->fam[fam] : s;
    if (fork) CUDA_TRY(cudaStreamWaitEvent(fs, B->fork, 0));
    cudaEvent_t ta = nullptr;
    // (in a graph capture the timing events become external event-record nodes, re-recorded by every replay)
    const unsigned evflags = B->capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
    const bool fam_t = B->timing && B->timing_mode != 2, ker_t = B->timing && B->timing_mode == 2;
    if (fam_t) { ta = ev_get(B, evk++); CUDA_TRY(cudaEventRecordWithFlags(ta, fs, evflags)); }
    // one launch, bracketed by its own events in per-kernel timing mode (which serialises PDL pairs)
    auto timed = [&](int kind, auto&& launch) -> cdm_status {
      cudaEvent_t ka = nullptr;
      if (ker_t) { ka = ev_get(B, evk++); CUDA_TRY(cudaEventRecordWithFlags(ka, fs, evflags)); }
      CUDA_TRY(launch());
      if (ker_t) {
        cudaEvent_t kb = ev_get(B, evk++);
        CUDA_TRY(cudaEventRecordWithFlags(kb, fs, evflags));
        B->pending.push_back({100 + kind, ka, kb});
      }
      return CDM_OK;
    };
    cdm_status st = CDM_OK;
    switch (fam) {
      case F_FP:
        for (size_t i = 0; i < B->fp.size() && !st; i++) {
          st = timed(B->fp_char[i] ? K_FPC : K_FP, [&] { return launch_fp(B->fp[i], B->fp_maxw[i], fs); });
          n++; B->fam_launches[F_FP]++;
        }
        break;
      case F_SCAN:
        for (size_t i = 0; i < B->scan.size() && !st; i++) {
          st = timed(K_SCAN, [&] { return launch_scan(B->scan[i], fs); });
          n++; B->fam_launches[F_SCAN]++;
        }
        break;
      case F_RLE: {
        // sums -> expand, round by round (lineage rounds first); the expansions are programmatically dependent
        // launches; a counts-lineage level's sums follow the round that wrote its counts
        size_t si = 0;
        auto sums_upto = [&](int phase) {
          for (; si < B->sums.size() && B->sums_phase[si] <= phase && !st; si++) {
            st = timed(K_RLE_SUMS, [&] { return launch_rle_sums(B->sums[si], fs); });
            n++; B->fam_launches[F_RLE]++;
          }
        };
        sums_upto(-1);
        for (size_t i = 0; i < B->rle.size() && !st; i++) {
          auto& rb = B->rle[i];
          st = timed(i < B->rle_level0 ? K_RLE_L0 : K_RLE_L1, [&] { return launch_rle(rb, fs); });
          n++; B->fam_launches[F_RLE]++;
          if (rb.big_enabled && !st) {
            st = timed(K_RLE_BIG, [&] { return launch_rle_big(rb, fs); });
            n++; B->fam_launches[F_RLE]++;
          }
          if (i + 1 == B->rle.size() || B->rle_round[i + 1] != B->rle_round[i]) sums_upto(B->rle_round[i]);
        }
        break;
      }
      case F_LZ4:  // the chunk-sequential family: LZ4 here, range ANS (+ String-dictionary) on S_ANS
        for (size_t i = 0; i < B->lz4.size() && !st; i++) {
          st = timed(K_LZ4, [&] { return launch_lz4(B->lz4[i], B->lz4_max_sub[i], B->lz4_max_csub[i], fs); });
          n++; B->fam_launches[F_LZ4]++;
        }
        break;
      case S_ANS:
        for (size_t i = 0; i < B->ans.size() && !st; i++) {
          st = timed(K_ANS, [&] { return launch_ans(B->ans[i], B->ans[i].n && B->ans[i].d[0].il == 32, fs); });
          n++; B->fam_launches[F_LZ4]++;
        }
        for (size_t i = 0; i < B->sd.size() && !st; i++) {  // after the ANS launches that feed them
          st = timed(K_SD, [&] { return launch_strdict(B->sd[i], fs); });
          n += 3; B->fam_launches[F_LZ4] += 3;
        }
        break;
      case F_COPY:
        st = timed(K_COPY, [&] {
          for (auto& c : B->copies) {
            cudaError_t ce = cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyDeviceToDevice, fs);
            if (ce != cudaSuccess) return ce;
            B->fam_launches[F_COPY]++;
          }
          for (void* p : B->zero_offsets) {
            cudaError_t ce = cudaMemsetAsync(p, 0, 4, fs);
            if (ce != cudaSuccess) return ce;
          }
          return cudaSuccess;
        });
        break;
    }
    if (st) return st;
    if (fam_t) {
      cudaEvent_t tb = ev_get(B, evk++);
      CUDA_TRY(cudaEventRecordWithFlags(tb, fs, evflags));
      B->pending.push_back({acct, ta, tb});
    }
    if (fork) {
      CUDA_TRY(cudaEventRecord(B->join[fam], fs));
      CUDA_TRY(cudaStreamWaitEvent(s, B->join[fam], 0));
    }
  }
  }
  if (nl) *nl = n;
  return CDM_OK;
}

void fill_results(const cdm_batch* B, const uint32_t* errw, cdm_result* res) {
  for (size_t i = 0; i < B->jobs.size(); i++) {
    const Bound& b = B->jobs[i];
    cdm_result& r = res[i];
    r.rows = b.rows;
    r.payload_bytes = b.payload;
    r.offsets_bytes = b.offsets_bytes;
    r.compressed_bytes = b.total;
    r.chunk_id = b.chunk_id;
    r.error_bits = errw[i];
    r.status = errw[i] ? CDM_E_CORRUPT : CDM_OK;
  }
}

}  // namespace

// ============================================================================ engine
struct cdm_engine {
  int device = 0;
  cudaStream_t copy = nullptr, decode = nullptr;
  bool own_copy = false, own_decode = false;
  cdm_engine_opts opts{};
  struct Slot {
    uint8_t* dev = nullptr;
    cudaEvent_t copied = nullptr, freed = nullptr;
    bool used = false;
    uint8_t* arena = nullptr;  // decode scratch of the group held by this slot
    size_t arena_bytes = 0;
    // decode + family streams of this slot: groups in different slots decode concurrently (a latency-bound
    // RLE group does not hold back the bandwidth-bound group behind it); shared when the user passed one
    cudaStream_t ds = nullptr;
    cudaStream_t fam[kStreams] = {};
    bool own_streams = false;
  };
  std::vector<Slot> slots;
  uint32_t next_slot = 0;
  struct Group {  // chunks copied + decoded together from one slot
    cudaEvent_t done = nullptr;
    uint32_t err_pos = 0, njobs = 0, pending = 0;
    bool harvested = false;
  };
  struct Ticket {
    cdm_result res{};
    uint64_t group = 0;
    uint32_t index = 0;  // position in the group
  };
  std::map<uint64_t, Group> groups;
  std::map<uint64_t, Ticket> tickets;
  uint64_t next_ticket = 1, next_group = 1;
  std::vector<cudaEvent_t> event_pool;
  cudaStream_t fam[kStreams] = {};  // concurrent kernel families
  uint32_t* err_host = nullptr;  // pinned (mapped) ring of per-chunk error words
  uint32_t* err_mapped = nullptr;  // its device alias: harvest_kernel stores there
  uint32_t err_ring = 0, err_next = 0;
  std::map<uint32_t, uint64_t> err_owner;  // ring start position -> group whose words live there
  // H9 checksums (opts.flags & CDM_ENGINE_CHECKSUM): per job, accumulated on the device, copied to pinned
  // host memory at the end of its group (same ring positions as the error words)
  bool checksum = false;
  uint64_t* cs_dev = nullptr;
  uint64_t* cs_host = nullptr;
  cudaEvent_t complete = nullptr;  // recorded once at creation: an event that has always completed
  // NEXT-4 multi-link ingestion (cdm_engine_set_ingest; Vortex): groups are copied H2D over the
  // PCIe links of these devices, in turn, into a staging buffer on that device, then peer-copied (NVLink) into
  // the engine's staging slot.  Empty: every copy goes over the engine device's own link.
  struct Ingest {
    int device = 0;
    cudaStream_t stream = nullptr;       // on `device`: H2D copy, then the peer copy (ordered)
    uint8_t* buf = nullptr;              // on `device`: one group's chunks (slot_bytes)
    std::vector<cudaEvent_t> copied;     // on `device`, one per engine slot: the slot's data has arrived
  };
  std::vector<Ingest> ingest;
  uint64_t ingest_rr = 0;
  uint64_t kernel_launches = 0;  // kernels enqueued by cdm_submit* (decode kernels, checksums, harvests)
  // submit / wait / synchronize / ticket_event are serialised by this mutex (PAPER.md:207-208's submit path
  // may be driven by several host threads); a wait blocks on its group's event with the mutex released
  std::mutex mu;
};


static cdm_status harvest_group(cdm_engine* e, uint64_t gid) {
  auto it = e->groups.find(gid);
  if (it == e->groups.end()) return CDM_OK;
  cdm_engine::Group& g = it->second;
  if (g.harvested) return CDM_OK;
  CUDA_TRY(cudaEventSynchronize(g.done));
  for (auto& kv : e->tickets)
    if (kv.second.group == gid) {
      const uint32_t w = e->err_host[g.err_pos + kv.second.index];
      kv.second.res.error_bits = w;
      kv.second.res.checksum = e->checksum ? e->cs_host[g.err_pos + kv.second.index] : 0ull;
      kv.second.res.status = w ? CDM_E_CORRUPT : CDM_OK;
    }
  g.harvested = true;
  e->event_pool.push_back(g.done);
  g.done = nullptr;
  e->err_owner.erase(g.err_pos);
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_engine_create(int device, const cdm_engine_opts* opts, cdm_engine** out) {
  if (!out) return fail(CDM_E_INVALID_ARG, "null out");
  auto e = std::make_unique<cdm_engine>();
  e->device = device;
  cdm_engine_opts o{};
  if (opts) o = *opts;
  if (o.n_slots == 0) o.n_slots = 4;
  if (o.n_slots < 2) return fail(CDM_E_INVALID_ARG, "n_slots must be >= 2");
  if (o.slot_bytes == 0) o.slot_bytes = 64ull << 20;
  if (o.pcie_gbps <= 0) o.pcie_gbps = 55.0;
  if (o.decode_gbps <= 0) o.decode_gbps = 5000.0;
  e->opts = o;
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(cudaFree(nullptr));  // create the context
  if (o.copy_stream) e->copy = static_cast<cudaStream_t>(o.copy_stream);
  else { CUDA_TRY(cudaStreamCreateWithFlags(&e->copy, cudaStreamNonBlocking)); e->own_copy = true; }
  if (o.decode_stream) e->decode = static_cast<cudaStream_t>(o.decode_stream);
  else { CUDA_TRY(cudaStreamCreateWithFlags(&e->decode, cudaStreamNonBlocking)); e->own_decode = true; }
  int prio_lo = 0, prio_hi = 0;  // numerically: least (lowest) and greatest (highest) priority
  CUDA_TRY(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  auto make_fams = [&](cudaStream_t* fam) -> cudaError_t {
    for (int f = 0; f < kStreams; f++) {
      cudaError_t ce = cudaStreamCreateWithPriority(&fam[f], cudaStreamNonBlocking, fam_priority(f, prio_lo, prio_hi));
      if (ce != cudaSuccess) return ce;
    }
    return cudaSuccess;
  };
  CUDA_TRY(make_fams(e->fam));
  e->slots.resize(o.n_slots);
  for (auto& s : e->slots) {
    if (o.decode_stream) {  // the caller's decode stream orders every group
      s.ds = e->decode;
      for (int f = 0; f < kStreams; f++) s.fam[f] = e->fam[f];
    } else {
      CUDA_TRY(cudaStreamCreateWithPriority(&s.ds, cudaStreamNonBlocking, prio_hi));
      CUDA_TRY(make_fams(s.fam));
      s.own_streams = true;
    }
    if (cudaMalloc(&s.dev, o.slot_bytes) != cudaSuccess) return fail(CDM_E_OOM, "staging slot cudaMalloc failed");
    CUDA_TRY(cudaEventCreateWithFlags(&s.copied, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&s.freed, cudaEventDisableTiming));
  }
  e->err_ring = 4096;
  CUDA_TRY(cudaHostAlloc(&e->err_host, sizeof(uint32_t) * e->err_ring, cudaHostAllocMapped));
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->err_mapped), e->err_host, 0));
  e->checksum = (o.flags & CDM_ENGINE_CHECKSUM) != 0;
  if (e->checksum) {
    if (cudaMalloc(&e->cs_dev, sizeof(uint64_t) * e->err_ring) != cudaSuccess)
      return fail(CDM_E_OOM, "checksum ring cudaMalloc failed");
    CUDA_TRY(cudaHostAlloc(&e->cs_host, sizeof(uint64_t) * e->err_ring, cudaHostAllocDefault));
  }
  CUDA_TRY(cudaEventCreateWithFlags(&e->complete, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(e->complete, e->copy));
  CUDA_TRY(cudaEventSynchronize(e->complete));
  *out = e.release();
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_engine_destroy(cdm_engine* e) {
  if (!e) return CDM_OK;
  cudaSetDevice(e->device);
  cudaStreamSynchronize(e->copy);
  cudaStreamSynchronize(e->decode);
  for (auto& kv : e->groups) if (kv.second.done) cudaEventDestroy(kv.second.done);
  for (auto ev : e->event_pool) cudaEventDestroy(ev);
  for (auto& s : e->slots) {
    if (s.own_streams) {
      cudaStreamSynchronize(s.ds);
      cudaStreamDestroy(s.ds);
      for (auto fs : s.fam) { cudaStreamSynchronize(fs); cudaStreamDestroy(fs); }
    }
    cudaFree(s.dev);
    cudaFree(s.arena);
    cudaEventDestroy(s.copied);
    cudaEventDestroy(s.freed);
  }
  if (e->err_host) cudaFreeHost(e->err_host);
  if (e->cs_dev) cudaFree(e->cs_dev);
  if (e->cs_host) cudaFreeHost(e->cs_host);
  if (e->complete) cudaEventDestroy(e->complete);
  for (auto& ig : e->ingest) {
    cudaSetDevice(ig.device);
    if (ig.stream) { cudaStreamSynchronize(ig.stream); cudaStreamDestroy(ig.stream); }
    if (ig.buf) cudaFree(ig.buf);
    for (auto ev : ig.copied) if (ev) cudaEventDestroy(ev);
  }
  cudaSetDevice(e->device);
  for (auto fs : e->fam) if (fs) { cudaStreamSynchronize(fs); cudaStreamDestroy(fs); }
  if (e->own_copy) cudaStreamDestroy(e->copy);
  if (e->own_decode) cudaStreamDestroy(e->decode);
  delete e;
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_chunk_info(const void* host_chunk, size_t bytes, cdm_result* out) {
  if (!out) return fail(CDM_E_INVALID_ARG, "null out");
  Chunk c;
  std::string e = parse_chunk(host_chunk, bytes, &c);
  if (!e.empty()) return fail(CDM_E_CORRUPT, e);
  std::memset(out, 0, sizeof *out);
  out->rows = c.rows;
  out->payload_bytes = c.payload_bytes;
  out->offsets_bytes = c.offsets_bytes;
  out->compressed_bytes = c.total_bytes;
  out->chunk_id = c.chunk_id;
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_chunk_check(const cdm_cascade* c, const void* host_chunk, size_t bytes) {
  if (!c || !host_chunk) return fail(CDM_E_INVALID_ARG, "null argument");
  cdm_job job{};
  job.cascade = c;
  job.host_chunk = host_chunk;
  job.chunk_bytes = bytes;
  job.dev_out_bytes = SIZE_MAX;
  Bound b;
  return bind_job(job, &b);
}

// H4: one group = consecutive jobs copied into one staging slot (a single H2D copy when their host bytes
// are contiguous) and decoded by one multi-chunk batch after the copy's event.  The copy stream waits on
// the slot's `freed` event, so copies of later groups run ahead of decodes without host stalls.
struct PendingGroup {
  uint32_t slot = 0;
  std::vector<Bound> bs;
  std::vector<const cdm_job*> js;
  cudaEvent_t copied = nullptr;  // the event the decode waits on (the slot's, or an ingest device's)
};

// Phase 1: enqueue the group's H2D copies into its slot (copy stream) and record the slot's `copied` event.
static cdm_status group_copy(cdm_engine* e, PendingGroup& pg) {
  const uint32_t si = e->next_slot;
  e->next_slot = (e->next_slot + 1) % uint32_t(e->slots.size());
  pg.slot = si;
  cdm_engine::Slot& s = e->slots[si];
  // NEXT-4: the copy runs over an ingest device's PCIe link into its buffer, then over NVLink into the slot
  cdm_engine::Ingest* ig = e->ingest.empty() ? nullptr : &e->ingest[e->ingest_rr++ % e->ingest.size()];
  cudaStream_t cs = ig ? ig->stream : e->copy;
  uint8_t* const base = ig ? ig->buf : s.dev;
  if (ig) CUDA_TRY(cudaSetDevice(ig->device));
  if (s.used) CUDA_TRY(cudaStreamWaitEvent(cs, s.freed, 0));  // (a cross-device wait for an ingest device)
  auto& bs = pg.bs;
  auto& js = pg.js;
  // Lay the chunks out in the slot in host-address order: exactly contiguous host neighbours keep their
  // relative offsets and share one H2D copy (if the driver rejects a copy spanning two host allocations,
  // the run is copied chunk by chunk).  Decode order inside the batch does not depend on this layout.
  std::vector<size_t> by_addr(bs.size());
  std::iota(by_addr.begin(), by_addr.end(), size_t(0));
  std::sort(by_addr.begin(), by_addr.end(), [&](size_t a, size_t b) { return js[a]->host_chunk < js[b]->host_chunk; });
  size_t pos = 0, k = 0;
  while (k < by_addr.size()) {
    const size_t first = by_addr[k];
    const uint8_t* h0 = static_cast<const uint8_t*>(js[first]->host_chunk);
    pos = (pos + 255) & ~size_t(255);
    bs[first].dev_chunk = s.dev + pos;
    size_t end = bs[first].total;
    size_t m = k + 1;
    while (m < by_addr.size()) {
      const size_t j = by_addr[m];
      // the appended chunk lands at pos + end: only a run whose running length is a 16-byte multiple keeps
      // it 16-byte aligned (TMA bulk copies and vector loads read its streams in place)
      if (static_cast<const uint8_t*>(js[j]->host_chunk) != h0 + end || end % 16 ||
          pos + end + bs[j].total > e->opts.slot_bytes)
        break;
      bs[j].dev_chunk = s.dev + pos + end;
      end += bs[j].total;
      m++;
    }
    if (pos + end > e->opts.slot_bytes) { if (ig) cudaSetDevice(e->device); return fail(CDM_E_CAPACITY, "group larger than a staging slot"); }
    cudaError_t ce = cudaMemcpyAsync(base + pos, h0, end, cudaMemcpyHostToDevice, cs);
    if (ce == cudaErrorInvalidValue && m > k + 1) {
      cudaGetLastError();
      for (size_t q = k; q < m; q++) {
        const size_t j = by_addr[q];
        ce = cudaMemcpyAsync(base + (bs[j].dev_chunk - s.dev), js[j]->host_chunk, bs[j].total,
                             cudaMemcpyHostToDevice, cs);
        if (ce != cudaSuccess) break;
      }
    }
    if (ce != cudaSuccess) {
      if (ig) cudaSetDevice(e->device);
      return fail(CDM_E_CUDA, std::string("H2D copy: ") + cudaGetErrorString(ce));
    }
    pos += end;
    k = m;
  }
  if (ig) {  // the group's bytes: ingest device -> engine device (NVLink peer copy; a D2D copy for the device itself)
    cudaError_t ce = cudaMemcpyPeerAsync(s.dev, e->device, ig->buf, ig->device, pos, cs);
    if (ce == cudaSuccess) ce = cudaEventRecord(ig->copied[si], cs);
    cudaSetDevice(e->device);
    if (ce != cudaSuccess) return fail(CDM_E_CUDA, std::string("ingest peer copy: ") + cudaGetErrorString(ce));
    pg.copied = ig->copied[si];
  } else {
    CUDA_TRY(cudaEventRecord(s.copied, e->copy));
    pg.copied = s.copied;
  }
  s.used = true;
  return CDM_OK;
}

// Phase 2: the decode stream waits for the copy, runs the group's fused kernels, reads back the error words.
static cdm_status group_decode(cdm_engine* e, PendingGroup& pg, uint64_t* tickets_out) {
  cdm_engine::Slot& s = e->slots[pg.slot];
  auto& bs = pg.bs;
  auto batch = std::make_unique<cdm_batch>();
  batch->e = e;
  batch->device = e->device;
  batch->fam = s.fam;
  for (auto& b : bs) batch->jobs.push_back(b);
  Alloc sizing;
  size_t zb = 0;
  size_t need = layout_batch(batch.get(), sizing, &zb);
  if (need > s.arena_bytes) {
    if (s.arena) { CUDA_TRY(cudaStreamSynchronize(s.ds)); cudaFree(s.arena); s.arena = nullptr; }
    size_t cap = std::max(need, size_t(1) << 20);
    if (cudaMalloc(&s.arena, cap) != cudaSuccess) return fail(CDM_E_OOM, "scratch cudaMalloc failed");
    s.arena_bytes = cap;
  }
  cdm_status st = batch_build(batch.get(), s.arena, s.arena_bytes);
  if (st) return st;
  // fresh error words / counters for this group, zeroed while the group's copy is still in flight
  CUDA_TRY(launch_zero(s.arena, batch->zero_bytes, s.ds));
  batch->zeroed_by_caller = true;
  CUDA_TRY(cudaStreamWaitEvent(s.ds, pg.copied ? pg.copied : s.copied, 0));
  uint32_t nl = 0;
  st = batch_enqueue(batch.get(), s.ds, &nl);
  if (st) return st;
  e->kernel_launches += nl + 2;  // + zero + harvest
  // pinned error words for this group (contiguous ring slice; an old group still there is harvested)
  const uint32_t nj = uint32_t(bs.size());
  if (nj > e->err_ring) return fail(CDM_E_CAPACITY, "too many chunks in one group");
  if (e->err_next + nj > e->err_ring) e->err_next = 0;
  const uint32_t ep = e->err_next;
  e->err_next += nj;
  for (auto it = e->err_owner.begin(); it != e->err_owner.end();) {
    const uint32_t p0 = it->first;
    const auto& g = e->groups[it->second];
    if (p0 < ep + nj && p0 + g.njobs > ep) {
      const uint64_t gid = it->second;
      ++it;
      st = harvest_group(e, gid);
      if (st) return st;
    } else {
      ++it;
    }
  }
  if (e->checksum) {  // H9: positional checksum of every decoded chunk (payload, then offsets under id ^ 2^63)
    CUDA_TRY(cudaMemsetAsync(e->cs_dev + ep, 0, sizeof(uint64_t) * nj, s.ds));
    for (uint32_t j = 0; j < nj; j++) {
      const Bound& b = bs[j];
      if (b.payload) { CUDA_TRY(launch_checksum(b.out, b.payload, b.chunk_id, e->cs_dev + ep + j, s.ds)); e->kernel_launches++; }
      if (b.offs && b.offsets_bytes) {
        CUDA_TRY(launch_checksum(b.offs, b.offsets_bytes, b.chunk_id ^ (1ull << 63), e->cs_dev + ep + j, s.ds));
        e->kernel_launches++;
      }
    }
    CUDA_TRY(cudaMemcpyAsync(e->cs_host + ep, e->cs_dev + ep, sizeof(uint64_t) * nj, cudaMemcpyDeviceToHost, s.ds));
  }
  CUDA_TRY(launch_harvest(batch->err_dev, e->err_mapped + ep, nj, s.ds));
  CUDA_TRY(cudaEventRecord(s.freed, s.ds));
  const uint64_t gid = e->next_group++;
  cdm_engine::Group& g = e->groups[gid];
  if (!e->event_pool.empty()) { g.done = e->event_pool.back(); e->event_pool.pop_back(); }
  else CUDA_TRY(cudaEventCreateWithFlags(&g.done, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(g.done, s.ds));
  g.err_pos = ep;
  g.njobs = nj;
  g.pending = nj;
  e->err_owner[ep] = gid;
  for (uint32_t j = 0; j < nj; j++) {
    const uint64_t id = e->next_ticket++;
    cdm_engine::Ticket& t = e->tickets[id];
    t.group = gid;
    t.index = j;
    t.res.rows = bs[j].rows;
    t.res.payload_bytes = bs[j].payload;
    t.res.offsets_bytes = bs[j].offsets_bytes;
    t.res.compressed_bytes = bs[j].total;
    t.res.chunk_id = bs[j].chunk_id;
    tickets_out[j] = id;
  }
  return CDM_OK;
}

static cdm_status submit_group(cdm_engine* e, std::vector<Bound>& bs, const std::vector<const cdm_job*>& js,
                               uint64_t* tickets_out) {
  PendingGroup pg;
  pg.bs = bs;
  pg.js = js;
  cdm_status st = group_copy(e, pg);
  if (st) return st;
  return group_decode(e, pg, tickets_out);
}

extern "C" CDM_API cdm_status cdm_submit(cdm_engine* e, const cdm_job* job, uint64_t* ticket) {
  if (!e || !job || !ticket) return fail(CDM_E_INVALID_ARG, "null argument");
  std::lock_guard<std::mutex> lock(e->mu);
  CUDA_TRY(cudaSetDevice(e->device));
  std::vector<Bound> bs(1);
  cdm_status st = bind_job(*job, &bs[0]);
  if (st) return st;
  if (bs[0].total > e->opts.slot_bytes) return fail(CDM_E_CAPACITY, "chunk larger than a staging slot");
  return submit_group(e, bs, {job}, ticket);
}

// Relative decode rate of a bound job's kernel family (measured on B200, config 2/3 bench lines): the
// Johnson cost d_i must rank a Delta|RLE chunk (latency-bound expansion) above a Dict|BitPack chunk of
// the same decoded size, or the slowest decode lands at the end of the pipeline.
static double family_rate(const Bound& b) {
  // relative single-chunk decode rates (measured on B200): a chunk-sequential LZ4 / ANS chunk decodes as one
  // chain per sub-chunk, so ONE column chunk is latency bound (~40 GB/s for 16 KiB LZ4 sub-chunks, ~8 GB/s
  // for 4 KiB ANS chunks) -- Johnson's rule then issues those decode-heavy chunks first, and the pipeline
  // ends on short element-parallel decodes instead of a long chain
  switch (b.kind) {
    case PlanKind::Fp: return 1.0;
    case PlanKind::Scan: return 0.5;
    case PlanKind::Rle: return 0.125;
    case PlanKind::Str: return b.lz4 ? 0.008 : b.ans ? (b.ans_il == 32 ? 0.05 : 0.002) : b.strdict ? 0.25 : 0.5;
    case PlanKind::Ans: return b.ans_il == 32 ? 0.05 : 0.002;
    case PlanKind::RawCopy: return 1.0;
  }
  return 1.0;
}

// H3: Johnson's rule on (t_i = compressed / PCIe, d_i = decoded / decode rate):
// jobs with t <= d first ascending t, then the rest descending d; ties by submission index.
static void johnson(const double* tt, const double* dd, size_t n, std::vector<size_t>* order) {
  std::vector<size_t> first, second;
  for (size_t i = 0; i < n; i++) (tt[i] <= dd[i] ? first : second).push_back(i);
  std::stable_sort(first.begin(), first.end(), [&](size_t a, size_t b) { return tt[a] < tt[b]; });
  std::stable_sort(second.begin(), second.end(), [&](size_t a, size_t b) { return dd[a] > dd[b]; });
  *order = first;
  order->insert(order->end(), second.begin(), second.end());
}

extern "C" CDM_API cdm_status cdm_johnson_order(const double* t, const double* d, size_t n, size_t* order) {
  if (n && (!t || !d || !order)) return fail(CDM_E_INVALID_ARG, "null argument");
  std::vector<size_t> o;
  johnson(t, d, n, &o);
  for (size_t i = 0; i < n; i++) order[i] = o[i];
  return CDM_OK;
}

// H3 + H4 planning shared by cdm_submit_batch and cdm_pipeline_create: bind every job, order them by
// Johnson's rule, cut the order into groups (each group = one staging region + one multi-chunk batch).
static cdm_status plan_groups(cdm_engine* e, const cdm_job* jobs, size_t n, uint64_t cap_bytes,
                              std::vector<PendingGroup>* groups_out, std::vector<size_t>* order_out,
                              std::vector<size_t>* first_job_out) {
  std::vector<Bound> all(n);
  uint64_t total = 0;
  for (size_t i = 0; i < n; i++) {
    cdm_status st = bind_job(jobs[i], &all[i]);
    if (st) { g_last = "job " + std::to_string(i) + ": " + g_last; return st; }
    if (all[i].total > cap_bytes) return fail(CDM_E_CAPACITY, "chunk larger than a staging slot");
    total += all[i].total;
  }
  std::vector<size_t>& order = *order_out;
  order.resize(n);
  std::iota(order.begin(), order.end(), size_t(0));
  if (e->opts.order_policy == 1) {
    std::vector<double> tt(n), dd(n);
    for (size_t i = 0; i < n; i++) {
      tt[i] = double(all[i].total) / (e->opts.pcie_gbps * 1e9);
      dd[i] = double(all[i].payload + all[i].offsets_bytes) / (e->opts.decode_gbps * 1e9 * family_rate(all[i]));
    }
    johnson(tt.data(), dd.data(), n, &order);
  }
  // groups: consecutive jobs (in issue order) up to a target size, so several groups pipeline
  uint64_t min_group = 2ull << 20;
  if (const char* g = std::getenv("CDM_GROUP_MIN_BYTES")) min_group = std::strtoull(g, nullptr, 10);
  const uint64_t target = std::min<uint64_t>(cap_bytes, std::max<uint64_t>(min_group, total / 8));
  // a group also closes as soon as its decode estimate exceeds its copy estimate (with Johnson order
  // those lead the pipeline: their decode should start as soon as their own bytes have arrived)
  static const bool split_decode_heavy = !(std::getenv("CDM_GROUP_SPLIT") && std::getenv("CDM_GROUP_SPLIT")[0] == '0');
  auto& groups = *groups_out;
  auto& first_job = *first_job_out;
  groups.clear();
  first_job.clear();
  size_t k = 0;
  while (k < n) {
    PendingGroup pg;
    uint64_t bytes = 0;
    double gt = 0, gd = 0;
    size_t m = k;
    while (m < n && pg.js.size() < size_t(kMaxBatch)) {
      const uint64_t add = ((all[order[m]].total + 255) & ~uint64_t(255));
      if (!pg.js.empty() && (bytes + add > cap_bytes || bytes >= target)) break;
      if (!pg.js.empty() && split_decode_heavy && gd > gt) break;
      const Bound& bj = all[order[m]];
      gt += double(bj.total) / (e->opts.pcie_gbps * 1e9);
      gd += double(bj.payload + bj.offsets_bytes) / (e->opts.decode_gbps * 1e9 * family_rate(bj));
      bytes += add;
      pg.bs.push_back(all[order[m]]);
      pg.js.push_back(&jobs[order[m]]);
      m++;
    }
    first_job.push_back(k);
    groups.push_back(std::move(pg));
    k = m;
  }
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_submit_batch(cdm_engine* e, const cdm_job* jobs, size_t n, uint64_t* tickets) {
  if (!e || (n && (!jobs || !tickets))) return fail(CDM_E_INVALID_ARG, "null argument");
  std::lock_guard<std::mutex> lock(e->mu);
  CUDA_TRY(cudaSetDevice(e->device));
  std::vector<PendingGroup> groups;
  std::vector<size_t> order, first_job;
  cdm_status st0 = plan_groups(e, jobs, n, e->opts.slot_bytes, &groups, &order, &first_job);
  if (st0) return st0;
  // the copy engine runs up to n_slots groups ahead of the decodes: copies are enqueued before the host
  // spends time building a group's launches
  const size_t ahead = e->slots.size();
  size_t copied = 0;
  for (size_t g = 0; g < groups.size(); g++) {
    while (copied < groups.size() && copied < g + ahead) {
      cdm_status st = group_copy(e, groups[copied]);
      if (st) return st;
      copied++;
    }
    std::vector<uint64_t> tk(groups[g].bs.size());
    cdm_status st = group_decode(e, groups[g], tk.data());
    if (st) return st;
    for (size_t j = 0; j < tk.size(); j++) tickets[order[first_job[g] + j]] = tk[j];
  }
  return CDM_OK;
}

// ============================================================================ pipelines (CUDA graphs)
// The whole H2D -> decode schedule of a fixed job set, captured once into a CUDA graph: copies of every
// group on one copy branch, each group's zero / fused kernels / error harvest on a decode branch that
// depends on its own copy.  A launch is one cudaGraphLaunch, so the GPU runs the pipeline without the
// host enqueueing each group (the submit path costs ~20 us of host time per group).
struct cdm_pipeline {
  cdm_engine* e = nullptr;
  int device = 0;
  size_t n = 0;
  uint8_t* staging = nullptr;  // every group's chunks, back to back (no slot reuse inside a pipeline)
  uint8_t* arena = nullptr;    // every group's decode scratch
  uint32_t* err_host = nullptr, *err_mapped = nullptr;  // per job in ISSUE order, mapped pinned
  uint32_t* err_dev = nullptr;  // per job in issue order: every group's kernels OR into their slice
  std::vector<std::unique_ptr<cdm_batch>> batches;
  std::vector<Bound> bound;    // per job (submission index)
  std::vector<size_t> pos;     // issue position of job i
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> events;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t last_stream = nullptr;
  uint32_t n_launches = 0, n_groups = 0, n_copies = 0;  // kernel launches / groups / H2D copies per launch
  ~cdm_pipeline() {
    if (exec) cudaGraphExecDestroy(exec);
    if (err_dev) cudaFree(err_dev);
    if (graph) cudaGraphDestroy(graph);
    for (auto ev : events) cudaEventDestroy(ev);
    for (auto st : streams) cudaStreamDestroy(st);
    batches.clear();
    if (staging) cudaFree(staging);
    if (arena) cudaFree(arena);
    if (err_host) cudaFreeHost(err_host);
  }
};

extern "C" CDM_API cdm_status cdm_pipeline_create(cdm_engine* e, const cdm_job* jobs, size_t n, cdm_pipeline** out) {
  if (!e || !out || (n && !jobs)) return fail(CDM_E_INVALID_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(e->device));
  auto P = std::make_unique<cdm_pipeline>();
  P->e = e;
  P->device = e->device;
  P->n = n;
  std::vector<PendingGroup> groups;
  std::vector<size_t> order, first_job;
  cdm_status st = plan_groups(e, jobs, n, e->opts.slot_bytes, &groups, &order, &first_job);
  if (st) return st;
  // staging layout: group after group; inside a group the chunks in host-address order, exactly contiguous
  // host neighbours (16-byte multiples) keep their relative offsets and share ONE H2D copy (pinned H2D runs
  // at ~41 GB/s for 1 MB copies vs ~55 GB/s from 8 MB up); other chunks start 256-aligned
  struct CopyRun { size_t off, bytes; const void* src; };
  std::vector<std::vector<CopyRun>> runs(groups.size());
  std::vector<std::vector<size_t>> stage_off(groups.size());
  size_t stage_bytes = 0;
  for (size_t g = 0; g < groups.size(); g++) {
    auto& G = groups[g];
    std::vector<size_t> by_addr(G.bs.size());
    std::iota(by_addr.begin(), by_addr.end(), size_t(0));
    std::sort(by_addr.begin(), by_addr.end(),
              [&](size_t a, size_t b) { return G.js[a]->host_chunk < G.js[b]->host_chunk; });
    stage_off[g].resize(G.bs.size());
    for (size_t k = 0; k < by_addr.size(); k++) {
      const size_t j = by_addr[k];
      const uint8_t* h = static_cast<const uint8_t*>(G.js[j]->host_chunk);
      CopyRun* last = runs[g].empty() ? nullptr : &runs[g].back();
      // a chunk that starts at most kCopyGap bytes after the previous run's end (the alignment padding of a
      // column store) joins that run: the copy spans the gap and the chunk keeps its 16-byte-aligned
      // relative offset in the staging region
      const uint8_t* last_end = last ? static_cast<const uint8_t*>(last->src) + last->bytes : nullptr;
      constexpr size_t kCopyGap = 256;
      if (last && h >= last_end && size_t(h - last_end) <= kCopyGap &&
          size_t(h - static_cast<const uint8_t*>(last->src)) % 16 == 0 && !getenv_flag("CDM_PIPE_NOMERGE")) {
        stage_off[g][j] = last->off + size_t(h - static_cast<const uint8_t*>(last->src));
        last->bytes = size_t(h - static_cast<const uint8_t*>(last->src)) + G.bs[j].total;
      } else {
        stage_bytes = (stage_bytes + 255) & ~size_t(255);
        stage_off[g][j] = stage_bytes;
        runs[g].push_back({stage_bytes, size_t(G.bs[j].total), h});
      }
      stage_bytes = stage_off[g][j] + G.bs[j].total;
    }
  }
  if (cudaMalloc(&P->staging, std::max<size_t>(stage_bytes, 256)) != cudaSuccess)
    return fail(CDM_E_OOM, "pipeline staging cudaMalloc failed");
  for (size_t g = 0; g < groups.size(); g++)
    for (size_t j = 0; j < groups[g].bs.size(); j++) groups[g].bs[j].dev_chunk = P->staging + stage_off[g][j];
  {
    // a copy may not span two host allocations that merely touch: try every merged run once, outside the
    // capture; the driver rejects such a copy at the call (cudaErrorInvalidValue) -> split it per chunk
    cudaStream_t probe = nullptr;
    CUDA_TRY(cudaStreamCreateWithFlags(&probe, cudaStreamNonBlocking));
    for (size_t g = 0; g < groups.size(); g++) {
      std::vector<CopyRun> fixed;
      for (const CopyRun& r : runs[g]) {
        bool whole = true;
        if (r.bytes > 0) {
          const cudaError_t ce = cudaMemcpyAsync(P->staging + r.off, r.src, r.bytes, cudaMemcpyHostToDevice, probe);
          if (ce == cudaErrorInvalidValue) { cudaGetLastError(); whole = false; }
          else if (ce != cudaSuccess) { cudaStreamDestroy(probe); return fail(CDM_E_CUDA, std::string("H2D probe: ") + cudaGetErrorString(ce)); }
        }
        if (whole) { fixed.push_back(r); continue; }
        for (size_t j = 0; j < groups[g].bs.size(); j++) {  // the run's chunks, one copy each
          const size_t o = stage_off[g][j];
          if (o >= r.off && o < r.off + r.bytes)
            fixed.push_back({o, size_t(groups[g].bs[j].total), groups[g].js[j]->host_chunk});
        }
      }
      runs[g].swap(fixed);
    }
    const cudaError_t se = cudaStreamSynchronize(probe);
    cudaStreamDestroy(probe);
    if (se != cudaSuccess) return fail(CDM_E_CUDA, std::string("H2D probe: ") + cudaGetErrorString(se));
  }
  // one batch per group over its own arena slice; error words in one array (issue order)
  if (cudaMalloc(&P->err_dev, sizeof(uint32_t) * std::max<size_t>(1, n)) != cudaSuccess)
    return fail(CDM_E_OOM, "pipeline error words cudaMalloc failed");
  CUDA_TRY(cudaMemset(P->err_dev, 0, sizeof(uint32_t) * std::max<size_t>(1, n)));
  std::vector<size_t> arena_off, zero_bytes;
  size_t arena_bytes = 0;
  for (size_t gi = 0; gi < groups.size(); gi++) {
    auto& g = groups[gi];
    auto B = std::make_unique<cdm_batch>();
    B->e = e;
    B->device = e->device;
    B->err_external = P->err_dev + first_job[gi];
    for (auto& b : g.bs) B->jobs.push_back(b);
    Alloc sizing;
    size_t zb = 0;
    const size_t need = layout_batch(B.get(), sizing, &zb);
    arena_off.push_back(arena_bytes);
    arena_bytes += (need + 255) & ~size_t(255);
    P->batches.push_back(std::move(B));
  }
  if (cudaMalloc(&P->arena, std::max<size_t>(arena_bytes, 256)) != cudaSuccess)
    return fail(CDM_E_OOM, "pipeline scratch cudaMalloc failed");
  // counters and look-back words reset themselves at the end of every launch; they start at zero once
  CUDA_TRY(cudaMemset(P->arena, 0, std::max<size_t>(arena_bytes, 256)));
  for (size_t g = 0; g < groups.size(); g++) {
    cdm_batch* B = P->batches[g].get();
    st = batch_build(B, P->arena + arena_off[g], arena_bytes - arena_off[g]);
    if (st) return st;
    B->zeroed_by_caller = true;
  }
  P->bound.resize(n);
  P->pos.resize(n);
  for (size_t g = 0; g < groups.size(); g++)
    for (size_t j = 0; j < groups[g].bs.size(); j++) {
      P->bound[order[first_job[g] + j]] = groups[g].bs[j];
      P->pos[order[first_job[g] + j]] = first_job[g] + j;
    }
  CUDA_TRY(cudaHostAlloc(&P->err_host, sizeof(uint32_t) * std::max<size_t>(1, n), cudaHostAllocMapped));
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&P->err_mapped), P->err_host, 0));
  std::memset(P->err_host, 0, sizeof(uint32_t) * std::max<size_t>(1, n));
  // streams for the capture: origin, copy, and up to 4 decode lanes (each with its 5 family streams)
  int prio_lo = 0, prio_hi = 0;
  CUDA_TRY(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  auto mk = [&](int prio) -> cudaStream_t {
    cudaStream_t x = nullptr;
    if (cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, prio) == cudaSuccess) P->streams.push_back(x);
    return x;
  };
  auto mkev = [&]() -> cudaEvent_t {
    cudaEvent_t x = nullptr;
    if (cudaEventCreateWithFlags(&x, cudaEventDisableTiming) == cudaSuccess) P->events.push_back(x);
    return x;
  };
  size_t max_lanes = 4;
  if (const char* v = std::getenv("CDM_PIPE_LANES")) max_lanes = std::max(1, std::atoi(v));
  const bool use_prio = !(std::getenv("CDM_PIPE_PRIO") && std::getenv("CDM_PIPE_PRIO")[0] == '0');
  if (!use_prio) prio_lo = prio_hi = 0;
  const size_t lanes = std::min<size_t>(std::max<size_t>(groups.size(), 1), max_lanes);
  cudaStream_t origin = mk(prio_hi), copy = mk(prio_hi);
  std::vector<cudaStream_t> ds(lanes);
  std::vector<std::array<cudaStream_t, kStreams>> fam(lanes);
  for (size_t l = 0; l < lanes; l++) {
    ds[l] = mk(prio_hi);
    for (int f = 0; f < kStreams; f++) fam[l][f] = mk(fam_priority(f, prio_lo, prio_hi));
  }
  for (auto x : P->streams) if (!x) return fail(CDM_E_CUDA, "pipeline stream creation failed");
  std::vector<cudaEvent_t> copied(groups.size());
  for (auto& ev : copied) ev = mkev();
  cudaEvent_t start = mkev(), copy_end = mkev();
  std::vector<cudaEvent_t> lane_end(lanes);
  for (auto& ev : lane_end) ev = mkev();
  for (auto x : P->events) if (!x) return fail(CDM_E_CUDA, "pipeline event creation failed");

  CUDA_TRY(cudaStreamBeginCapture(origin, cudaStreamCaptureModeRelaxed));
  auto abort_capture = [&](cdm_status s2) {
    cudaGraph_t g2 = nullptr;
    cudaStreamEndCapture(origin, &g2);
    if (g2) cudaGraphDestroy(g2);
    cudaGetLastError();
    return s2;
  };
#define CAP_TRY(x)                                                                                   \
  do {                                                                                               \
    cudaError_t ce_ = (x);                                                                           \
    if (ce_ != cudaSuccess) return abort_capture(fail(CDM_E_CUDA, std::string(#x ": ") + cudaGetErrorString(ce_))); \
  } while (0)
  CAP_TRY(cudaEventRecord(start, origin));
  CAP_TRY(cudaStreamWaitEvent(copy, start, 0));
  for (size_t l = 0; l < lanes; l++) CAP_TRY(cudaStreamWaitEvent(ds[l], start, 0));
  // copy branch: Johnson order of groups, one copy per run of host-contiguous chunks
  for (size_t g = 0; g < groups.size(); g++) {
    for (const CopyRun& r : runs[g]) {
      CAP_TRY(cudaMemcpyAsync(P->staging + r.off, r.src, r.bytes, cudaMemcpyHostToDevice, copy));
      P->n_copies++;
    }
    CAP_TRY(cudaEventRecord(copied[g], copy));
  }
  CAP_TRY(cudaEventRecord(copy_end, copy));
  // decode branches: group g on lane g % lanes
  for (size_t g = 0; g < groups.size(); g++) {
    const size_t l = g % lanes;
    cdm_batch* B = P->batches[g].get();
    B->fam = fam[l].data();
    CAP_TRY(cudaStreamWaitEvent(ds[l], copied[g], 0));
    uint32_t nl = 0;
    cdm_status s2 = batch_enqueue(B, ds[l], &nl);
    if (s2) return abort_capture(s2);
    P->n_launches += nl;
  }
  P->n_groups = uint32_t(groups.size());
  for (size_t l = 0; l < lanes; l++) {
    CAP_TRY(cudaEventRecord(lane_end[l], ds[l]));
    CAP_TRY(cudaStreamWaitEvent(origin, lane_end[l], 0));
  }
  CAP_TRY(cudaStreamWaitEvent(origin, copy_end, 0));
  // one harvest at the end: every job's error word to mapped pinned memory, then zeroed for the next launch
  CAP_TRY(launch_harvest(P->err_dev, P->err_mapped, uint32_t(n), origin));
  P->n_launches += 1;
#undef CAP_TRY
  CUDA_TRY(cudaStreamEndCapture(origin, &P->graph));
  // kernel nodes keep the priority of the stream they were captured on (RLE lowest, the rest highest)
  CUDA_TRY(cudaGraphInstantiate(&P->exec, P->graph, use_prio ? cudaGraphInstantiateFlagUseNodePriority : 0));
  *out = P.release();
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_pipeline_launch(cdm_pipeline* p, void* stream) {
  if (!p) return fail(CDM_E_INVALID_ARG, "null pipeline");
  CUDA_TRY(cudaSetDevice(p->device));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : p->e->decode;
  CUDA_TRY(cudaGraphLaunch(p->exec, s));
  p->last_stream = s;
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_pipeline_results(cdm_pipeline* p, cdm_result* results) {
  if (!p) return fail(CDM_E_INVALID_ARG, "null pipeline");
  CUDA_TRY(cudaSetDevice(p->device));
  if (p->last_stream) CUDA_TRY(cudaStreamSynchronize(p->last_stream));
  bool bad = false;
  for (size_t i = 0; i < p->n; i++) {
    const uint32_t w = p->err_host[p->pos[i]];
    if (results) {
      const Bound& b = p->bound[i];
      cdm_result& r = results[i];
      r.rows = b.rows;
      r.payload_bytes = b.payload;
      r.offsets_bytes = b.offsets_bytes;
      r.compressed_bytes = b.total;
      r.chunk_id = b.chunk_id;
      r.error_bits = w;
      r.status = w ? CDM_E_CORRUPT : CDM_OK;
    }
    if (w && !bad) {
      bad = true;
      g_last = "job " + std::to_string(i) + ": device error bits " + std::to_string(w);
    }
  }
  return bad ? CDM_E_CORRUPT : CDM_OK;
}

extern "C" CDM_API cdm_status cdm_pipeline_info(const cdm_pipeline* p, uint32_t* n_launches, uint32_t* n_groups,
                                               uint32_t* n_copies) {
  if (!p) return fail(CDM_E_INVALID_ARG, "null pipeline");
  if (n_launches) *n_launches = p->n_launches;
  if (n_groups) *n_groups = p->n_groups;
  if (n_copies) *n_copies = p->n_copies;
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_host_register(void* p, size_t bytes) {
  if (!p || !bytes) return fail(CDM_E_INVALID_ARG, "null / empty host range");
  CUDA_TRY(cudaHostRegister(p, bytes, cudaHostRegisterDefault));
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_host_alloc(size_t bytes, void** out) {
  if (!out || !bytes) return fail(CDM_E_INVALID_ARG, "null out / zero bytes");
  *out = nullptr;
  const cudaError_t ce = cudaHostAlloc(out, bytes, cudaHostAllocDefault);
  if (ce != cudaSuccess) { *out = nullptr; return fail(CDM_E_OOM, std::string("cudaHostAlloc: ") + cudaGetErrorString(ce)); }
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_host_free(void* p) {
  if (p) CUDA_TRY(cudaFreeHost(p));
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_host_unregister(void* p) {
  if (!p) return fail(CDM_E_INVALID_ARG, "null host pointer");
  CUDA_TRY(cudaHostUnregister(p));
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_pipeline_destroy(cdm_pipeline* p) {
  if (!p) return CDM_OK;
  cudaSetDevice(p->device);
  if (p->last_stream) cudaStreamSynchronize(p->last_stream);
  delete p;
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_wait(cdm_engine* e, uint64_t ticket, cdm_result* out) {
  if (!e) return fail(CDM_E_INVALID_ARG, "null engine");
  std::unique_lock<std::mutex> lock(e->mu);
  auto it = e->tickets.find(ticket);
  if (it == e->tickets.end()) return fail(CDM_E_BUSY, "unknown or consumed ticket");
  const uint64_t gid = it->second.group;
  {  // block on the group's event with the engine unlocked (other threads keep submitting / waiting)
    auto g = e->groups.find(gid);
    if (g != e->groups.end() && !g->second.harvested && g->second.done) {
      cudaEvent_t ev = g->second.done;
      lock.unlock();
      cudaError_t ce = cudaEventSynchronize(ev);  // a recycled event only makes this wait longer
      lock.lock();
      if (ce != cudaSuccess) return fail(CDM_E_CUDA, std::string("wait: ") + cudaGetErrorString(ce));
    }
  }
  it = e->tickets.find(ticket);  // another thread may have consumed it meanwhile
  if (it == e->tickets.end()) return fail(CDM_E_BUSY, "unknown or consumed ticket");
  cdm_status st = harvest_group(e, gid);
  if (st) return st;
  if (out) *out = it->second.res;
  cdm_status r = it->second.res.error_bits ? CDM_E_CORRUPT : CDM_OK;
  if (r) g_last = "chunk " + std::to_string(it->second.res.chunk_id) + ": device error bits " + std::to_string(it->second.res.error_bits);
  e->tickets.erase(it);
  auto g = e->groups.find(gid);
  if (g != e->groups.end() && --g->second.pending == 0) e->groups.erase(g);
  return r;
}

extern "C" CDM_API cdm_status cdm_engine_set_ingest(cdm_engine* e, const int* devices, size_t n) {
  if (!e || (n && !devices)) return fail(CDM_E_INVALID_ARG, "null argument");
  std::lock_guard<std::mutex> lock(e->mu);
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  for (size_t i = 0; i < n; i++)
    if (devices[i] < 0 || devices[i] >= ndev) return fail(CDM_E_INVALID_ARG, "ingest device out of range");
  // drain and drop the previous set
  for (auto& s : e->slots) CUDA_TRY(cudaStreamSynchronize(s.ds));
  for (auto& ig : e->ingest) {
    CUDA_TRY(cudaSetDevice(ig.device));
    CUDA_TRY(cudaStreamSynchronize(ig.stream));
    cudaStreamDestroy(ig.stream);
    cudaFree(ig.buf);
    for (auto ev : ig.copied) cudaEventDestroy(ev);
  }
  e->ingest.clear();
  e->ingest_rr = 0;
  for (size_t i = 0; i < n; i++) {
    cdm_engine::Ingest ig;
    ig.device = devices[i];
    CUDA_TRY(cudaSetDevice(ig.device));
    if (ig.device != e->device) {  // NVLink peer access both ways where the topology allows it
      int can = 0;
      cudaDeviceCanAccessPeer(&can, ig.device, e->device);
      if (can) {
        cudaError_t pe = cudaDeviceEnablePeerAccess(e->device, 0);
        if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) return fail(CDM_E_CUDA, "peer access");
        cudaGetLastError();
      }
    }
    CUDA_TRY(cudaStreamCreateWithFlags(&ig.stream, cudaStreamNonBlocking));
    if (cudaMalloc(&ig.buf, e->opts.slot_bytes) != cudaSuccess) { cudaSetDevice(e->device); return fail(CDM_E_OOM, "ingest buffer"); }
    ig.copied.resize(e->slots.size());
    for (auto& ev : ig.copied) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->ingest.push_back(ig);
  }
  CUDA_TRY(cudaSetDevice(e->device));
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_engine_launches(cdm_engine* e, uint64_t* n) {
  if (!e || !n) return fail(CDM_E_INVALID_ARG, "null argument");
  std::lock_guard<std::mutex> lock(e->mu);
  *n = e->kernel_launches;
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_ticket_event(cdm_engine* e, uint64_t ticket, void** cuda_event) {
  if (!e || !cuda_event) return fail(CDM_E_INVALID_ARG, "null argument");
  std::lock_guard<std::mutex> lock(e->mu);
  auto it = e->tickets.find(ticket);
  if (it == e->tickets.end()) return fail(CDM_E_BUSY, "unknown or consumed ticket");
  auto g = e->groups.find(it->second.group);
  if (g == e->groups.end() || g->second.harvested || !g->second.done) *cuda_event = e->complete;
  else *cuda_event = g->second.done;
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_synchronize(cdm_engine* e) {
  if (!e) return fail(CDM_E_INVALID_ARG, "null engine");
  std::lock_guard<std::mutex> lock(e->mu);
  CUDA_TRY(cudaStreamSynchronize(e->copy));
  CUDA_TRY(cudaStreamSynchronize(e->decode));
  for (auto& s : e->slots) CUDA_TRY(cudaStreamSynchronize(s.ds));
  std::vector<uint64_t> gids;
  for (auto& kv : e->groups) gids.push_back(kv.first);
  for (uint64_t gid : gids) {
    cdm_status st = harvest_group(e, gid);
    if (st) return st;
  }
  return CDM_OK;
}

// ============================================================================ device batch API
extern "C" CDM_API cdm_status cdm_batch_create(cdm_engine* e, const cdm_job* jobs, size_t n, cdm_batch** out) {
  if (!e || !out || (n && !jobs)) return fail(CDM_E_INVALID_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(e->device));
  auto B = std::make_unique<cdm_batch>();
  B->e = e;
  B->fam = e->fam;
  B->device = e->device;
  for (size_t i = 0; i < n; i++) {
    if (!jobs[i].dev_chunk) return fail(CDM_E_INVALID_ARG, "job " + std::to_string(i) + ": dev_chunk is null");
    if (reinterpret_cast<uintptr_t>(jobs[i].dev_chunk) % 16) return fail(CDM_E_INVALID_ARG, "dev_chunk must be 16-byte aligned");
    Bound b;
    cdm_status st = bind_job(jobs[i], &b);
    if (st) { g_last = "job " + std::to_string(i) + ": " + g_last; return st; }
    B->jobs.push_back(b);
  }
  cdm_status st = batch_build(B.get(), nullptr, 0);  // zeroes the scratch prefix once
  if (st) return st;
  B->sticky_errors = true;
  CUDA_TRY(cudaHostAlloc(&B->err_host, sizeof(uint32_t) * std::max<size_t>(1, n), cudaHostAllocDefault));
  *out = B.release();
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_batch_launch(cdm_batch* b, void* stream, uint32_t* n_launches) {
  if (!b) return fail(CDM_E_INVALID_ARG, "null batch");
  CUDA_TRY(cudaSetDevice(b->device));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : b->e->decode;
  if (!b->use_graph) return batch_enqueue(b, s, n_launches);
  if (b->graph_pending) {  // the previous replay's timing was not collected: it is lost
    b->graph_pending = false;
  }
  if (!b->gexec || b->gstream != s || b->graph_timing != b->timing || b->graph_mode != b->timing_mode) {
    b->drop_graph();
    uint64_t before[5];
    for (int f = 0; f < 5; f++) before[f] = b->fam_launches[f];
    const size_t pend0 = b->pending.size();
    CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    b->capturing = true;
    uint32_t nl = 0;
    cdm_status st = batch_enqueue(b, s, &nl);
    b->capturing = false;
    cudaGraph_t g = nullptr;
    cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (st) { if (g) cudaGraphDestroy(g); return st; }
    if (ce != cudaSuccess) return fail(CDM_E_CUDA, std::string("batch graph capture: ") + cudaGetErrorString(ce));
    b->graph = g;
    CUDA_TRY(cudaGraphInstantiate(&b->gexec, g, 0));
    b->gstream = s;
    b->graph_timing = b->timing;
    b->graph_mode = b->timing_mode;
    b->graph_nl = nl;
    for (int f = 0; f < 5; f++) {
      b->graph_fam_launches[f] = b->fam_launches[f] - before[f];
      b->fam_launches[f] = before[f];
    }
    b->graph_events.assign(b->pending.begin() + pend0, b->pending.end());
    b->pending.resize(pend0);
  }
  CUDA_TRY(cudaGraphLaunch(b->gexec, s));
  for (int f = 0; f < 5; f++) b->fam_launches[f] += b->graph_fam_launches[f];
  b->graph_pending = b->timing;
  if (n_launches) *n_launches = b->graph_nl;
  return CDM_OK;
}

// Graph mode with timing: the replay's per-family events are read after it completes (call between replays,
// outside any caller-timed region).
extern "C" CDM_API cdm_status cdm_batch_collect_timing(cdm_batch* b) {
  if (!b) return fail(CDM_E_INVALID_ARG, "null batch");
  if (!b->graph_pending) return CDM_OK;
  for (auto& p : b->graph_events) {
    CUDA_TRY(cudaEventSynchronize(p.b));
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, p.a, p.b));
    if (p.fam >= 100) { b->k_ms[p.fam - 100] += ms; b->k_n[p.fam - 100]++; }
    else b->fam_ms[p.fam] += ms;
  }
  b->graph_pending = false;
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_batch_set_graph(cdm_batch* b, int enable) {
  if (!b) return fail(CDM_E_INVALID_ARG, "null batch");
  b->use_graph = enable != 0;
  if (!b->use_graph) b->drop_graph();
  return CDM_OK;
}

// CDM_TRACE: append "kernel,launch,tile,t_start,t_unpacked,t_scanned,t_lookback,t_end,smid" rows (ns)
static void dump_trace(cdm_batch* b, const char* path) {
  FILE* f = std::fopen(path, "a");
  if (!f) return;
  auto dump = [&](const char* name, int li, uint64_t* dev, uint32_t tiles) {
    if (!dev || !tiles) return;
    std::vector<uint64_t> h(size_t(tiles) * 8);
    if (cudaMemcpy(h.data(), dev, h.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return;
    for (uint32_t t = 0; t < tiles; t++) {
      const uint64_t* r = &h[size_t(t) * 8];
      std::fprintf(f, "%s,%d,%u,%llu,%llu,%llu,%llu,%llu,%llu,%llu,%llu\n", name, li, t, (unsigned long long)r[0],
                   (unsigned long long)r[1], (unsigned long long)r[2], (unsigned long long)r[3],
                   (unsigned long long)r[4], (unsigned long long)r[7], (unsigned long long)r[5],
                   (unsigned long long)r[6]);
    }
  };
  for (size_t i = 0; i < b->scan.size(); i++) dump("scan", int(i), b->scan[i].trace, b->scan[i].total_tiles);
  for (size_t i = 0; i < b->sums.size(); i++) dump("sums", int(i), b->sums[i].trace, b->sums[i].total_units);
  for (size_t i = 0; i < b->rle.size(); i++) dump("rle", int(i), b->rle[i].trace, b->rle[i].total_tiles);
  std::fclose(f);
}

extern "C" CDM_API cdm_status cdm_batch_results(cdm_batch* b, void* stream, cdm_result* results) {
  if (!b) return fail(CDM_E_INVALID_ARG, "null batch");
  CUDA_TRY(cudaSetDevice(b->device));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : b->e->decode;
  CUDA_TRY(cudaMemcpyAsync(b->err_host, b->err_dev, sizeof(uint32_t) * std::max<size_t>(1, b->jobs.size()),
                           cudaMemcpyDeviceToHost, s));
  if (b->sticky_errors)  // the next launch starts from clean error words
    CUDA_TRY(cudaMemsetAsync(b->err_dev, 0, sizeof(uint32_t) * std::max<size_t>(1, b->jobs.size()), s));
  CUDA_TRY(cudaStreamSynchronize(s));
  for (auto& p : b->pending) {
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, p.a, p.b));
    if (p.fam >= 100) { b->k_ms[p.fam - 100] += ms; b->k_n[p.fam - 100]++; }
    else b->fam_ms[p.fam] += ms;
  }
  b->pending.clear();
  if (const char* path = std::getenv("CDM_TRACE")) dump_trace(b, path);
  if (results) fill_results(b, b->err_host, results);
  for (size_t i = 0; i < b->jobs.size(); i++)
    if (b->err_host[i]) {
      g_last = "job " + std::to_string(i) + ": device error bits " + std::to_string(b->err_host[i]);
      return CDM_E_CORRUPT;
    }
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_batch_destroy(cdm_batch* b) {
  if (!b) return CDM_OK;
  cudaSetDevice(b->device);
  delete b;
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_batch_set_timing(cdm_batch* b, int enable) {
  if (!b) return fail(CDM_E_INVALID_ARG, "null batch");
  b->timing = enable != 0;
  b->timing_mode = enable;
  for (int i = 0; i < 5; i++) { b->fam_ms[i] = 0; b->fam_launches[i] = 0; }
  for (int i = 0; i < kKernelKinds; i++) { b->k_ms[i] = 0; b->k_n[i] = 0; }
  b->pending.clear();
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_checksum(const void* dev_data, uint64_t bytes, uint64_t chunk_id, void* stream,
                                           uint64_t* out) {
  if (!out || (bytes && !dev_data)) return fail(CDM_E_INVALID_ARG, "null argument");
  if (reinterpret_cast<uintptr_t>(dev_data) % 8) return fail(CDM_E_INVALID_ARG, "dev_data must be 8-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint64_t* d = nullptr;
  CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d), 8, s));
  cudaError_t e = cudaMemsetAsync(d, 0, 8, s);
  if (e == cudaSuccess) e = cdm::launch_checksum(dev_data, bytes, chunk_id, d, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, 8, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(d, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(CDM_E_CUDA, std::string("checksum: ") + cudaGetErrorString(e));
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_tune_set(const char* knob, int value) {
  if (!knob) return fail(CDM_E_INVALID_ARG, "null knob");
  const std::string k(knob);
  if (k == "fp_ctas_per_sm") {
    if (value < 0 || value > 16) return fail(CDM_E_INVALID_ARG, "fp_ctas_per_sm must be 0..16");
    cdm::tune_set(cdm::TUNE_FP_CTAS_PER_SM, value);
  } else if (k == "lz4_lanes") {
    if (value != 1 && value != 2 && value != 4 && value != 8 && value != 16 && value != 32)
      return fail(CDM_E_INVALID_ARG, "lz4_lanes must be 1, 2, 4, 8, 16 or 32");
    cdm::tune_set(cdm::TUNE_LZ4_LANES, value);
  } else if (k == "gp_ctas_per_sm") {
    if (value < 0 || value > 8) return fail(CDM_E_INVALID_ARG, "gp_ctas_per_sm must be 0..8");
    cdm::tune_set(cdm::TUNE_GP_CTAS_PER_SM, value);
  } else if (k == "scan_mode") {
    if (value < 0 || value > 2) return fail(CDM_E_INVALID_ARG, "scan_mode must be 0 (reduce-then-scan), 1 (look-back) or 2 (warp tiles)");
    cdm::tune_set(cdm::TUNE_SCAN_MODE, value);
  } else if (k == "lz4_split") {
    if (value != 0 && value != 1) return fail(CDM_E_INVALID_ARG, "lz4_split must be 0 (lz4_lanes schedules) or 1 (split parse/copy)");
    cdm::tune_set(cdm::TUNE_LZ4_SPLIT, value);
  } else if (k == "lz4_split_g") {
    if (value != 0 && value != 1 && value != 2 && value != 4 && value != 8)
      return fail(CDM_E_INVALID_ARG, "lz4_split_g must be 0 (per launch size) or 1, 2, 4, 8");
    cdm::tune_set(cdm::TUNE_LZ4_SPLIT_G, value);
  } else if (k == "lz4_spec") {
    if (value < 0 || value > 2) return fail(CDM_E_INVALID_ARG, "lz4_spec must be 0 (never), 1 (small launches) or 2 (always: speculative parallel parse)");
    cdm::tune_set(cdm::TUNE_LZ4_SPEC, value);
  } else {
    return fail(CDM_E_INVALID_ARG, "unknown tuning knob '" + k + "'");
  }
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_tune_get(const char* knob, int* value) {
  if (!knob || !value) return fail(CDM_E_INVALID_ARG, "null argument");
  const std::string k(knob);
  if (k == "fp_ctas_per_sm") *value = cdm::tune_get(cdm::TUNE_FP_CTAS_PER_SM);
  else if (k == "lz4_lanes") *value = cdm::tune_get(cdm::TUNE_LZ4_LANES);
  else if (k == "scan_mode") *value = cdm::tune_get(cdm::TUNE_SCAN_MODE);
  else if (k == "gp_ctas_per_sm") *value = cdm::tune_get(cdm::TUNE_GP_CTAS_PER_SM);
  else if (k == "lz4_split") *value = cdm::tune_get(cdm::TUNE_LZ4_SPLIT);
  else if (k == "lz4_split_g") *value = cdm::tune_get(cdm::TUNE_LZ4_SPLIT_G);
  else if (k == "lz4_spec") *value = cdm::tune_get(cdm::TUNE_LZ4_SPEC);
  else return fail(CDM_E_INVALID_ARG, "unknown tuning knob '" + k + "'");
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_batch_kernel_times(cdm_batch* b, double* ms, uint64_t* launches) {
  if (!b) return fail(CDM_E_INVALID_ARG, "null batch");
  for (int i = 0; i < kKernelKinds; i++) {
    if (ms) ms[i] = b->k_ms[i];
    if (launches) launches[i] = b->k_n[i];
  }
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_batch_kernel_bytes(cdm_batch* b, uint64_t* bytes) {
  if (!b || !bytes) return fail(CDM_E_INVALID_ARG, "null argument");
  for (int i = 0; i < kKernelKinds; i++) bytes[i] = b->k_bytes[i];
  return CDM_OK;
}

extern "C" CDM_API cdm_status cdm_batch_kernel_ms(cdm_batch* b, double* ms5, uint64_t* launches5) {
  if (!b) return fail(CDM_E_INVALID_ARG, "null batch");
  for (int i = 0; i < 5; i++) {
    if (ms5) ms5[i] = b->fam_ms[i];
    if (launches5) launches5[i] = b->fam_launches[i];
  }
  return CDM_OK;
}
