// plan.h -- H1: cascade text (Table 2 notation) -> fused decode plan.
//
// The runtime's own parser (the encoder and the oracle have theirs).  Grammar:
//   node := NAME [ "(" k=v {, k=v} ")" ] [ "|" ( node | "[" node {, node} "]" ) ]
// Codec names are case-insensitive with non-alphanumerics ignored ("Bit-packing", "Dictionary encoding").
// Arity completion (reading R30): 0 children -> all outputs Raw; 1 child binds the primary
// stream (Dict->indices, RLE->values, Str->bytes); BitPack and LZ4 children are always Raw.
//
// Fusion ("fusing Fully-Parallel patterns to nearby patterns"): FP chains collapse into
// one map (H5); an FP producer of RLE values is absorbed into the expansion and an FP producer of counts
// into the counts scan (H7); Delta over BitPack is one single-pass scan (H6); LZ4 is a fusion barrier.
#pragma once
#include <cctype>
#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "format.h"

namespace cdm {

struct TNode {
  uint8_t codec = RAW;
  std::vector<std::unique_ptr<TNode>> kids;
};

inline int codec_from_name(const std::string& raw) {
  std::string b;
  for (char ch : raw)
    if (std::isalnum(static_cast<unsigned char>(ch))) b += char(std::tolower(static_cast<unsigned char>(ch)));
  if (b == "raw") return RAW;
  if (b == "bitpack" || b == "bitpacking" || b == "for") return BITPACK;
  if (b == "dict" || b == "dictionary" || b == "dictionaryencoding") return DICT;
  if (b == "float2int") return FLOAT2INT;
  if (b == "delta" || b == "deltaencoding") return DELTA;
  if (b == "rle") return RLE;
  if (b == "deltastride") return DSTRIDE;
  if (b == "strdict" || b == "stringdictionary") return STRDICT;
  if (b == "lz4") return LZ4;
  if (b == "str" || b == "string" || b == "varchar") return STR;
  if (b == "ans" || b == "rans") return ANS;
  return -1;
}

struct CascadeParser {
  const std::string& s;
  size_t pos = 0;
  std::string err;
  explicit CascadeParser(const std::string& t) : s(t) {}
  void ws() { while (pos < s.size() && std::isspace(static_cast<unsigned char>(s[pos]))) pos++; }
  bool fail(const std::string& m) { if (err.empty()) err = "parse error at " + std::to_string(pos) + ": " + m; return false; }

  std::unique_ptr<TNode> node() {
    ws();
    std::string name;
    while (pos < s.size() && (std::isalnum(static_cast<unsigned char>(s[pos])) || s[pos] == '-' || s[pos] == '_' ||
                              (s[pos] == ' ' && !name.empty() && pos + 1 < s.size() &&
                               std::isalpha(static_cast<unsigned char>(s[pos + 1]))))) {
      name += s[pos++];
    }
    if (name.empty()) { fail("expected codec name"); return nullptr; }
    int c = codec_from_name(name);
    if (c < 0) { err = "unknown codec '" + name + "'"; return nullptr; }
    auto t = std::make_unique<TNode>();
    t->codec = uint8_t(c);
    ws();
    if (pos < s.size() && s[pos] == '(') {  // options: accepted and ignored by the decoder
      while (pos < s.size() && s[pos] != ')') pos++;
      if (pos >= s.size()) { fail("expected ')'"); return nullptr; }
      pos++;
      ws();
    }
    if (pos < s.size() && s[pos] == '|') {
      pos++;
      ws();
      if (pos < s.size() && s[pos] == '[') {
        pos++;
        for (;;) {
          if (t->kids.size() == 2) { fail("too many children"); return nullptr; }
          auto ch = node();
          if (!ch) return nullptr;
          t->kids.push_back(std::move(ch));
          ws();
          if (pos < s.size() && s[pos] == ',') { pos++; continue; }
          if (pos < s.size() && s[pos] == ']') { pos++; break; }
          fail("expected ',' or ']'");
          return nullptr;
        }
      } else {
        auto ch = node();
        if (!ch) return nullptr;
        t->kids.push_back(std::move(ch));
      }
    }
    return t;
  }
};

inline std::unique_ptr<TNode> mk_raw() { auto t = std::make_unique<TNode>(); t->codec = RAW; return t; }

inline bool complete_tree(TNode* t, std::string* err) {
  auto& k = t->kids;
  switch (t->codec) {
    case RAW:
      if (!k.empty()) { *err = "arity error: Raw takes no children"; return false; }
      return true;
    case BITPACK:
      if (k.empty()) k.push_back(mk_raw());
      if (k.size() != 1 || (k[0]->codec != RAW && k[0]->codec != ANS)) {
        *err = "arity error: BitPack's only child is Raw or ANS";
        return false;
      }
      break;
    case LZ4:
    case ANS:
      if (!k.empty()) { *err = "arity error: LZ4/ANS take no children"; return false; }
      k.push_back(mk_raw());
      k.push_back(mk_raw());
      return true;
    case DICT:
    case STRDICT:
      if (k.empty()) { k.push_back(mk_raw()); k.push_back(mk_raw()); }
      else if (k.size() == 1) k.insert(k.begin(), mk_raw());
      if (k[0]->codec != RAW) { *err = "arity error: a dictionary stream is Raw"; return false; }
      break;
    case FLOAT2INT:
    case DELTA:
      if (k.empty()) k.push_back(mk_raw());
      if (k.size() != 1) { *err = "arity error: Float2Int/Delta take one child"; return false; }
      break;
    case RLE:
    case STR:
    case DSTRIDE:
      if (k.empty()) { k.push_back(mk_raw()); k.push_back(mk_raw()); }
      else if (k.size() == 1) k.push_back(mk_raw());
      break;
    default:
      *err = "unknown codec";
      return false;
  }
  for (auto& c : k)
    if (!complete_tree(c.get(), err)) return false;
  return true;
}

inline const char* codec_name(uint8_t c) {
  static const char* N[] = {"RAW", "BITPACK", "DICT", "FLOAT2INT", "DELTA", "RLE", "LZ4", "STR", "ANS", "DELTASTRIDE", "STRDICT"};
  return c < 11 ? N[c] : "?";
}

inline void render_tree(const TNode* t, std::string* out) {
  *out += codec_name(t->codec);
  if (t->kids.empty()) return;
  *out += "|";
  if (t->kids.size() == 1) { render_tree(t->kids[0].get(), out); return; }
  *out += "[";
  for (size_t i = 0; i < t->kids.size(); i++) {
    if (i) *out += ",";
    render_tree(t->kids[i].get(), out);
  }
  *out += "]";
}

inline uint64_t fnv1a64(const std::string& s) {
  uint64_t h = 14695981039346656037ull;
  for (unsigned char ch : s) { h ^= ch; h *= 1099511628211ull; }
  return h;
}

// ------------------------------------------------------------------ fused plans
enum class PlanKind : uint8_t { RawCopy, Fp, Scan, Rle, Str, Ans };

struct Plan {
  PlanKind kind = PlanKind::RawCopy;
  uint8_t fp_mode = 0;   // FpMode
  uint8_t vmode = 0;     // RleValueMode
  bool str_lz4 = false;
  bool str_ans = false;
  std::string text;      // human-readable fused plan
};

// Recognise the fused shapes; anything else is a valid cascade without a device plan.
inline bool compile_plan(const TNode* r, uint8_t dtype, Plan* p, std::string* err) {
  auto is = [](const TNode* t, uint8_t c) { return t && t->codec == c; };
  auto bp = [&](const TNode* t) { return is(t, BITPACK) && is(t->kids[0].get(), RAW); };
  auto kid = [](const TNode* t, size_t i) -> const TNode* { return i < t->kids.size() ? t->kids[i].get() : nullptr; };
  if (dtype == T_VARBYTES) {
    // String-dictionary bytes (NEXT-2, Table 2 O_COMMENT P:540): token ids BitPack'd, the packed bytes
    // optionally ANS-coded
    const TNode* sd = kid(r, 0);
    const bool strdict = is(sd, STRDICT) && is(kid(sd, 1), BITPACK) &&
                         (is(kid(kid(sd, 1), 0), RAW) || is(kid(kid(sd, 1), 0), ANS));
    if (is(r, STR) && bp(kid(r, 1)) && (is(sd, LZ4) || is(sd, RAW) || is(sd, ANS) || strdict)) {
      p->kind = PlanKind::Str;
      p->str_lz4 = is(sd, LZ4);
      p->str_ans = is(sd, ANS);
      p->text = p->str_lz4 ? "scan_offsets(unpack lengths) + lz4_group_decode"
              : p->str_ans ? "scan_offsets(unpack lengths) + ans_chunk_decode"
              : strdict    ? (is(kid(kid(sd, 1), 0), ANS)
                                  ? "scan_offsets(unpack lengths) + ans_chunk_decode(ids) + strdict_expand"
                                  : "scan_offsets(unpack lengths) + strdict_expand")
                           : "scan_offsets(unpack lengths) + copy";
      return true;
    }
    *err = "VARBYTES needs Str|[LZ4,BitPack], Str|[ANS,BitPack], Str|[StrDict|BitPack(|ANS),BitPack] or Str|[Raw,BitPack]";
    return false;
  }
  if (is(r, ANS)) {
    if (dtype != T_FIXED) { *err = "an ANS root needs a FIXED(n) byte column"; return false; }
    p->kind = PlanKind::Ans;
    p->text = "ans_chunk_decode (one chunk per thread, SIMT)";
    return true;
  }
  if (is(r, STR) || is(r, LZ4)) { *err = "Str/LZ4 roots need a VARBYTES column"; return false; }
  if (is(r, RAW)) { p->kind = PlanKind::RawCopy; p->text = "copy"; return true; }
  if (bp(r)) { p->kind = PlanKind::Fp; p->fp_mode = 0; p->text = "fp(unpack+FOR+cast)"; return true; }
  if (is(r, DICT) && bp(kid(r, 1))) { p->kind = PlanKind::Fp; p->fp_mode = 1; p->text = "fp(unpack+FOR+dict gather)"; return true; }
  if (is(r, FLOAT2INT) && bp(kid(r, 0))) { p->kind = PlanKind::Fp; p->fp_mode = 2; p->text = "fp(unpack+FOR+float2int)"; return true; }
  if (is(r, DELTA) && bp(kid(r, 0))) { p->kind = PlanKind::Scan; p->text = "scan(unpack+FOR+delta, decoupled look-back)"; return true; }
  // Table 2's PS_SUPPKEY (reading R36): the deltas are Dict|BitPack-coded; the gather fuses into the scan
  if (is(r, DELTA) && is(kid(r, 0), DICT) && bp(kid(kid(r, 0), 1))) {
    p->kind = PlanKind::Scan; p->fp_mode = 1;
    p->text = "scan(unpack+FOR+dict gather+delta)";
    return true;
  }
  auto is_delta_rle = [&](const TNode* t) {
    return is(t, DELTA) && is(kid(t, 0), RLE) && bp(kid(kid(t, 0), 0)) && bp(kid(kid(t, 0), 1));
  };
  if (is_delta_rle(r)) {
    p->kind = PlanKind::Rle; p->vmode = 4;
    p->text = "rle(arithmetic runs: unpack dv,dc + 2-component look-back + expand)";
    return true;
  }
  // RLE-family lineages (H7; DeltaStride = RLE with arithmetic runs): an RLE / DeltaStride node
  // with BitPack counts whose values are BitPack, (top-level RLE only) Dict|BitPack or Float2Int|BitPack, or a
  // lower level -- Delta|RLE arithmetic runs or another RLE / DeltaStride node -- up to 3 levels (Table 2's
  // L_ORDERKEY).  Each non-final level expands into an L2-resident array the next level reads.
  // The counts may themselves be an RLE-family node (Table 2's PS_PARTKEY `RLE|[DeltaStride, RLE]`): a
  // lower level expands them into an L2-resident u32 array.  Depth = the longest chain; at most 3.
  std::function<int(const TNode*, bool)> levels = [&](const TNode* t, bool top) -> int {
    if (is_delta_rle(t)) return 1;
    if (!(is(t, RLE) || is(t, DSTRIDE))) return 0;
    const TNode* cn = kid(t, 1);
    int cd = 0;
    if (!bp(cn)) {
      cd = levels(cn, false);
      if (!cd) return 0;
    }
    const TNode* v = kid(t, 0);
    int vd = 0;
    if (!bp(v)) {
      if (top && is(t, RLE) && ((is(v, DICT) && bp(kid(v, 1))) || (is(v, FLOAT2INT) && bp(kid(v, 0))))) {
        if (cd) return 0;  // dictionary / Float2Int values take the single-level path only
        return 1;
      }
      vd = levels(v, false);
      if (!vd) return 0;
    }
    const int below = vd > cd ? vd : cd;
    return below < 3 ? below + 1 : 0;
  };
  auto counts_lineage = [&](const TNode* t) { return (is(t, RLE) || is(t, DSTRIDE)) && !bp(kid(t, 1)); };
  if (const int nl = levels(r, true)) {
    const TNode* v = kid(r, 0);
    p->kind = PlanKind::Rle;
    const char* what = is(r, DSTRIDE) ? "arithmetic runs start + j*stride" : "expand";
    if (nl > 1) {
      p->vmode = 3;
      const bool vl = !bp(v), cl = counts_lineage(r);
      p->text = std::string("rle lineage levels") + (vl ? " (run values -> u64 array in L2)" : "") +
                (cl ? " (run counts -> u32 array in L2)" : "") + " + rle level " + std::to_string(nl - 1) +
                " (" + what + (vl ? ", values = a lower level's array" : "") +
                (cl ? ", counts = a lower level's array" : "") + ")";
    } else if (bp(v)) {
      p->vmode = 0; p->text = std::string("rle(unpack counts+values, ") + what + ")";
    } else if (is(v, DICT)) {
      p->vmode = 1; p->text = "rle(values = dict gather fused, look-back, expand)";
    } else {
      p->vmode = 2; p->text = "rle(values = float2int fused, look-back, expand)";
    }
    return true;
  }
  *err = "no fused device plan for this cascade";
  return false;
}

}  // namespace cdm
