/*
 * cdm_oracle.c -- the CPU ORACLE for the cascaded-columnar decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library.  It shares no code, header, table or helper with the
 * CUDA path (paper_2602_08190_b200/csrc) or with the encoder; it parses the CDM1 container on its own
 * (layout: DESIGN.md "CDM1 chunk container") and decodes every node with plain scalar loops, in the
 * order the paper defines each codec, with no blocking, fusion or reordering:
 *
 *   BitPack + FOR  PAPER.md:155-156 (Sec. 2.1 "Bit-packing and Frame of Reference"): v_i = bits
 *                  [i*w, i*w+w) LSB-first, out_i = FOR + v_i (mod 2^64).
 *   Dictionary     PAPER.md:145 (Sec. 2.1) and :240 (Fully-Parallel example): out_i = dict[idx_i].
 *   Float2Int      PAPER.md:159 (Sec. 2.1): out_i = (double)int_i / 10^d, one IEEE division.
 *   Delta          PAPER.md:148 (Sec. 2.1): out_i = base + sum_{k<=i} d_k (mod 2^64).
 *   RLE            PAPER.md:151 (Sec. 2.1) and :248 (Group-Parallel example): repeat value_g count_g
 *                  times; presum = cumsum(count) must end at n.
 *   LZ4            PAPER.md:179 (LZ77 family), :258-259 (Non-Parallel, independent chunks): the LZ4
 *                  block format, decoded byte by byte, one independent sub-chunk at a time.
 *   ANS            PAPER.md:176 (entropy family), :260 ("each intermediate decode state ... depends on its
 *                  predecessor", sequential within a chunk), reading R32: range
 *                  ANS, state x in [2^16, 2^32); per symbol slot = x mod 2^tl, the symbol s with
 *                  cum_s <= slot < cum_s + f_s (found by a linear scan), x = f_s (x div 2^tl) + slot - cum_s,
 *                  then while x < 2^16: x = x*2^16 + next word; a chunk must end at x = 2^16 with every word
 *                  read.
 *   DeltaStride    PAPER.md:481 (Sec. 5.3, "(start, stride, count) triples", an RLE variant), DESIGN.md reading
 *                  R9: children [starts, counts], one stride per node; run g fills [presum_{g-1}, presum_g)
 *                  with start_g + j*stride, j = 0, 1, ... (mod 2^64); presum must end at n.
 *   StrDict        PAPER.md:163 (Sec. 2.1 String-dictionary: "substituting them with dictionary indices"), :498
 *                  (each unique word a group expanded from the dictionary), reading R34: children
 *                  [dictionary = u32 offsets[E+1] + token bytes, token ids]; out = concatenation of the
 *                  ids' tokens, which must total the node's n bytes.
 *   Str            DESIGN.md reading R17: offsets_0 = 0, offsets_{i+1} = offsets_i + len_i.
 *   Checksum       SURVEY Sec. 8a H9 (optional positional checksum): h = sum over the 8-byte little-endian
 *                  words w_i of the decoded buffer (last one zero padded) of splitmix64(chunk_id ^ i ^ w_i),
 *                  mod 2^64; splitmix64 = the SplitMix64 output function (golden-gamma add, two xor-shift
 *                  multiplies, final xor-shift).
 *   Nesting        PAPER.md:509 (Table 2 notation), decoded depth-first: children first, then parent
 *                  (no fusion exists in the oracle).
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): hand-derived golden vectors (tests/golden/), brute force
 * over every bit width on tiny columns with a test-local bit writer, numpy repeat/cumsum/take, liblz4
 * cross-decoding, closed forms (c/100.0), invariants (sum of counts = n), truncation at every byte.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#include <pthread.h>

#define EXPORT __attribute__((visibility("default")))

/* oracle's own constants (the format spec is DESIGN.md's, restated here independently) */
#define O_MAGIC 0x314D4443u
enum { OC_RAW = 0, OC_BITPACK = 1, OC_DICT = 2, OC_FLOAT2INT = 3, OC_DELTA = 4, OC_RLE = 5, OC_LZ4 = 6, OC_STR = 7, OC_ANS = 8, OC_DSTRIDE = 9, OC_STRDICT = 10 };
enum { OT_I32 = 0, OT_I64 = 1, OT_F64 = 2, OT_FIXED = 3, OT_VARBYTES = 4 };
enum { OK = 0, ERR_ARG = 1, ERR_UNSUPPORTED = 3, ERR_CORRUPT = 4, ERR_CAPACITY = 5, ERR_OOM = 7 };

typedef struct {
  uint64_t rows;
  uint64_t payload_bytes;
  uint64_t offsets_bytes;
  uint64_t chunk_id;
  int32_t status;
  char detail[200];
} oracle_result;

typedef struct {
  const uint8_t *base;
  uint64_t total;
  uint32_t n_nodes, n_streams;
  const uint8_t *nodes;
  const uint8_t *stab;
  char *detail;
} ochunk;

/* a decoded stream: n elements of eb bytes; is_int => eb == 8 and elements are int64 (mod 2^64) */
typedef struct { uint64_t n; uint32_t eb; int is_int; uint8_t *data; } ostream;

static uint64_t rd64(const uint8_t *p) { uint64_t v; memcpy(&v, p, 8); return v; }
static uint32_t rd32(const uint8_t *p) { uint32_t v; memcpy(&v, p, 4); return v; }
static uint16_t rd16(const uint8_t *p) { uint16_t v; memcpy(&v, p, 2); return v; }

/* allocation of n elements of eb bytes; NULL when the product overflows or is implausibly large */
static void *alloc_n(uint64_t n, uint64_t eb) {
  uint64_t bytes;
  if (__builtin_mul_overflow(n, eb, &bytes) || bytes > (1ull << 40)) return NULL;
  return malloc(bytes ? bytes : 1);
}

static int bad(ochunk *c, const char *msg, unsigned long long a, unsigned long long b) {
  snprintf(c->detail, 200, msg, a, b);
  return ERR_CORRUPT;
}

static int decode_node(ochunk *c, uint32_t *idx, ostream *out);

/* a child that must be read as integers */
static int decode_int_child(ochunk *c, uint32_t *idx, ostream *out) {
  int rc = decode_node(c, idx, out);
  if (rc) return rc;
  if (!out->is_int) {
    if (out->eb != 8) { free(out->data); return bad(c, "node %llu: integer stream expected (elem bytes %llu)", *idx, out->eb); }
    out->is_int = 1; /* a Raw stream read as int64 little-endian */
  }
  return 0;
}

static int decode_node(ochunk *c, uint32_t *idx, ostream *out) {
  if (*idx >= c->n_nodes) return bad(c, "node %llu: missing (only %llu nodes)", *idx, c->n_nodes);
  const uint8_t *nd = c->nodes + 32ull * (*idx);
  uint32_t me = *idx;
  (*idx)++;
  uint8_t codec = nd[0], nch = nd[1];
  uint16_t sid = rd16(nd + 2);
  uint32_t raw_eb = rd32(nd + 4);
  uint64_t n = rd64(nd + 8);
  const uint8_t *pr = nd + 16;
  memset(out, 0, sizeof *out);

  switch (codec) {
  case OC_RAW: {
    if (nch != 0) return bad(c, "node %llu: Raw with %llu children", me, nch);
    if (sid >= c->n_streams) return bad(c, "node %llu: stream %llu out of range", me, sid);
    uint64_t off = rd64(c->stab + 16ull * sid), len = rd64(c->stab + 16ull * sid + 8);
    if (off > c->total || len > c->total - off) return bad(c, "stream %llu: bytes %llu beyond chunk", sid, len);
    if (raw_eb == 0 || n > len / raw_eb || n * raw_eb != len) return bad(c, "node %llu: raw stream length %llu mismatch", me, len);
    out->n = n; out->eb = raw_eb; out->is_int = 0;
    out->data = (uint8_t *)malloc(len ? len : 1);
    if (!out->data) return ERR_OOM;
    memcpy(out->data, c->base + off, len);
    return OK;
  }
  case OC_BITPACK: {
    /* "pack integers into the minimum bit-width ... the minimum value is stored
     * separately as a FOR".  Bits are LSB-first contiguous (reading R1). */
    if (nch != 1) return bad(c, "node %llu: BitPack needs 1 child, has %llu", me, nch);
    uint32_t w = pr[0];
    uint64_t forv = rd64(pr + 8);
    if (w > 64) return bad(c, "node %llu: bit width %llu > 64", me, w);
    ostream pk;
    int rc = decode_node(c, idx, &pk);
    if (rc) return rc;
    if (pk.eb != 1 || pk.is_int) { free(pk.data); return bad(c, "node %llu: packed stream must be bytes", me, 0); }
    if (w && n > (pk.n * 8) / w) { free(pk.data); return bad(c, "node %llu: packed stream too short (%llu bytes)", me, pk.n); }
    uint64_t *v = (uint64_t *)alloc_n(n, 8);
    if (!v) { free(pk.data); return bad(c, "node %llu: cannot hold %llu elements", me, n); }
    for (uint64_t i = 0; i < n; i++) {
      uint64_t field = 0;
      for (uint32_t b = 0; b < w; b++) {
        uint64_t k = i * (uint64_t)w + b;
        uint64_t bit = (pk.data[k >> 3] >> (k & 7)) & 1u;
        field |= bit << b;
      }
      v[i] = forv + field;
    }
    free(pk.data);
    out->n = n; out->eb = 8; out->is_int = 1; out->data = (uint8_t *)v;
    return OK;
  }
  case OC_DICT: {
    /* "the index maps original data values to their corresponding entries". */
    if (nch != 2) return bad(c, "node %llu: Dict needs 2 children, has %llu", me, nch);
    uint32_t entries = rd32(pr), E = rd32(pr + 4);
    ostream dict, ix;
    int rc = decode_node(c, idx, &dict);
    if (rc) return rc;
    if (dict.n != entries || dict.eb != E || E == 0) { free(dict.data); return bad(c, "node %llu: dictionary shape mismatch (%llu entries)", me, dict.n); }
    rc = decode_int_child(c, idx, &ix);
    if (rc) { free(dict.data); return rc; }
    if (ix.n != n) { free(dict.data); free(ix.data); return bad(c, "node %llu: %llu indices", me, ix.n); }
    uint8_t *o = (uint8_t *)alloc_n(n, E);
    if (!o) { free(dict.data); free(ix.data); return bad(c, "node %llu: cannot hold %llu elements", me, n); }
    const uint64_t *iv = (const uint64_t *)ix.data;
    for (uint64_t i = 0; i < n; i++) {
      if (iv[i] >= entries) {
        free(dict.data); free(ix.data); free(o);
        return bad(c, "row %llu: dictionary index %llu out of range", i, iv[i]);
      }
      memcpy(o + i * E, dict.data + iv[i] * E, E);
    }
    free(dict.data); free(ix.data);
    out->n = n; out->eb = E; out->is_int = 0; out->data = o;
    return OK;
  }
  case OC_FLOAT2INT: {
    /* "converting [floats] into integers"; decode divides by 10^d (IEEE, RN-even). */
    static const double TEN[23] = {1e0, 1e1, 1e2, 1e3, 1e4, 1e5, 1e6, 1e7, 1e8, 1e9, 1e10, 1e11,
                                   1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
    if (nch != 1) return bad(c, "node %llu: Float2Int needs 1 child, has %llu", me, nch);
    uint32_t d = pr[0];
    if (d > 22) return bad(c, "node %llu: decimal exponent %llu > 22", me, d);
    ostream iv;
    int rc = decode_int_child(c, idx, &iv);
    if (rc) return rc;
    if (iv.n != n) { free(iv.data); return bad(c, "node %llu: %llu ints", me, iv.n); }
    double *o = (double *)alloc_n(n, 8);
    if (!o) { free(iv.data); return bad(c, "node %llu: cannot hold %llu elements", me, n); }
    for (uint64_t i = 0; i < n; i++) {
      int64_t q; memcpy(&q, iv.data + 8 * i, 8);
      o[i] = (double)q / TEN[d];
    }
    free(iv.data);
    out->n = n; out->eb = 8; out->is_int = 0; out->data = (uint8_t *)o;
    return OK;
  }
  case OC_DELTA: {
    /* "replaces each value with the difference ... storing the initial value as a base". */
    if (nch != 1) return bad(c, "node %llu: Delta needs 1 child, has %llu", me, nch);
    uint64_t base = rd64(pr + 8);
    ostream dv;
    int rc = decode_int_child(c, idx, &dv);
    if (rc) return rc;
    if (dv.n != n) { free(dv.data); return bad(c, "node %llu: %llu deltas", me, dv.n); }
    uint64_t *o = (uint64_t *)dv.data, acc = base;
    for (uint64_t i = 0; i < n; i++) { acc += o[i]; o[i] = acc; }
    *out = dv; out->is_int = 1;
    return OK;
  }
  case OC_RLE: {
    /* PAPER.md:151 + :276: presum = cumsum(count); value g fills [presum_{g-1}, presum_g). */
    if (nch != 2) return bad(c, "node %llu: RLE needs 2 children, has %llu", me, nch);
    uint32_t nruns = rd32(pr);
    ostream vals, cnt;
    int rc = decode_node(c, idx, &vals);
    if (rc) return rc;
    rc = decode_int_child(c, idx, &cnt);
    if (rc) { free(vals.data); return rc; }
    if (vals.n != nruns || cnt.n != nruns) { free(vals.data); free(cnt.data); return bad(c, "node %llu: run arrays %llu", me, vals.n); }
    uint64_t eb = vals.eb;
    uint8_t *o = (uint8_t *)alloc_n(n, eb);
    if (!o) { free(vals.data); free(cnt.data); return bad(c, "node %llu: cannot hold %llu elements", me, n); }
    uint64_t pos = 0;
    for (uint64_t g = 0; g < nruns; g++) {
      uint64_t k = rd64(cnt.data + 8 * g);
      if (k > n - pos) { free(vals.data); free(cnt.data); free(o); return bad(c, "run %llu: count overflows the %llu rows", g, n); }
      for (uint64_t r = 0; r < k; r++) memcpy(o + (pos + r) * eb, vals.data + g * eb, eb);
      pos += k;
    }
    if (pos != n) { free(vals.data); free(cnt.data); free(o); return bad(c, "run sum %llu != %llu rows", pos, n); }
    int is_int = vals.is_int;
    free(vals.data); free(cnt.data);
    out->n = n; out->eb = (uint32_t)eb; out->is_int = is_int; out->data = o;
    return OK;
  }
  case OC_DSTRIDE: {
    /* "(start, stride, count) triples"; run g = start_g, start_g + stride, ... (count_g terms). */
    if (nch != 2) return bad(c, "node %llu: DeltaStride needs 2 children, has %llu", me, nch);
    uint32_t nruns = rd32(pr);
    uint64_t stride = rd64(pr + 8);
    ostream st, cnt;
    int rc = decode_int_child(c, idx, &st);
    if (rc) return rc;
    rc = decode_int_child(c, idx, &cnt);
    if (rc) { free(st.data); return rc; }
    if (st.n != nruns || cnt.n != nruns) { free(st.data); free(cnt.data); return bad(c, "node %llu: run arrays %llu", me, st.n); }
    uint64_t *o = (uint64_t *)alloc_n(n, 8);
    if (!o) { free(st.data); free(cnt.data); return bad(c, "node %llu: cannot hold %llu elements", me, n); }
    uint64_t pos = 0;
    for (uint64_t g = 0; g < nruns; g++) {
      uint64_t k = rd64(cnt.data + 8 * g), start = rd64(st.data + 8 * g);
      if (k > n - pos) { free(st.data); free(cnt.data); free(o); return bad(c, "run %llu: count overflows the %llu rows", g, n); }
      for (uint64_t j = 0; j < k; j++) o[pos + j] = start + j * stride;
      pos += k;
    }
    free(st.data); free(cnt.data);
    if (pos != n) { free(o); return bad(c, "run sum %llu != %llu rows", pos, n); }
    out->n = n; out->eb = 8; out->is_int = 1; out->data = (uint8_t *)o;
    return OK;
  }
  case OC_STRDICT: {
    /* "each unique word serve as a group ... and expands according to the lookup dictionary". */
    if (nch != 2) return bad(c, "node %llu: StrDict needs 2 children, has %llu", me, nch);
    uint32_t E = rd32(pr), dbytes = rd32(pr + 4);
    ostream dict, ix;
    int rc = decode_node(c, idx, &dict);
    if (rc) return rc;
    if (dict.eb != 1 || dict.is_int || dict.n != 4ull * (E + 1ull) + dbytes) { free(dict.data); return bad(c, "node %llu: dictionary stream of %llu bytes", me, dict.n); }
    const uint8_t *tok = dict.data + 4ull * (E + 1ull);
    for (uint32_t e = 0; e < E; e++)
      if (rd32(dict.data + 4ull * e) > rd32(dict.data + 4ull * e + 4)) { free(dict.data); return bad(c, "token %llu: offsets decrease (%llu)", e, 0); }
    if (rd32(dict.data) != 0 || rd32(dict.data + 4ull * E) != dbytes) { free(dict.data); return bad(c, "node %llu: dictionary offsets end at %llu", me, rd32(dict.data + 4ull * E)); }
    rc = decode_int_child(c, idx, &ix);
    if (rc) { free(dict.data); return rc; }
    uint8_t *o = (uint8_t *)alloc_n(n, 1);
    if (!o) { free(dict.data); free(ix.data); return bad(c, "node %llu: cannot hold %llu bytes", me, n); }
    uint64_t pos = 0;
    for (uint64_t k = 0; k < ix.n; k++) {
      uint64_t id = rd64(ix.data + 8 * k);
      if (id >= E) { free(dict.data); free(ix.data); free(o); return bad(c, "token %llu: dictionary index %llu out of range", k, id); }
      uint32_t a = rd32(dict.data + 4 * id), l = rd32(dict.data + 4 * id + 4) - a;
      if (l > n - pos) { free(dict.data); free(ix.data); free(o); return bad(c, "token %llu: bytes overflow the %llu output bytes", k, n); }
      memcpy(o + pos, tok + a, l);
      pos += l;
    }
    free(dict.data); free(ix.data);
    if (pos != n) { free(o); return bad(c, "token bytes %llu != %llu", pos, n); }
    out->n = n; out->eb = 1; out->is_int = 0; out->data = o;
    return OK;
  }
  case OC_LZ4: {
    /* LZ4 block format [ext]: token = (literal length:4 | match length-4:4), extension bytes of 255,
     * literals, 2-byte little-endian offset, match copied forward byte by byte (overlap allowed). */
    if (nch != 2) return bad(c, "node %llu: LZ4 needs 2 children, has %llu", me, nch);
    uint32_t nsub = rd32(pr);
    ostream pay, tab;
    int rc = decode_node(c, idx, &pay);
    if (rc) return rc;
    rc = decode_node(c, idx, &tab);
    if (rc) { free(pay.data); return rc; }
    if (pay.eb != 1 || tab.eb != 12 || tab.n != nsub) { free(pay.data); free(tab.data); return bad(c, "node %llu: LZ4 streams malformed (%llu)", me, tab.n); }
    uint8_t *o = (uint8_t *)alloc_n(n, 1);
    if (!o) { free(pay.data); free(tab.data); return bad(c, "node %llu: cannot hold %llu bytes", me, n); }
    uint64_t opos = 0;
    for (uint32_t s = 0; s < nsub; s++) {
      uint32_t co = rd32(tab.data + 12ull * s), cl = rd32(tab.data + 12ull * s + 4), dl = rd32(tab.data + 12ull * s + 8);
      if ((uint64_t)co + cl > pay.n || dl > n - opos) { free(pay.data); free(tab.data); free(o); return bad(c, "sub-chunk %llu: bounds (%llu)", s, co); }
      const uint8_t *ip = pay.data + co, *iend = ip + cl;
      uint8_t *dst = o + opos;
      uint64_t op = 0;
      for (;;) {
        if (ip >= iend) { free(pay.data); free(tab.data); free(o); return bad(c, "sub-chunk %llu: truncated at output %llu", s, op); }
        uint32_t token = *ip++;
        uint64_t lit = token >> 4;
        if (lit == 15) {
          uint32_t b;
          do {
            if (ip >= iend) { free(pay.data); free(tab.data); free(o); return bad(c, "sub-chunk %llu: truncated literal length %llu", s, lit); }
            b = *ip++; lit += b;
          } while (b == 255);
        }
        if (lit > (uint64_t)(iend - ip) || lit > dl - op) { free(pay.data); free(tab.data); free(o); return bad(c, "sub-chunk %llu: literal run %llu out of bounds", s, lit); }
        for (uint64_t k = 0; k < lit; k++) dst[op++] = *ip++;
        if (ip == iend) break; /* last sequence carries literals only */
        if (iend - ip < 2) { free(pay.data); free(tab.data); free(o); return bad(c, "sub-chunk %llu: truncated offset at %llu", s, op); }
        uint64_t offset = (uint64_t)ip[0] | ((uint64_t)ip[1] << 8);
        ip += 2;
        if (offset == 0 || offset > op) { free(pay.data); free(tab.data); free(o); return bad(c, "sub-chunk %llu: match offset %llu invalid", s, offset); }
        uint64_t ml = token & 15;
        if (ml == 15) {
          uint32_t b;
          do {
            if (ip >= iend) { free(pay.data); free(tab.data); free(o); return bad(c, "sub-chunk %llu: truncated match length %llu", s, ml); }
            b = *ip++; ml += b;
          } while (b == 255);
        }
        ml += 4;
        if (ml > dl - op) { free(pay.data); free(tab.data); free(o); return bad(c, "sub-chunk %llu: match length %llu out of bounds", s, ml); }
        for (uint64_t k = 0; k < ml; k++) { dst[op] = dst[op - offset]; op++; }
      }
      if (op != dl) { free(pay.data); free(tab.data); free(o); return bad(c, "sub-chunk %llu: decoded %llu bytes", s, op); }
      opos += dl;
    }
    free(pay.data); free(tab.data);
    if (opos != n) { free(o); return bad(c, "LZ4 node: decoded %llu of %llu bytes", opos, n); }
    out->n = n; out->eb = 1; out->is_int = 0; out->data = o;
    return OK;
  }
  case OC_ANS: {
    /* il interleaved states per chunk (1 or 32): symbol i of a chunk uses state i mod il, and the words are
     * consumed in symbol order (reading R32) */
    if (nch != 2) return bad(c, "node %llu: ANS needs 2 children, has %llu", me, nch);
    uint32_t nchunks = rd32(pr), chunk = rd32(pr + 4), tl = pr[8], il = pr[9] ? pr[9] : 1;
    if (tl < 8 || tl > 15 || chunk == 0 || (il != 1 && il != 32)) return bad(c, "node %llu: ANS params (table log %llu)", me, tl);
    const uint64_t rec = 8 + 4ull * il;
    ostream wds, tab;
    int rc = decode_node(c, idx, &wds);
    if (rc) return rc;
    rc = decode_node(c, idx, &tab);
    if (rc) { free(wds.data); return rc; }
    if (wds.eb != 2 || tab.eb != 1 || tab.n != 512 + rec * nchunks || (uint64_t)nchunks * chunk < n ||
        (n && (uint64_t)(nchunks - 1) * chunk >= n) || (!n && nchunks)) {
      free(wds.data); free(tab.data); return bad(c, "node %llu: ANS streams malformed (%llu)", me, tab.n);
    }
    const uint64_t M = 1ull << tl, L = 1ull << 16;
    uint64_t f[256], cum[256], acc = 0;
    for (int sy = 0; sy < 256; sy++) { f[sy] = rd16(tab.data + 2 * sy); cum[sy] = acc; acc += f[sy]; }
    if (n && acc != M) { free(wds.data); free(tab.data); return bad(c, "node %llu: ANS frequencies sum to %llu", me, acc); }
    uint8_t *o = (uint8_t *)alloc_n(n, 1);
    if (!o) { free(wds.data); free(tab.data); return bad(c, "node %llu: cannot hold %llu bytes", me, n); }
    for (uint32_t k = 0; k < nchunks; k++) {
      const uint8_t *ce = tab.data + 512 + rec * k;
      uint64_t w0 = rd32(ce), nw = rd32(ce + 4), x[32];
      for (uint32_t l = 0; l < il; l++) x[l] = rd32(ce + 8 + 4 * l);
      if (w0 + nw > wds.n) { free(wds.data); free(tab.data); free(o); return bad(c, "ANS chunk %llu: words beyond the stream (%llu)", k, w0 + nw); }
      uint64_t pos = 0;
      const uint64_t i0 = (uint64_t)k * chunk, i1 = i0 + chunk < n ? i0 + chunk : n;
      for (uint64_t i = i0; i < i1; i++) {
        uint64_t *xs = &x[(i - i0) % il];
        const uint64_t slot = *xs % M;
        int sy = 0;
        while (sy < 256 && !(cum[sy] <= slot && slot < cum[sy] + f[sy])) sy++;
        if (sy == 256) { free(wds.data); free(tab.data); free(o); return bad(c, "ANS chunk %llu: no symbol for slot %llu", k, slot); }
        o[i] = (uint8_t)sy;
        *xs = f[sy] * (*xs / M) + slot - cum[sy];
        while (*xs < L) {
          if (pos >= nw) { free(wds.data); free(tab.data); free(o); return bad(c, "ANS chunk %llu: words exhausted at byte %llu", k, i); }
          *xs = (*xs << 16) | rd16(wds.data + 2 * (w0 + pos));
          pos++;
        }
      }
      for (uint32_t l = 0; l < il; l++)
        if (x[l] != L) { free(wds.data); free(tab.data); free(o); return bad(c, "ANS chunk %llu: final state %llu", k, x[l]); }
      if (pos != nw) { free(wds.data); free(tab.data); free(o); return bad(c, "ANS chunk %llu: %llu words unread", k, nw - pos); }
    }
    free(wds.data); free(tab.data);
    out->n = n; out->eb = 1; out->is_int = 0; out->data = o;
    return OK;
  }
  default:
    return bad(c, "node %llu: codec %llu not decodable here", me, codec);
  }
}

/*
 * Decode one CDM1 chunk.  out receives payload_bytes (rows * width, or the VARBYTES bytes); for
 * VARBYTES, offsets receives rows+1 int32 (chunk-relative, exclusive end).  Returns 0 or an error
 * code; res->detail names the first violated field or the failing row.
 */
static uint64_t o_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

EXPORT uint64_t oracle_checksum(const void *data, uint64_t bytes, uint64_t chunk_id) {
  const uint8_t *p = (const uint8_t *)data;
  uint64_t h = 0;
  for (uint64_t i = 0; i * 8 < bytes; i++) {
    uint64_t w = 0;
    for (uint64_t k = 0; k < 8 && i * 8 + k < bytes; k++) w |= (uint64_t)p[i * 8 + k] << (8 * k);
    h += o_splitmix64(chunk_id ^ i ^ w);
  }
  return h;
}

EXPORT int oracle_decode_chunk(const void *chunk, size_t bytes, void *out, size_t out_cap, int32_t *offsets,
                               size_t offsets_cap, oracle_result *res) {
  oracle_result dummy;
  if (!res) res = &dummy;
  memset(res, 0, sizeof *res);
  ochunk c;
  memset(&c, 0, sizeof c);
  c.detail = res->detail;
  const uint8_t *p = (const uint8_t *)chunk;
  if (!p) { snprintf(res->detail, 200, "null chunk"); return res->status = ERR_ARG; }
  if (bytes < 64) { snprintf(res->detail, 200, "header: truncated (%zu bytes)", bytes); return res->status = ERR_CORRUPT; }
  if (rd32(p) != O_MAGIC) { snprintf(res->detail, 200, "header: bad magic"); return res->status = ERR_CORRUPT; }
  if (rd16(p + 4) != 1) { snprintf(res->detail, 200, "header: unsupported version %u", rd16(p + 4)); return res->status = ERR_CORRUPT; }
  c.n_nodes = rd16(p + 6);
  c.n_streams = rd16(p + 8);
  uint32_t dtype = p[10], width = rd32(p + 12);
  uint64_t rows = rd64(p + 16), payload = rd64(p + 24), offs_bytes = rd64(p + 32), total = rd64(p + 40);
  res->rows = rows; res->payload_bytes = payload; res->offsets_bytes = offs_bytes; res->chunk_id = rd64(p + 56);
  if (total > bytes) { snprintf(res->detail, 200, "header: total %llu > %zu bytes available", (unsigned long long)total, bytes); return res->status = ERR_CORRUPT; }
  if (64 + 32ull * c.n_nodes + 16ull * c.n_streams > total) { snprintf(res->detail, 200, "header: node/stream tables beyond chunk"); return res->status = ERR_CORRUPT; }
  c.base = p; c.total = total; c.nodes = p + 64; c.stab = p + 64 + 32ull * c.n_nodes;

  uint32_t W;
  switch (dtype) {
    case OT_I32: W = 4; break;
    case OT_I64: case OT_F64: W = 8; break;
    case OT_FIXED: W = width; break;
    case OT_VARBYTES: W = 1; break;
    default: snprintf(res->detail, 200, "header: bad dtype %u", dtype); return res->status = ERR_CORRUPT;
  }
  if (W == 0) { snprintf(res->detail, 200, "header: zero width"); return res->status = ERR_CORRUPT; }

  uint32_t idx = 0;
  int rc;
  if (dtype == OT_VARBYTES) {
    /* Str root: [bytes, lengths] -> offsets by running sum of lengths (reading R17). */
    if (c.n_nodes < 1 || c.nodes[0] != OC_STR || c.nodes[1] != 2) { snprintf(res->detail, 200, "VARBYTES needs a Str root"); return res->status = ERR_CORRUPT; }
    if (rd64(c.nodes + 8) != rows) { snprintf(res->detail, 200, "root rows mismatch"); return res->status = ERR_CORRUPT; }
    idx = 1;
    ostream by, ln;
    if ((rc = decode_node(&c, &idx, &by))) return res->status = rc;
    if ((rc = decode_int_child(&c, &idx, &ln))) { free(by.data); return res->status = rc; }
    if (by.eb != 1 || by.is_int || ln.n != rows || by.n != payload) {
      free(by.data); free(ln.data); snprintf(res->detail, 200, "Str: stream shapes mismatch"); return res->status = ERR_CORRUPT;
    }
    if (offs_bytes != 4 * (rows + 1) || offsets_cap < rows + 1 || out_cap < payload) {
      free(by.data); free(ln.data); snprintf(res->detail, 200, "output capacity"); return res->status = ERR_CAPACITY;
    }
    uint64_t acc = 0;
    offsets[0] = 0;
    for (uint64_t i = 0; i < rows; i++) {
      uint64_t l = rd64(ln.data + 8 * i);
      if (l > payload - acc) { free(by.data); free(ln.data); snprintf(res->detail, 200, "row %llu: length overflows payload", (unsigned long long)i); return res->status = ERR_CORRUPT; }
      acc += l;
      offsets[i + 1] = (int32_t)acc;
    }
    if (acc != payload) { free(by.data); free(ln.data); snprintf(res->detail, 200, "Str: lengths sum %llu != %llu", (unsigned long long)acc, (unsigned long long)payload); return res->status = ERR_CORRUPT; }
    if (payload) memcpy(out, by.data, payload);
    free(by.data); free(ln.data);
  } else {
    ostream r;
    if ((rc = decode_node(&c, &idx, &r))) return res->status = rc;
    /* a byte-stream root (ANS over FIXED(W) rows) decodes rows * W one-byte elements */
    const int byte_root = !r.is_int && r.eb == 1 && W > 1 && r.n == rows * W;
    if (r.n != rows && !byte_root) { free(r.data); snprintf(res->detail, 200, "root decodes %llu of %llu rows", (unsigned long long)r.n, (unsigned long long)rows); return res->status = ERR_CORRUPT; }
    if (payload != rows * W || out_cap < payload) { free(r.data); snprintf(res->detail, 200, "output capacity / payload size"); return res->status = ERR_CAPACITY; }
    uint8_t *o = (uint8_t *)out;
    if (r.is_int && W <= 8) {
      for (uint64_t i = 0; i < rows; i++) memcpy(o + i * W, r.data + 8 * i, W); /* low W bytes (LE) */
    } else if (!r.is_int && (r.eb == W || byte_root)) {
      if (payload) memcpy(o, r.data, payload);
    } else {
      free(r.data); snprintf(res->detail, 200, "root element width %u != dtype width %u", r.eb, W); return res->status = ERR_CORRUPT;
    }
    free(r.data);
  }
  if (idx != c.n_nodes) { snprintf(res->detail, 200, "%u nodes unused", c.n_nodes - idx); return res->status = ERR_CORRUPT; }
  return res->status = OK;
}

/* ---- chunk-parallel driver: each chunk still goes through the plain routine above ---- */
typedef struct {
  const void *const *chunks; const size_t *bytes; void *const *outs; const size_t *out_caps;
  int32_t *const *offs; const size_t *offs_caps; oracle_result *res;
  size_t n; size_t next; pthread_mutex_t mu;
} pool_t;

static void *worker(void *arg) {
  pool_t *P = (pool_t *)arg;
  for (;;) {
    pthread_mutex_lock(&P->mu);
    size_t i = P->next++;
    pthread_mutex_unlock(&P->mu);
    if (i >= P->n) return NULL;
    oracle_decode_chunk(P->chunks[i], P->bytes[i], P->outs[i], P->out_caps[i], P->offs ? P->offs[i] : NULL,
                        P->offs_caps ? P->offs_caps[i] : 0, &P->res[i]);
  }
}

EXPORT int oracle_decode_many(const void *const *chunks, const size_t *bytes, void *const *outs, const size_t *out_caps,
                              int32_t *const *offs, const size_t *offs_caps, oracle_result *res, size_t n, int nthreads) {
  pool_t P = {chunks, bytes, outs, out_caps, offs, offs_caps, res, n, 0, PTHREAD_MUTEX_INITIALIZER};
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, worker, &P);
  for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
  int worst = 0;
  for (size_t i = 0; i < n; i++) if (res[i].status) { worst = res[i].status; break; }
  return worst;
}
