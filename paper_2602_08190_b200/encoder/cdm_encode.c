/*
 * cdm_encode.c -- CPU cascade encoder producing self-contained CDM1 chunks.
 *
 * This is the paper's *offline* CPU side: "Raw data ... are first compressed utilizing [the
 * framework's] flexible nesting and customizable algorithms, with the resulting compressed
 * representations stored in CPU memory" (Sec. 3 Design).  It is an INPUT PRODUCER
 * for the decode hot path: it shares no code with the CUDA decode kernels (paper_2602_08190_b200/csrc)
 * nor with the CPU decode oracle (oracle/).  Its output is pinned by round trip through the oracle
 * against the generator's plain columns and by the hand-derived golden vectors in tests/golden/.
 *
 * Codec encode rules (readings in DESIGN.md "Readings of the paper"):
 *   BitPack+FOR  base = signed min, w = bits(max-min), LSB-first contiguous
 *   Dict         dictionary = unique elements sorted by unsigned bytes
 *   Float2Int    smallest d<=18 with (double)llrint(x*10^d)/10^d == x bitwise
 *   Delta        base = x[0], d[0] = 0, d[i] = x[i]-x[i-1] mod 2^64
 *   RLE          maximal runs, values + counts
 *   LZ4          LZ4 block format per independent sub-chunk (liblz4)
 *   ANS          range-ANS, 32-bit state / 16-bit words, shared table, chunks
 *   Str          VARBYTES -> [bytes, lengths]                                    (reading R17)
 * Container layout: DESIGN.md "CDM1 chunk container".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#include <ctype.h>
#include <math.h>

#define EXPORT __attribute__((visibility("default")))

/* liblz4 (no headers on this image; ABI from the LZ4 1.9 block API) */
extern int LZ4_compress_default(const char *src, char *dst, int srcSize, int dstCapacity);
extern int LZ4_compress_HC(const char *src, char *dst, int srcSize, int dstCapacity, int level);
extern int LZ4_compressBound(int inputSize);

enum { C_RAW = 0, C_BITPACK = 1, C_DICT = 2, C_FLOAT2INT = 3, C_DELTA = 4, C_RLE = 5, C_LZ4 = 6, C_STR = 7, C_ANS = 8, C_DSTRIDE = 9, C_STRDICT = 10 };
enum { D_I32 = 0, D_I64 = 1, D_F64 = 2, D_FIXED = 3, D_VARBYTES = 4 };
enum { E_OK = 0, E_INVALID_ARG = 1, E_PARSE = 2, E_UNSUPPORTED = 3, E_CORRUPT = 4, E_CAPACITY = 5, E_OOM = 7 };

static __thread char g_err[256];
static int fail(int code, const char *msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
EXPORT const char *cdm_encode_error(void) { return g_err; }

/* ------------------------------------------------------------------ cascade parser (encoder's own) */
typedef struct tnode {
  int codec;
  int nchild;
  struct tnode *child[2];
  uint32_t lz4_sub;   /* LZ4(sub=...) */
  int lz4_hc;         /* LZ4(hc=level) */
  uint32_t ans_chunk; /* ANS(chunk=...) bytes per independently coded chunk */
  uint32_t ans_tl;    /* ANS(tl=...) table log */
  uint32_t ans_il;    /* ANS(il=1|32) interleaved states per chunk (0 = default 32) */
  int64_t stride;     /* DeltaStride(stride=k), default 1 */
} tnode;

typedef struct { const char *s; size_t pos; int err; } parser;

static void skip_ws(parser *p) { while (p->s[p->pos] && isspace((unsigned char)p->s[p->pos])) p->pos++; }

static int codec_of(const char *name) {
  char b[64]; int k = 0;
  for (const char *c = name; *c && k < 63; c++) if (isalnum((unsigned char)*c)) b[k++] = (char)tolower((unsigned char)*c);
  b[k] = 0;
  if (!strcmp(b, "raw")) return C_RAW;
  if (!strcmp(b, "bitpack") || !strcmp(b, "bitpacking") || !strcmp(b, "for")) return C_BITPACK;
  if (!strcmp(b, "dict") || !strcmp(b, "dictionary") || !strcmp(b, "dictionaryencoding")) return C_DICT;
  if (!strcmp(b, "float2int")) return C_FLOAT2INT;
  if (!strcmp(b, "delta") || !strcmp(b, "deltaencoding")) return C_DELTA;
  if (!strcmp(b, "rle")) return C_RLE;
  if (!strcmp(b, "deltastride")) return C_DSTRIDE;
  if (!strcmp(b, "strdict") || !strcmp(b, "stringdictionary")) return C_STRDICT;
  if (!strcmp(b, "lz4")) return C_LZ4;
  if (!strcmp(b, "str") || !strcmp(b, "string") || !strcmp(b, "varchar")) return C_STR;
  if (!strcmp(b, "ans") || !strcmp(b, "rans")) return C_ANS;
  return -1;
}

static void free_tree(tnode *t) {
  if (!t) return;
  for (int i = 0; i < t->nchild; i++) free_tree(t->child[i]);
  free(t);
}

static tnode *parse_node(parser *p);

static tnode *parse_node(parser *p) {
  skip_ws(p);
  char name[64]; int k = 0;
  /* codec names may contain letters, digits, '-' and inner spaces ("Bit-packing", "Dictionary encoding") */
  while (p->s[p->pos] && (isalnum((unsigned char)p->s[p->pos]) || p->s[p->pos] == '-' || p->s[p->pos] == '_' ||
                          (p->s[p->pos] == ' ' && k > 0 && isalpha((unsigned char)p->s[p->pos + 1])))) {
    if (k < 63) name[k++] = p->s[p->pos];
    p->pos++;
  }
  name[k] = 0;
  if (!k) { p->err = 1; snprintf(g_err, sizeof g_err, "parse error at %zu: expected codec name", p->pos); return NULL; }
  int c = codec_of(name);
  if (c < 0) { p->err = 1; snprintf(g_err, sizeof g_err, "unknown codec '%s' at %zu", name, p->pos); return NULL; }
  tnode *t = (tnode *)calloc(1, sizeof(tnode));
  t->codec = c;
  t->lz4_sub = 65536;
  t->ans_chunk = 0;   /* default: 16384 with 32 interleaved states, 4096 with one */
  t->ans_tl = 12;
  t->ans_il = 32;
  t->stride = 1;
  skip_ws(p);
  if (p->s[p->pos] == '(') { /* options k=v,... */
    p->pos++;
    for (;;) {
      skip_ws(p);
      char key[32]; int kk = 0;
      while (isalnum((unsigned char)p->s[p->pos]) && kk < 31) key[kk++] = p->s[p->pos++];
      key[kk] = 0;
      skip_ws(p);
      if (p->s[p->pos] != '=') { p->err = 1; snprintf(g_err, sizeof g_err, "parse error at %zu: expected '='", p->pos); free_tree(t); return NULL; }
      p->pos++;
      skip_ws(p);
      char *end;
      unsigned long long v = strtoull(p->s + p->pos, &end, 10);
      if (end == p->s + p->pos) { p->err = 1; snprintf(g_err, sizeof g_err, "parse error at %zu: expected number", p->pos); free_tree(t); return NULL; }
      p->pos = (size_t)(end - p->s);
      if (!strcmp(key, "sub")) t->lz4_sub = (uint32_t)v;
      else if (!strcmp(key, "hc")) t->lz4_hc = (int)v;
      else if (!strcmp(key, "chunk")) t->ans_chunk = (uint32_t)v;
      else if (!strcmp(key, "tl")) t->ans_tl = (uint32_t)v;
      else if (!strcmp(key, "il")) t->ans_il = (uint32_t)v;
      else if (!strcmp(key, "stride")) t->stride = (int64_t)v;
      skip_ws(p);
      if (p->s[p->pos] == ',') { p->pos++; continue; }
      if (p->s[p->pos] == ')') { p->pos++; break; }
      p->err = 1; snprintf(g_err, sizeof g_err, "parse error at %zu: expected ',' or ')'", p->pos); free_tree(t); return NULL;
    }
    skip_ws(p);
  }
  if (p->s[p->pos] == '|') {
    p->pos++;
    skip_ws(p);
    if (p->s[p->pos] == '[') {
      p->pos++;
      for (;;) {
        if (t->nchild == 2) { p->err = 1; snprintf(g_err, sizeof g_err, "arity error: too many children at %zu", p->pos); free_tree(t); return NULL; }
        tnode *ch = parse_node(p);
        if (!ch) { free_tree(t); return NULL; }
        t->child[t->nchild++] = ch;
        skip_ws(p);
        if (p->s[p->pos] == ',') { p->pos++; continue; }
        if (p->s[p->pos] == ']') { p->pos++; break; }
        p->err = 1; snprintf(g_err, sizeof g_err, "parse error at %zu: expected ',' or ']'", p->pos); free_tree(t); return NULL;
      }
    } else {
      tnode *ch = parse_node(p);
      if (!ch) { free_tree(t); return NULL; }
      t->child[t->nchild++] = ch;
    }
  }
  return t;
}

static tnode *mk(int codec) {
  tnode *t = (tnode *)calloc(1, sizeof(tnode));
  t->codec = codec; t->lz4_sub = 65536; t->ans_chunk = 0; t->ans_tl = 12; t->ans_il = 32; t->stride = 1;
  return t;
}

/* Complete the tree to full arity (reading R30): 0 children -> all outputs Raw; 1 child binds
 * the primary stream (Dict->indices, RLE->values, Str->bytes); BitPack/LZ4 children are always Raw. */
static int complete(tnode *t) {
  switch (t->codec) {
    case C_RAW: return t->nchild == 0 ? 0 : fail(E_PARSE, "arity error: Raw takes no children");
    case C_BITPACK:
      if (t->nchild == 0) { t->child[t->nchild++] = mk(C_RAW); return 0; }
      if (t->nchild == 1 && t->child[0]->codec == C_RAW) return 0;
      if (t->nchild == 1 && t->child[0]->codec == C_ANS) break;  /* packed bytes entropy coded (Table 2 O_COMMENT) */
      return fail(E_PARSE, "arity error: BitPack's only child is Raw or ANS");
    case C_LZ4:
      if (t->nchild != 0) return fail(E_PARSE, "arity error: LZ4 takes no children");
      t->child[0] = mk(C_RAW); t->child[1] = mk(C_RAW); t->nchild = 2; return 0;
    case C_ANS:
      if (t->nchild != 0) return fail(E_PARSE, "arity error: ANS takes no children");
      t->child[0] = mk(C_RAW); t->child[1] = mk(C_RAW); t->nchild = 2; return 0;
    case C_DICT: case C_STRDICT:
      if (t->nchild == 0) { t->child[0] = mk(C_RAW); t->child[1] = mk(C_RAW); t->nchild = 2; }
      else if (t->nchild == 1) { t->child[1] = t->child[0]; t->child[0] = mk(C_RAW); t->nchild = 2; }
      if (t->child[0]->codec != C_RAW) return fail(E_PARSE, "arity error: Dict's dictionary stream is Raw");
      break;
    case C_FLOAT2INT: case C_DELTA:
      if (t->nchild == 0) { t->child[t->nchild++] = mk(C_RAW); }
      if (t->nchild != 1) return fail(E_PARSE, "arity error: Float2Int/Delta take one child");
      break;
    case C_RLE: case C_STR: case C_DSTRIDE:
      if (t->nchild == 0) { t->child[0] = mk(C_RAW); t->child[1] = mk(C_RAW); t->nchild = 2; }
      else if (t->nchild == 1) { t->child[1] = mk(C_RAW); t->nchild = 2; }
      break;
    default: return fail(E_PARSE, "unknown codec");
  }
  for (int i = 0; i < t->nchild; i++) { int rc = complete(t->child[i]); if (rc) return rc; }
  return 0;
}

static const char *NAMES[] = {"RAW", "BITPACK", "DICT", "FLOAT2INT", "DELTA", "RLE", "LZ4", "STR", "ANS", "DELTASTRIDE", "STRDICT"};
static void render(const tnode *t, char *buf, size_t cap) {
  strncat(buf, NAMES[t->codec], cap - strlen(buf) - 1);
  if (!t->nchild) return;
  strncat(buf, "|", cap - strlen(buf) - 1);
  if (t->nchild == 1) { render(t->child[0], buf, cap); return; }
  strncat(buf, "[", cap - strlen(buf) - 1);
  for (int i = 0; i < t->nchild; i++) {
    if (i) strncat(buf, ",", cap - strlen(buf) - 1);
    render(t->child[i], buf, cap);
  }
  strncat(buf, "]", cap - strlen(buf) - 1);
}

static uint64_t fnv1a(const char *s) {
  uint64_t h = 14695981039346656037ull;
  for (; *s; s++) { h ^= (uint8_t)*s; h *= 1099511628211ull; }
  return h;
}

static int parse_cascade(const char *text, tnode **out) {
  parser p = {text, 0, 0};
  tnode *t = parse_node(&p);
  if (!t) return E_PARSE;
  skip_ws(&p);
  if (p.s[p.pos]) { snprintf(g_err, sizeof g_err, "parse error at %zu: trailing input", p.pos); free_tree(t); return E_PARSE; }
  int rc = complete(t);
  if (rc) { free_tree(t); return rc; }
  *out = t;
  return 0;
}

/* Canonical text of a cascade (the text whose FNV-1a hash goes into the chunk header). */
EXPORT int cdm_encode_canonical(const char *text, char *buf, size_t cap) {
  tnode *t;
  int rc = parse_cascade(text, &t);
  if (rc) return rc;
  buf[0] = 0;
  render(t, buf, cap);
  free_tree(t);
  return 0;
}

/* ------------------------------------------------------------------ output builder */
typedef struct { uint8_t codec, nchild; uint16_t stream; uint32_t u32a; uint64_t n; uint8_t p[16]; } node_rec; /* 32 B */
typedef struct { uint8_t *data; uint64_t len; } stream_rec;

typedef struct {
  node_rec *nodes; int nn, ncap;
  stream_rec *streams; int ns, scap;
} builder;

static int add_node(builder *b, node_rec r) {
  if (b->nn == b->ncap) { b->ncap = b->ncap ? 2 * b->ncap : 16; b->nodes = (node_rec *)realloc(b->nodes, b->ncap * sizeof(node_rec)); }
  b->nodes[b->nn] = r;
  return b->nn++;
}
static int add_stream(builder *b, uint8_t *data, uint64_t len) { /* takes ownership */
  if (b->ns == b->scap) { b->scap = b->scap ? 2 * b->scap : 16; b->streams = (stream_rec *)realloc(b->streams, b->scap * sizeof(stream_rec)); }
  b->streams[b->ns].data = data; b->streams[b->ns].len = len;
  return b->ns++;
}

/* column representation during encoding */
typedef struct { uint64_t n; uint32_t eb; int is_int; uint8_t *data; const int64_t *offs; } col_t;

static int64_t *to_int(const col_t *c) {
  int64_t *v = (int64_t *)malloc((c->n ? c->n : 1) * sizeof(int64_t));
  if (!v) return NULL;
  for (uint64_t i = 0; i < c->n; i++) {
    const uint8_t *e = c->data + i * c->eb;
    if (c->is_int || c->eb == 8) { memcpy(&v[i], e, 8); }
    else if (c->eb == 4) { int32_t x; memcpy(&x, e, 4); v[i] = x; }
    else if (c->eb == 2) { uint16_t x; memcpy(&x, e, 2); v[i] = x; }
    else if (c->eb == 1) { v[i] = e[0]; }
    else { free(v); return NULL; }
  }
  return v;
}

static int encode_node(builder *b, const tnode *t, col_t in);

static int enc_int_child(builder *b, const tnode *t, int64_t *vals, uint64_t n) { /* takes ownership of vals */
  col_t c = {n, 8, 1, (uint8_t *)vals, NULL};
  int rc = encode_node(b, t, c);
  free(vals);
  return rc;
}

static int enc_raw(builder *b, col_t in) {
  uint32_t eb = in.is_int ? 8 : in.eb;
  uint64_t len = in.n * eb;
  uint8_t *d = (uint8_t *)malloc(len ? len : 1);
  if (!d) return fail(E_OOM, "out of memory");
  if (len) memcpy(d, in.data, len);
  node_rec r; memset(&r, 0, sizeof r);
  r.codec = C_RAW; r.nchild = 0; r.stream = (uint16_t)add_stream(b, d, len); r.n = in.n; r.u32a = eb;
  add_node(b, r);
  return 0;
}

/* BitPack + FOR: base = min, w = ceil(log2(max-min+1)), LSB-first contiguous bits. */
static int enc_bitpack(builder *b, const tnode *t, col_t in) {
  int64_t *v = to_int(&in);
  if (!v) return fail(E_UNSUPPORTED, "BitPack needs an integer stream");
  int64_t mn = 0, mx = 0;
  for (uint64_t i = 0; i < in.n; i++) { if (!i || v[i] < mn) mn = v[i]; if (!i || v[i] > mx) mx = v[i]; }
  uint64_t range = (uint64_t)mx - (uint64_t)mn;
  int w = 0;
  while (w < 64 && (range >> w) != 0) w++;
  uint64_t nbytes = (in.n * (uint64_t)w + 7) / 8;
  uint8_t *pk = (uint8_t *)calloc(nbytes + 16, 1);
  if (!pk) { free(v); return fail(E_OOM, "out of memory"); }
  /* value i occupies bits [i*w, i*w + w): OR it into the little-endian 8-byte word at its first byte, and
   * its top bits into the next word when it crosses (the buffer has 16 slack bytes) */
  for (uint64_t i = 0; w && i < in.n; i++) {
    uint64_t f = (uint64_t)v[i] - (uint64_t)mn;
    uint64_t bit = i * (uint64_t)w;
    unsigned sh = (unsigned)(bit & 7);
    uint8_t *p = pk + (bit >> 3);
    uint64_t word;
    memcpy(&word, p, 8); word |= f << sh; memcpy(p, &word, 8);
    if (sh + (unsigned)w > 64) { memcpy(&word, p + 8, 8); word |= f >> (64 - sh); memcpy(p + 8, &word, 8); }
  }
  free(v);
  node_rec r; memset(&r, 0, sizeof r);
  r.codec = C_BITPACK; r.nchild = 1; r.stream = 0xFFFF; r.n = in.n;
  r.p[0] = (uint8_t)w; memcpy(r.p + 8, &mn, 8);
  add_node(b, r);
  if (t && t->nchild == 1 && t->child[0]->codec == C_ANS) {  /* the packed bytes go through ANS */
    col_t pc = {nbytes, 1, 0, pk, NULL};
    int rc = encode_node(b, t->child[0], pc);
    free(pk);
    return rc;
  }
  node_rec raw; memset(&raw, 0, sizeof raw);
  raw.codec = C_RAW; raw.stream = (uint16_t)add_stream(b, pk, nbytes); raw.n = nbytes; raw.u32a = 1;
  add_node(b, raw);
  return 0;
}

static uint32_t g_sort_eb;
static const uint8_t *g_sort_base;
static int cmp_elem(const void *a, const void *c) { return memcmp(a, c, g_sort_eb); }

static uint64_t hash_bytes(const uint8_t *p, uint32_t n) {
  uint64_t h = 14695981039346656037ull;
  for (uint32_t i = 0; i < n; i++) { h ^= p[i]; h *= 1099511628211ull; }
  return h ^ (h >> 29);
}

/* Dictionary: unique elements sorted by unsigned bytes; indices into the dictionary.
 * Unique elements are found with an open-addressing hash table (O(n)), then only the uniques are sorted. */
static int enc_dict(builder *b, const tnode *t, col_t in) {
  uint32_t eb = in.is_int ? 8 : in.eb;
  uint64_t cap = 16;
  while (cap < 2 * (in.n ? in.n : 1) && cap < (1ull << 33)) cap <<= 1;
  /* table of first-occurrence element indices, +1 (0 = empty) */
  uint64_t *tab = (uint64_t *)calloc(cap, sizeof(uint64_t));
  int64_t *idx = (int64_t *)malloc((in.n ? in.n : 1) * sizeof(int64_t));
  uint8_t *uniq = (uint8_t *)malloc((in.n ? in.n : 1) * eb);
  uint64_t *slot_of = (uint64_t *)malloc((in.n ? in.n : 1) * sizeof(uint64_t));
  if (!tab || !idx || !uniq || !slot_of) { free(tab); free(idx); free(uniq); free(slot_of); return fail(E_OOM, "out of memory"); }
  uint64_t nu = 0;
  for (uint64_t i = 0; i < in.n; i++) {
    const uint8_t *e = in.data + i * eb;
    uint64_t h = hash_bytes(e, eb) & (cap - 1);
    for (;;) {
      if (!tab[h]) { memcpy(uniq + nu * eb, e, eb); tab[h] = ++nu; break; }
      if (!memcmp(uniq + (tab[h] - 1) * eb, e, eb)) break;
      h = (h + 1) & (cap - 1);
    }
    slot_of[i] = tab[h] - 1;  /* provisional (first-appearance) id */
  }
  /* sort the uniques by bytes; remap provisional ids to sorted positions */
  uint8_t *sorted = (uint8_t *)malloc((nu ? nu : 1) * eb);
  memcpy(sorted, uniq, nu * eb);
  g_sort_eb = eb;
  qsort(sorted, nu, eb, cmp_elem);
  uint64_t *remap = (uint64_t *)malloc((nu ? nu : 1) * sizeof(uint64_t));
  for (uint64_t u = 0; u < nu; u++) {
    /* binary search uniq[u] in sorted */
    uint64_t lo = 0, hi = nu;
    while (lo < hi) {
      uint64_t mid = (lo + hi) / 2;
      if (memcmp(sorted + mid * eb, uniq + u * eb, eb) < 0) lo = mid + 1; else hi = mid;
    }
    remap[u] = lo;
  }
  for (uint64_t i = 0; i < in.n; i++) idx[i] = (int64_t)remap[slot_of[i]];
  free(tab); free(uniq); free(slot_of); free(remap);
  if (nu > 0xFFFFFFFFull) { free(sorted); free(idx); return fail(E_UNSUPPORTED, "dictionary too large"); }
  node_rec r; memset(&r, 0, sizeof r);
  r.codec = C_DICT; r.nchild = 2; r.stream = 0xFFFF; r.n = in.n;
  uint32_t ent32 = (uint32_t)nu; memcpy(r.p, &ent32, 4); memcpy(r.p + 4, &eb, 4);
  add_node(b, r);
  col_t dc = {nu, eb, 0, sorted, NULL};
  int rc = enc_raw(b, dc);
  free(sorted);
  if (rc) { free(idx); return rc; }
  return enc_int_child(b, t->child[1], idx, in.n);
}

/* Float2Int: smallest d with (double)llrint(x*10^d) / 10^d reproducing x bit-exactly. */
static const double POW10[19] = {1e0, 1e1, 1e2, 1e3, 1e4, 1e5, 1e6, 1e7, 1e8, 1e9, 1e10, 1e11, 1e12, 1e13,
                                 1e14, 1e15, 1e16, 1e17, 1e18};
static int enc_float2int(builder *b, const tnode *t, col_t in) {
  if (in.is_int || in.eb != 8) return fail(E_UNSUPPORTED, "Float2Int needs a float64 stream");
  const double *x = (const double *)in.data;
  int64_t *v = (int64_t *)malloc((in.n ? in.n : 1) * sizeof(int64_t));
  int d;
  for (d = 0; d <= 18; d++) {
    uint64_t i;
    for (i = 0; i < in.n; i++) {
      double s = x[i] * POW10[d];
      if (!(s > -9.2e18 && s < 9.2e18)) break;
      long long q = llrint(s);
      double back = (double)q / POW10[d];
      if (memcmp(&back, &x[i], 8)) break;
      v[i] = q;
    }
    if (i == in.n) break;
  }
  if (d > 18) { free(v); return fail(E_UNSUPPORTED, "Float2Int: column not decimal-representable (d<=18)"); }
  node_rec r; memset(&r, 0, sizeof r);
  r.codec = C_FLOAT2INT; r.nchild = 1; r.stream = 0xFFFF; r.n = in.n; r.p[0] = (uint8_t)d;
  add_node(b, r);
  return enc_int_child(b, t->child[0], v, in.n);
}

/* Delta: base = x[0], d[0] = 0, d[i] = x[i] - x[i-1] (mod 2^64). */
static int enc_delta(builder *b, const tnode *t, col_t in) {
  int64_t *v = to_int(&in);
  if (!v) return fail(E_UNSUPPORTED, "Delta needs an integer stream");
  int64_t base = in.n ? v[0] : 0;
  for (uint64_t i = in.n; i-- > 1;) v[i] = (int64_t)((uint64_t)v[i] - (uint64_t)v[i - 1]);
  if (in.n) v[0] = 0;
  node_rec r; memset(&r, 0, sizeof r);
  r.codec = C_DELTA; r.nchild = 1; r.stream = 0xFFFF; r.n = in.n; memcpy(r.p + 8, &base, 8);
  add_node(b, r);
  return enc_int_child(b, t->child[0], v, in.n);
}

/* RLE: maximal runs of equal elements -> values, counts. */
static int enc_rle(builder *b, const tnode *t, col_t in) {
  uint32_t eb = in.is_int ? 8 : in.eb;
  uint8_t *vals = (uint8_t *)malloc((in.n ? in.n : 1) * eb);
  int64_t *cnt = (int64_t *)malloc((in.n ? in.n : 1) * sizeof(int64_t));
  uint64_t nr = 0, maxrun = 0;
  for (uint64_t i = 0; i < in.n; i++) {
    const uint8_t *e = in.data + i * eb;
    if (nr && !memcmp(vals + (nr - 1) * eb, e, eb)) cnt[nr - 1]++;
    else { memcpy(vals + nr * eb, e, eb); cnt[nr] = 1; nr++; }
  }
  for (uint64_t g = 0; g < nr; g++) if ((uint64_t)cnt[g] > maxrun) maxrun = (uint64_t)cnt[g];
  node_rec r; memset(&r, 0, sizeof r);
  r.codec = C_RLE; r.nchild = 2; r.stream = 0xFFFF; r.n = in.n;
  uint32_t nr32 = (uint32_t)nr, mr32 = (uint32_t)(maxrun > 0xFFFFFFFFull ? 0xFFFFFFFFull : maxrun);
  memcpy(r.p, &nr32, 4); memcpy(r.p + 4, &mr32, 4);
  add_node(b, r);
  col_t vc = {nr, eb, in.is_int, vals, NULL};
  int rc = encode_node(b, t->child[0], vc);
  free(vals);
  if (rc) { free(cnt); return rc; }
  return enc_int_child(b, t->child[1], cnt, nr);
}

/* DeltaStride (reading R9): greedy maximal arithmetic runs x, x+k, x+2k, ... for the node's stride
 * k (mod 2^64) -> starts, counts. */
static int enc_dstride(builder *b, const tnode *t, col_t in) {
  int64_t *v = to_int(&in);
  if (!v) return fail(E_UNSUPPORTED, "DeltaStride needs an integer stream");
  const uint64_t k = (uint64_t)t->stride;
  int64_t *st = (int64_t *)malloc((in.n ? in.n : 1) * sizeof(int64_t));
  int64_t *cnt = (int64_t *)malloc((in.n ? in.n : 1) * sizeof(int64_t));
  uint64_t nr = 0, maxrun = 0;
  for (uint64_t i = 0; i < in.n; i++) {
    if (nr && (uint64_t)v[i] - (uint64_t)v[i - 1] == k) cnt[nr - 1]++;
    else { st[nr] = v[i]; cnt[nr] = 1; nr++; }
  }
  free(v);
  for (uint64_t g = 0; g < nr; g++) if ((uint64_t)cnt[g] > maxrun) maxrun = (uint64_t)cnt[g];
  node_rec r; memset(&r, 0, sizeof r);
  r.codec = C_DSTRIDE; r.nchild = 2; r.stream = 0xFFFF; r.n = in.n;
  uint32_t nr32 = (uint32_t)nr, mr32 = (uint32_t)(maxrun > 0xFFFFFFFFull ? 0xFFFFFFFFull : maxrun);
  memcpy(r.p, &nr32, 4); memcpy(r.p + 4, &mr32, 4); memcpy(r.p + 8, &k, 8);
  add_node(b, r);
  int rc = enc_int_child(b, t->child[0], st, nr);
  if (rc) { free(cnt); return rc; }
  return enc_int_child(b, t->child[1], cnt, nr);
}

/* LZ4 block format per independent sub-chunk of `sub` decompressed bytes. */
static int enc_lz4(builder *b, const tnode *t, col_t in) {
  if (in.is_int || in.eb != 1) return fail(E_UNSUPPORTED, "LZ4 needs a byte stream");
  uint32_t sub = t->lz4_sub;
  if (sub < 16 || sub > (1u << 24)) return fail(E_INVALID_ARG, "LZ4 sub-chunk size out of range");
  uint64_t nsub = (in.n + sub - 1) / sub;
  uint64_t cap = nsub * (uint64_t)LZ4_compressBound((int)sub) + 16;
  uint8_t *pay = (uint8_t *)malloc(cap);
  uint8_t *tab = (uint8_t *)malloc(nsub * 12 + 1);
  if (!pay || !tab) { free(pay); free(tab); return fail(E_OOM, "out of memory"); }
  uint64_t pos = 0;
  for (uint64_t s = 0; s < nsub; s++) {
    uint32_t dl = (uint32_t)((s + 1 == nsub) ? in.n - s * sub : sub);
    int cl = t->lz4_hc ? LZ4_compress_HC((const char *)in.data + s * sub, (char *)pay + pos, (int)dl, (int)(cap - pos), t->lz4_hc)
                       : LZ4_compress_default((const char *)in.data + s * sub, (char *)pay + pos, (int)dl, (int)(cap - pos));
    if (cl <= 0) { free(pay); free(tab); return fail(E_UNSUPPORTED, "LZ4 compression failed"); }
    uint32_t co = (uint32_t)pos, cl32 = (uint32_t)cl;
    memcpy(tab + s * 12, &co, 4); memcpy(tab + s * 12 + 4, &cl32, 4); memcpy(tab + s * 12 + 8, &dl, 4);
    pos += (uint64_t)cl;
    if (pos > 0xFFFFFFFFull) { free(pay); free(tab); return fail(E_UNSUPPORTED, "LZ4 payload too large"); }
  }
  node_rec r; memset(&r, 0, sizeof r);
  r.codec = C_LZ4; r.nchild = 2; r.stream = 0xFFFF; r.n = in.n;
  uint32_t ns32 = (uint32_t)nsub; memcpy(r.p, &ns32, 4); memcpy(r.p + 4, &sub, 4);
  add_node(b, r);
  node_rec raw; memset(&raw, 0, sizeof raw);
  raw.codec = C_RAW; raw.stream = (uint16_t)add_stream(b, pay, pos); raw.n = pos; raw.u32a = 1;
  add_node(b, raw);
  memset(&raw, 0, sizeof raw);
  raw.codec = C_RAW; raw.stream = (uint16_t)add_stream(b, tab, nsub * 12); raw.n = nsub; raw.u32a = 12;
  add_node(b, raw);
  return 0;
}

/* ANS (reading R32): range-ANS over a byte stream, cut
 * into independently coded chunks of `chunk` bytes that share one table normalised to 2^tl.  32-bit states
 * in [L, 2^32), L = 2^16, 16-bit renormalisation words (at most one per symbol for tl <= 16).
 * il = 1: one state per chunk; symbols are coded back to front from state L.
 * il = 32 (default): 32 interleaved states per chunk, symbol i belongs to state i mod 32 at step i div 32.
 *   Decode order = step-major, state-minor; the encoder runs exactly the reverse order (steps descending,
 *   states descending) pushing its words, and the chunk's word list is that push order reversed -- so at
 *   every decode step the states that renormalise take consecutive words in state order.
 * Every chunk stores its initial decoder state(s) and its words in decode order; a decoder must end with
 * every state at L and every word read.
 * Streams: [0] u16 words of all chunks; [1] table = 256 x u16 frequencies, then per chunk
 * {u32 first word, u32 words, il x u32 initial decoder states}.  Node params: u32 chunks @0,
 * u32 chunk bytes @4, u8 tl @8, u8 il @9. */
static int enc_ans(builder *b, const tnode *t, col_t in) {
  if (in.is_int) return fail(E_UNSUPPORTED, "ANS needs a byte stream");
  const uint32_t tl = t->ans_tl, il = t->ans_il;
  const uint32_t chunk = t->ans_chunk ? t->ans_chunk : (il == 32 ? 16384 : 4096);
  if (tl < 8 || tl > 15) return fail(E_INVALID_ARG, "ANS table log out of range [8, 15]");
  if (il != 1 && il != 32) return fail(E_INVALID_ARG, "ANS interleave must be 1 or 32");
  if (chunk < 16 || chunk > (1u << 24) || (chunk & 15)) return fail(E_INVALID_ARG, "ANS chunk size: multiple of 16 in [16, 2^24]");
  const uint64_t n = in.n * in.eb;
  const uint8_t *src = in.data;
  const uint32_t M = 1u << tl;
  uint64_t cnt[256] = {0};
  for (uint64_t i = 0; i < n; i++) cnt[src[i]]++;
  uint32_t f[256] = {0}, cum[257];
  if (n) {  /* normalise: floor(cnt*M/n), at least 1 for present symbols, then fix the sum on the largest */
    int64_t sum = 0;
    for (int s = 0; s < 256; s++) {
      if (!cnt[s]) continue;
      uint64_t v = cnt[s] * M / n;
      f[s] = (uint32_t)(v ? v : 1);
      sum += f[s];
    }
    while (sum != (int64_t)M) {
      int s_adj = -1;  /* the largest frequency that can still move */
      for (int s = 0; s < 256; s++)
        if (f[s] && (sum < (int64_t)M || f[s] > 1) && (s_adj < 0 || f[s] > f[s_adj])) s_adj = s;
      if (s_adj < 0) return fail(E_UNSUPPORTED, "ANS: more distinct symbols than 2^tl");
      if (sum < (int64_t)M) { f[s_adj] += (uint32_t)((int64_t)M - sum); sum = M; }
      else { f[s_adj]--; sum--; }
    }
  }
  cum[0] = 0;
  for (int s = 0; s < 256; s++) cum[s + 1] = cum[s] + f[s];
  const uint64_t nch = (n + chunk - 1) / chunk;
  const uint32_t L = 1u << 16;
  const uint64_t rec = 8 + 4ull * il;
  uint16_t *words = (uint16_t *)malloc((n + 16) * sizeof(uint16_t));  /* <= 1 word per symbol */
  uint16_t *tmp = (uint16_t *)malloc(((uint64_t)chunk + 16) * sizeof(uint16_t));
  uint64_t tbytes = 512 + rec * nch;
  uint8_t *tab = (uint8_t *)calloc(tbytes + 16, 1);
  if (!words || !tmp || !tab) { free(words); free(tmp); free(tab); return fail(E_OOM, "out of memory"); }
  for (int s = 0; s < 256; s++) { uint16_t v = (uint16_t)f[s]; memcpy(tab + 2 * s, &v, 2); }
  uint64_t wpos = 0;
  for (uint64_t c = 0; c < nch; c++) {
    const uint64_t c0 = c * chunk, c1 = (c0 + chunk < n) ? c0 + chunk : n;
    uint32_t x[32];
    for (uint32_t l = 0; l < il; l++) x[l] = L;
    uint64_t k = 0;
    for (uint64_t i = c1; i-- > c0;) {  /* reverse decode order: steps descending, states descending */
      const uint32_t l = il == 1 ? 0 : (uint32_t)((i - c0) & 31);
      const uint32_t s = src[i], fs = f[s];
      const uint64_t x_max = ((uint64_t)(L >> tl) << 16) * fs;
      while ((uint64_t)x[l] >= x_max) { tmp[k++] = (uint16_t)(x[l] & 0xFFFF); x[l] >>= 16; }
      x[l] = ((x[l] / fs) << tl) + (x[l] % fs) + cum[s];
    }
    const uint32_t first = (uint32_t)wpos, nw = (uint32_t)k;
    for (uint64_t j = 0; j < k; j++) words[wpos++] = tmp[k - 1 - j];  /* decode order */
    memcpy(tab + 512 + rec * c, &first, 4); memcpy(tab + 512 + rec * c + 4, &nw, 4);
    for (uint32_t l = 0; l < il; l++) memcpy(tab + 512 + rec * c + 8 + 4 * l, &x[l], 4);
    if (wpos > 0xFFFFFFFFull) { free(words); free(tmp); free(tab); return fail(E_UNSUPPORTED, "ANS payload too large"); }
  }
  free(tmp);
  node_rec r; memset(&r, 0, sizeof r);
  r.codec = C_ANS; r.nchild = 2; r.stream = 0xFFFF; r.n = n;
  uint32_t nch32 = (uint32_t)nch;
  memcpy(r.p, &nch32, 4); memcpy(r.p + 4, &chunk, 4); r.p[8] = (uint8_t)tl; r.p[9] = (uint8_t)il;
  add_node(b, r);
  node_rec raw; memset(&raw, 0, sizeof raw);
  raw.codec = C_RAW; raw.stream = (uint16_t)add_stream(b, (uint8_t *)words, wpos * 2); raw.n = wpos; raw.u32a = 2;
  add_node(b, raw);
  memset(&raw, 0, sizeof raw);
  raw.codec = C_RAW; raw.stream = (uint16_t)add_stream(b, tab, tbytes); raw.n = tbytes; raw.u32a = 1;
  add_node(b, raw);
  return 0;
}

/* Str: VARBYTES rows -> [concatenated bytes, per-row lengths]. */
/* String-dictionary ("tokenizing on spaces and periods"; reading R34): a token
 * is a maximal run of non-delimiter bytes followed by its trailing delimiters (space, period), cut at string
 * boundaries and at kStrDictMaxTok bytes; the dictionary holds the unique tokens in first-appearance order.
 * Children: [Raw dictionary = u32 offsets[E+1] (from the token bytes' start) + token bytes, token ids]. */
static __thread const int64_t *g_str_offs;
static __thread uint64_t g_str_rows;
#define kStrDictMaxTok 32u
static int sd_delim(uint8_t c) { return c == ' ' || c == '.'; }
static int enc_strdict(builder *b, const tnode *t, col_t in) {
  if (in.is_int || in.eb != 1) return fail(E_UNSUPPORTED, "StrDict needs a byte stream");
  const uint8_t *d = in.data;
  uint64_t *ts = (uint64_t *)malloc((in.n + 1) * sizeof(uint64_t)); /* token starts; ts[ntok] = n */
  uint64_t ntok = 0;
  const int64_t *so = g_str_offs;
  uint64_t srow = 0, next_bound = so ? (uint64_t)(so[1] - so[0]) : in.n;
  for (uint64_t i = 0; i < in.n; i++) {
    int start = ntok == 0;
    while (so && srow < g_str_rows && i >= next_bound) { /* string boundary (skips empty strings) */
      start = 1; srow++;
      next_bound = srow < g_str_rows ? (uint64_t)(so[srow + 1] - so[0]) : in.n;
    }
    if (!start && !sd_delim(d[i]) && sd_delim(d[i - 1])) start = 1;
    if (!start && i - ts[ntok - 1] >= kStrDictMaxTok) start = 1;
    if (start) ts[ntok++] = i;
  }
  ts[ntok] = in.n;
  uint64_t cap = 16;
  while (cap < 2 * (ntok ? ntok : 1)) cap <<= 1;
  uint64_t *tab = (uint64_t *)calloc(cap, sizeof(uint64_t)); /* slot -> 1 + first token index */
  int64_t *ids = (int64_t *)malloc((ntok ? ntok : 1) * sizeof(int64_t));
  uint64_t *first = (uint64_t *)malloc((ntok ? ntok : 1) * sizeof(uint64_t)); /* id -> a token index */
  uint32_t *id_of_slot = (uint32_t *)malloc(cap * sizeof(uint32_t));
  if (!ts || !tab || !ids || !first || !id_of_slot) { free(ts); free(tab); free(ids); free(first); free(id_of_slot); return fail(E_OOM, "out of memory"); }
  uint64_t E = 0, dbytes = 0;
  for (uint64_t k = 0; k < ntok; k++) {
    const uint8_t *tk = d + ts[k];
    const uint32_t tn = (uint32_t)(ts[k + 1] - ts[k]);
    uint64_t h = hash_bytes(tk, tn) & (cap - 1);
    for (;;) {
      if (!tab[h]) { tab[h] = k + 1; id_of_slot[h] = (uint32_t)E; first[E++] = k; dbytes += tn; break; }
      const uint64_t o = tab[h] - 1;
      if (ts[o + 1] - ts[o] == tn && !memcmp(d + ts[o], tk, tn)) break;
      h = (h + 1) & (cap - 1);
    }
    ids[k] = id_of_slot[h];
  }
  uint64_t dlen = 4 * (E + 1) + dbytes;
  uint8_t *dict = (uint8_t *)malloc(dlen ? dlen : 1);
  uint32_t off = 0;
  for (uint64_t e = 0; e < E; e++) {
    const uint32_t tn = (uint32_t)(ts[first[e] + 1] - ts[first[e]]);
    memcpy(dict + 4 * e, &off, 4);
    memcpy(dict + 4 * (E + 1) + off, d + ts[first[e]], tn);
    off += tn;
  }
  memcpy(dict + 4 * E, &off, 4);
  free(ts); free(tab); free(first); free(id_of_slot);
  if (E > 0xFFFFFFFFull || dbytes > 0xFFFFFFFFull) { free(dict); free(ids); return fail(E_CAPACITY, "StrDict dictionary too large"); }
  node_rec r; memset(&r, 0, sizeof r);
  r.codec = C_STRDICT; r.nchild = 2; r.stream = 0xFFFF; r.n = in.n;
  uint32_t e32 = (uint32_t)E, db32 = (uint32_t)dbytes, mt = kStrDictMaxTok;
  memcpy(r.p, &e32, 4); memcpy(r.p + 4, &db32, 4); memcpy(r.p + 8, &mt, 4);
  add_node(b, r);
  col_t dc = {dlen, 1, 0, dict, NULL};
  int rc = enc_raw(b, dc);
  free(dict);
  if (rc) { free(ids); return rc; }
  return enc_int_child(b, t->child[1], ids, ntok);
}

static int enc_str(builder *b, const tnode *t, col_t in) {
  if (!in.offs) return fail(E_UNSUPPORTED, "Str needs a VARBYTES column");
  int64_t *len = (int64_t *)malloc((in.n ? in.n : 1) * sizeof(int64_t));
  for (uint64_t i = 0; i < in.n; i++) len[i] = in.offs[i + 1] - in.offs[i];
  uint64_t nbytes = (uint64_t)(in.offs[in.n] - in.offs[0]);
  node_rec r; memset(&r, 0, sizeof r);
  r.codec = C_STR; r.nchild = 2; r.stream = 0xFFFF; r.n = in.n;
  add_node(b, r);
  col_t bc = {nbytes, 1, 0, in.data + in.offs[0], NULL};
  g_str_offs = in.offs; g_str_rows = in.n;  /* string boundaries for a String-dictionary bytes child */
  int rc = encode_node(b, t->child[0], bc);
  g_str_offs = NULL; g_str_rows = 0;
  if (rc) { free(len); return rc; }
  return enc_int_child(b, t->child[1], len, in.n);
}

static int encode_node(builder *b, const tnode *t, col_t in) {
  if (in.offs && t->codec != C_STR) return fail(E_UNSUPPORTED, "VARBYTES columns need a Str root");
  switch (t->codec) {
    case C_RAW: return enc_raw(b, in);
    case C_BITPACK: return enc_bitpack(b, t, in);
    case C_STRDICT: return enc_strdict(b, t, in);
    case C_DICT: return enc_dict(b, t, in);
    case C_FLOAT2INT: return enc_float2int(b, t, in);
    case C_DELTA: return enc_delta(b, t, in);
    case C_RLE: return enc_rle(b, t, in);
    case C_LZ4: return enc_lz4(b, t, in);
    case C_STR: return enc_str(b, t, in);
    case C_ANS: return enc_ans(b, t, in);
    case C_DSTRIDE: return enc_dstride(b, t, in);
  }
  return fail(E_UNSUPPORTED, "unknown codec");
}

static inline uint64_t rup16(uint64_t x) { return (x + 15) & ~15ull; }

/*
 * Encode `rows` rows of one column under `cascade` into a freshly malloc'ed CDM1 chunk.
 *   dtype: 0 I32, 1 I64, 2 F64, 3 FIXED(width), 4 VARBYTES (offsets = rows+1 int64, exclusive end)
 *   *out_buf must be released with cdm_encode_free().  Returns 0 or an error code (cdm_encode_error()).
 */
EXPORT int cdm_encode(const char *cascade, int dtype, uint32_t width, const void *plain, const int64_t *offsets,
                      uint64_t rows, uint64_t chunk_id, void **out_buf, size_t *out_len) {
  if (!cascade || !out_buf || !out_len || (rows && !plain)) return fail(E_INVALID_ARG, "null argument");
  uint32_t eb;
  switch (dtype) {
    case D_I32: eb = 4; break;
    case D_I64: case D_F64: eb = 8; break;
    case D_FIXED: eb = width; if (!eb) return fail(E_INVALID_ARG, "FIXED needs width > 0"); break;
    case D_VARBYTES: eb = 1; if (!offsets) return fail(E_INVALID_ARG, "VARBYTES needs offsets"); break;
    default: return fail(E_INVALID_ARG, "bad dtype");
  }
  if (rows >= (1ull << 31)) return fail(E_INVALID_ARG, "a chunk holds fewer than 2^31 rows");
  tnode *t;
  int rc = parse_cascade(cascade, &t);
  if (rc) return rc;
  char canon[512] = {0};
  render(t, canon, sizeof canon);
  builder b; memset(&b, 0, sizeof b);
  static const uint8_t empty[16] = {0};
  col_t in = {rows, eb, 0, plain ? (uint8_t *)plain : (uint8_t *)empty, dtype == D_VARBYTES ? offsets : NULL};
  rc = encode_node(&b, t, in);
  free_tree(t);
  if (!rc && (b.nn > 0xFFFF || b.ns > 0xFFFF)) rc = fail(E_UNSUPPORTED, "too many nodes");
  if (rc) {
    for (int i = 0; i < b.ns; i++) free(b.streams[i].data);
    free(b.streams); free(b.nodes);
    return rc;
  }
  uint64_t payload = dtype == D_VARBYTES ? (uint64_t)(offsets[rows] - offsets[0]) : rows * eb;
  uint64_t offs_bytes = dtype == D_VARBYTES ? 4 * (rows + 1) : 0;
  uint64_t hdr = rup16(64 + 32ull * b.nn + 16ull * b.ns);
  uint64_t total = hdr;
  uint64_t *soff = (uint64_t *)malloc((b.ns + 1) * sizeof(uint64_t));
  for (int i = 0; i < b.ns; i++) { soff[i] = total; total += rup16(b.streams[i].len) + 16; }
  uint8_t *o = (uint8_t *)calloc(total, 1);
  if (!o) { free(soff); return fail(E_OOM, "out of memory"); }
  uint32_t magic = 0x314D4443u; /* "CDM1" */
  uint16_t ver = 1, nn = (uint16_t)b.nn, ns = (uint16_t)b.ns;
  uint8_t dt = (uint8_t)dtype;
  uint64_t h = fnv1a(canon);
  memcpy(o + 0, &magic, 4); memcpy(o + 4, &ver, 2); memcpy(o + 6, &nn, 2); memcpy(o + 8, &ns, 2);
  o[10] = dt; memcpy(o + 12, &eb, 4); memcpy(o + 16, &rows, 8); memcpy(o + 24, &payload, 8);
  memcpy(o + 32, &offs_bytes, 8); memcpy(o + 40, &total, 8); memcpy(o + 48, &h, 8); memcpy(o + 56, &chunk_id, 8);
  memcpy(o + 64, b.nodes, 32ull * b.nn);
  for (int i = 0; i < b.ns; i++) {
    memcpy(o + 64 + 32ull * b.nn + 16ull * i, &soff[i], 8);
    memcpy(o + 64 + 32ull * b.nn + 16ull * i + 8, &b.streams[i].len, 8);
    if (b.streams[i].len) memcpy(o + soff[i], b.streams[i].data, b.streams[i].len);
    free(b.streams[i].data);
  }
  free(soff); free(b.streams); free(b.nodes);
  *out_buf = o;
  *out_len = total;
  return 0;
}

EXPORT void cdm_encode_free(void *p) { free(p); }
