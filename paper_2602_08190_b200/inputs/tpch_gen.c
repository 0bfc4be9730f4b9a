/*
 * tpch_gen.c -- seeded, counter-based, dbgen-LIKE synthetic TPC-H lineitem/orders columns.
 *
 * INPUT GENERATOR ONLY.  This module holds none of the decode method's arithmetic: it produces the
 * plain columns that the CPU encoder compresses and that both the CUDA path and the oracle are
 * checked against.  Every value is a pure function of
 * (seed, field, order index, line index), so any row range of any column is generated
 * independently (chunk-parallel, SURVEY §8d "Generator rules").
 *
 * The rules follow the TPC-H v3 dbgen conventions from memory [ext] -- they are "dbgen-like", not
 * dbgen's RNG streams:  orders = 1.5M*SF, sparse o_orderkey (first 8 of every 32), 1..7 lines per
 * order, l_partkey U[1,200k*SF], dbgen supplier formula, quantity U[1,50], discount U{0..10}/100,
 * tax U{0..8}/100, extendedprice = qty*retail(partkey) in cents, date rules around 1995-06-17,
 * grammar-text comments of length U[10,43] (lineitem) / U[19,78] (orders) / U[49,198] (partsupp);
 * partsupp = 4 rows per part (800K*SF): ps_partkey, dbgen's ps_suppkey formula, availqty U[1,9999],
 * supplycost U[100,100000] cents (Table 2's PS_PARTKEY / PS_SUPPKEY / PS_SUPPLYCOST rows).
 * Dates are date32 (days since 1970-01-01): 1992-01-01 = 8035, 1995-06-17 = 9298.
 * The paper pins: L_PARTKEY packs to 25 bits at SF=100, RLE counts are 12.5% of an
 * int64 L_ORDERKEY -> ~4 lines per order.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

#define EXPORT __attribute__((visibility("default")))

enum { T_LINEITEM = 0, T_ORDERS = 1, T_PARTSUPP = 2 };
enum {  /* lineitem columns */
  L_ORDERKEY = 0, L_PARTKEY, L_SUPPKEY, L_LINENUMBER, L_QUANTITY, L_EXTENDEDPRICE, L_DISCOUNT, L_TAX,
  L_RETURNFLAG, L_LINESTATUS, L_SHIPDATE, L_COMMITDATE, L_RECEIPTDATE, L_SHIPINSTRUCT, L_SHIPMODE,
  L_COMMENT, L_NCOLS
};
enum {  /* orders columns */
  O_ORDERKEY = 0, O_CUSTKEY, O_ORDERSTATUS, O_TOTALPRICE, O_ORDERDATE, O_ORDERPRIORITY, O_CLERK,
  O_SHIPPRIORITY, O_COMMENT, O_NCOLS
};
enum {  /* partsupp columns: 4 rows per part, PS_PARTKEY = the part's key (TPC-H 4.2.3) */
  PS_PARTKEY = 0, PS_SUPPKEY, PS_AVAILQTY, PS_SUPPLYCOST, PS_COMMENT, PS_NCOLS
};

#define STARTDATE 8035
#define ENDDATE 10591
#define CURRENTDATE 9298
#define POOL_BYTES (1u << 22)

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* field ids for the counter-based stream */
enum { F_LINES = 1, F_CUST, F_ODATE, F_OPRIO, F_CLERK, F_OCOMLEN, F_OCOMOFF,
       F_PART = 16, F_SUPPI, F_QTY, F_DISC, F_TAX, F_SHIPD, F_COMMITD, F_RECEIPTD, F_RFLAG,
       F_INSTR, F_MODE, F_LCOMLEN, F_LCOMOFF, F_AVAILQTY = 32, F_SUPPLYCOST, F_PSCOMLEN, F_PSCOMOFF,
       F_POOL = 40 };

typedef struct {
  double sf;
  uint64_t seed;
  uint64_t n_orders;
  uint64_t n_lines;
  uint32_t *line_prefix;  /* n_orders+1 cumulative line counts (fits u32 up to SF~700) */
  uint64_t *line_prefix64;/* used when n_lines >= 2^32 */
  char *pool;
} gen_ctx;

static inline uint64_t rnd(const gen_ctx *g, uint32_t field, uint64_t idx) {
  return splitmix64(splitmix64(g->seed ^ ((uint64_t)field << 48)) ^ idx);
}
static inline int64_t unif(const gen_ctx *g, uint32_t field, uint64_t idx, int64_t lo, int64_t hi) {
  return lo + (int64_t)((rnd(g, field, idx) >> 8) % (uint64_t)(hi - lo + 1));
}
static inline uint64_t lp(const gen_ctx *g, uint64_t o) {
  return g->line_prefix64 ? g->line_prefix64[o] : g->line_prefix[o];
}

/* Grammar word lists in the spirit of TPC-H 4.2.2.10 [ext]. */
static const char *NOUNS[] = {"foxes", "ideas", "theodolites", "pinto beans", "instructions", "dependencies",
  "excuses", "platelets", "asymptotes", "courts", "dolphins", "multipliers", "sauternes", "warthogs",
  "frets", "dinos", "attainments", "somas", "Tiresias'", "patterns", "forges", "braids", "hockey players",
  "frays", "warhorses", "dugouts", "notornis", "epitaphs", "pearls", "tithes", "waters", "orbits", "gifts",
  "sheaves", "depths", "sentiments", "decoys", "realms", "pains", "grouches", "escapades", "accounts",
  "deposits", "packages", "requests", "theodolites", "packages", "requests"};
static const char *VERBS[] = {"sleep", "wake", "are", "cajole", "haggle", "nag", "use", "boost", "affix",
  "detect", "integrate", "maintain", "nod", "was", "lose", "sublate", "solve", "thrash", "promise",
  "engage", "hinder", "print", "x-ray", "breach", "eat", "grow", "impress", "mold", "poach", "serve",
  "run", "dazzle", "snooze", "doze", "unwind", "kindle", "play", "hang", "believe", "doubt"};
static const char *ADJS[] = {"furious", "sly", "careful", "blithe", "quick", "fluffy", "slow", "quiet",
  "ruthless", "thin", "close", "dogged", "daring", "brave", "stealthy", "permanent", "enticing", "idle",
  "busy", "regular", "final", "ironic", "even", "bold", "silent"};
static const char *ADVS[] = {"sometimes", "always", "never", "furiously", "slyly", "carefully", "blithely",
  "quickly", "fluffily", "slowly", "quietly", "ruthlessly", "thinly", "closely", "doggedly", "daringly",
  "bravely", "stealthily", "permanently", "enticingly", "idly", "busily", "regularly", "finally",
  "ironically", "evenly", "boldly", "silently"};
static const char *PREPS[] = {"about", "above", "according to", "across", "after", "against", "along",
  "alongside of", "among", "around", "at", "atop", "before", "behind", "beneath", "beside", "besides",
  "between", "beyond", "by", "despite", "during", "except", "for", "from", "in place of", "inside",
  "instead of", "into", "near", "of", "on", "outside", "over", "past", "since", "through", "throughout",
  "to", "toward", "under", "until", "up", "upon", "without", "with", "within"};
static const char *TERMS[] = {".", ";", ":", "?", "!", "--"};
#define NEL(a) (sizeof(a) / sizeof((a)[0]))

static void build_pool(gen_ctx *g) {
  g->pool = (char *)malloc(POOL_BYTES + 256);
  uint64_t pos = 0, k = 0;
  while (pos < POOL_BYTES) {
    char sent[512];
    int m = 0;
#define PICK(arr) arr[rnd(g, F_POOL, k++) % NEL(arr)]
    /* sentence: [adj] noun [adv] verb [prep the adj noun] terminator */
    uint64_t shape = rnd(g, F_POOL, k++) % 4;
    if (shape & 1) m += snprintf(sent + m, sizeof(sent) - m, "%s ", PICK(ADJS));
    m += snprintf(sent + m, sizeof(sent) - m, "%s ", PICK(NOUNS));
    if (shape & 2) m += snprintf(sent + m, sizeof(sent) - m, "%s ", PICK(ADVS));
    m += snprintf(sent + m, sizeof(sent) - m, "%s", PICK(VERBS));
    if (rnd(g, F_POOL, k++) % 2) m += snprintf(sent + m, sizeof(sent) - m, " %s the %s %s", PICK(PREPS),
                                                PICK(ADJS), PICK(NOUNS));
    m += snprintf(sent + m, sizeof(sent) - m, "%s ", PICK(TERMS));
#undef PICK
    for (int i = 0; i < m && pos < POOL_BYTES; i++) g->pool[pos++] = sent[i];
  }
  memset(g->pool + POOL_BYTES, ' ', 256);
}

EXPORT void *gen_create(double sf, uint64_t seed) {
  gen_ctx *g = (gen_ctx *)calloc(1, sizeof(gen_ctx));
  g->sf = sf;
  g->seed = seed;
  g->n_orders = (uint64_t)(1500000.0 * sf + 0.5);
  if (g->n_orders < 1) g->n_orders = 1;
  uint64_t tot = 0;
  uint64_t *tmp = (uint64_t *)malloc((g->n_orders + 1) * sizeof(uint64_t));
  for (uint64_t o = 0; o < g->n_orders; o++) {
    tmp[o] = tot;
    tot += (uint64_t)unif(g, F_LINES, o, 1, 7);
  }
  tmp[g->n_orders] = tot;
  g->n_lines = tot;
  if (tot < (1ull << 32)) {
    g->line_prefix = (uint32_t *)malloc((g->n_orders + 1) * sizeof(uint32_t));
    for (uint64_t o = 0; o <= g->n_orders; o++) g->line_prefix[o] = (uint32_t)tmp[o];
    free(tmp);
  } else {
    g->line_prefix64 = tmp;
  }
  build_pool(g);
  return g;
}

EXPORT void gen_destroy(void *p) {
  gen_ctx *g = (gen_ctx *)p;
  if (!g) return;
  free(g->line_prefix);
  free(g->line_prefix64);
  free(g->pool);
  free(g);
}

static inline uint64_t n_parts(const gen_ctx *g) {
  int64_t n = (int64_t)(200000.0 * g->sf);
  return n < 1 ? 1 : (uint64_t)n;
}

EXPORT uint64_t gen_rows(void *p, int table) {
  gen_ctx *g = (gen_ctx *)p;
  if (table == T_PARTSUPP) return 4 * n_parts(g);
  return table == T_LINEITEM ? g->n_lines : g->n_orders;
}

/* Element byte width of each column (0 = VARBYTES). */
EXPORT int gen_col_width(int table, int col) {
  static const int LW[L_NCOLS] = {8, 4, 4, 4, 8, 8, 8, 8, 1, 1, 4, 4, 4, 25, 10, 0};
  static const int OW[O_NCOLS] = {8, 4, 1, 8, 4, 15, 15, 4, 0};
  static const int PW[PS_NCOLS] = {4, 4, 4, 8, 0};
  if (table == T_LINEITEM) return (col >= 0 && col < L_NCOLS) ? LW[col] : -1;
  if (table == T_PARTSUPP) return (col >= 0 && col < PS_NCOLS) ? PW[col] : -1;
  return (col >= 0 && col < O_NCOLS) ? OW[col] : -1;
}

static uint64_t find_order(const gen_ctx *g, uint64_t row) {
  uint64_t lo = 0, hi = g->n_orders; /* largest o with lp(o) <= row */
  while (hi - lo > 1) {
    uint64_t mid = (lo + hi) / 2;
    if (lp(g, mid) <= row) lo = mid; else hi = mid;
  }
  return lo;
}

static inline int64_t orderkey_of(uint64_t o) { return (int64_t)((o >> 3) * 32 + (o & 7) + 1); }
static inline int64_t retail_cents(int64_t pk) { return 90000 + ((pk / 10) % 20001) + 100 * (pk % 1000); }

typedef struct { int64_t part, supp, qty, ext_c, disc_c, tax_c; int32_t sd, cd, rd; char rflag, lstatus; } line_t;

/* Which line fields a column needs (each field is a pure function of (seed, field, order, line), so
 * computing only the needed ones gives the same values as computing all of them). */
enum { N_PART = 1, N_SUPP = 2, N_QTY = 4, N_EXT = 8, N_DISC = 16, N_TAX = 32, N_SD = 64, N_CD = 128, N_RD = 256,
       N_RFLAG = 512, N_LSTATUS = 1024, N_ALL = 2047 };

static void make_line_fields(const gen_ctx *g, uint64_t o, uint32_t l, unsigned need, line_t *L) {
  uint64_t id = o * 8 + l;
  if (need & (N_RFLAG | N_LSTATUS)) need |= N_SD | N_RD;
  if (need & N_RD) need |= N_SD;
  if (need & N_EXT) need |= N_QTY | N_PART;
  if (need & N_SUPP) need |= N_PART;
  int32_t od = 0;
  if (need & (N_SD | N_CD)) od = (int32_t)unif(g, F_ODATE, o, STARTDATE, ENDDATE - 151);
  if (need & N_PART) {
    int64_t nparts = (int64_t)(200000.0 * g->sf); if (nparts < 1) nparts = 1;
    L->part = unif(g, F_PART, id, 1, nparts);
  }
  if (need & N_SUPP) {
    int64_t nsupp = (int64_t)(10000.0 * g->sf); if (nsupp < 1) nsupp = 1;
    int64_t i = unif(g, F_SUPPI, id, 0, 3);
    L->supp = (L->part + (i * (nsupp / 4 + (L->part - 1) / nsupp))) % nsupp + 1;
  }
  if (need & N_QTY) L->qty = unif(g, F_QTY, id, 1, 50);
  if (need & N_EXT) L->ext_c = L->qty * retail_cents(L->part);
  if (need & N_DISC) L->disc_c = unif(g, F_DISC, id, 0, 10);
  if (need & N_TAX) L->tax_c = unif(g, F_TAX, id, 0, 8);
  if (need & N_SD) L->sd = od + (int32_t)unif(g, F_SHIPD, id, 1, 121);
  if (need & N_CD) L->cd = od + (int32_t)unif(g, F_COMMITD, id, 30, 90);
  if (need & N_RD) L->rd = L->sd + (int32_t)unif(g, F_RECEIPTD, id, 1, 30);
  if (need & N_RFLAG) L->rflag = (L->rd <= CURRENTDATE) ? ((rnd(g, F_RFLAG, id) >> 20) & 1 ? 'R' : 'A') : 'N';
  if (need & N_LSTATUS) L->lstatus = (L->sd > CURRENTDATE) ? 'O' : 'F';
}


static void put_padded(uint8_t *dst, const char *s, int w) {
  int n = (int)strlen(s);
  for (int i = 0; i < w; i++) dst[i] = (uint8_t)(i < n ? s[i] : ' ');
}

static const char *INSTR[] = {"DELIVER IN PERSON", "COLLECT COD", "NONE", "TAKE BACK RETURN"};
static const char *MODES[] = {"REG AIR", "AIR", "RAIL", "SHIP", "TRUCK", "MAIL", "FOB"};
static const char *PRIOS[] = {"1-URGENT", "2-HIGH", "3-MEDIUM", "4-NOT SPECIFIED", "5-LOW"};

/*
 * Fixed-width column rows [row0, row0+nrows) into out (nrows * width bytes, little-endian).
 * Returns 0, or -1 on a bad table/column/range.
 */
EXPORT int gen_fixed(void *p, int table, int col, uint64_t row0, uint64_t nrows, void *out) {
  gen_ctx *g = (gen_ctx *)p;
  int w = gen_col_width(table, col);
  if (w <= 0) return -1;
  uint8_t *dst = (uint8_t *)out;
  if (table == T_LINEITEM) {
    if (row0 + nrows > g->n_lines) return -1;
    if (nrows == 0) return 0;
    static const unsigned NEED[L_NCOLS] = {0, N_PART, N_SUPP, 0, N_QTY, N_EXT, N_DISC, N_TAX, N_RFLAG, N_LSTATUS,
                                           N_SD, N_CD, N_RD, 0, 0, 0};
    const unsigned need = NEED[col];
    uint64_t o = find_order(g, row0);
    uint32_t l = (uint32_t)(row0 - lp(g, o));
    for (uint64_t r = 0; r < nrows; r++) {
      while (lp(g, o) + l >= lp(g, o + 1)) { o++; l = 0; }
      line_t L;
      if (need) make_line_fields(g, o, l, need, &L);
      uint8_t *d = dst + r * (uint64_t)w;
      int64_t i64; int32_t i32; double f;
      switch (col) {
        case L_ORDERKEY: i64 = orderkey_of(o); memcpy(d, &i64, 8); break;
        case L_PARTKEY: i32 = (int32_t)L.part; memcpy(d, &i32, 4); break;
        case L_SUPPKEY: i32 = (int32_t)L.supp; memcpy(d, &i32, 4); break;
        case L_LINENUMBER: i32 = (int32_t)l + 1; memcpy(d, &i32, 4); break;
        case L_QUANTITY: f = (double)L.qty; memcpy(d, &f, 8); break;
        case L_EXTENDEDPRICE: f = (double)L.ext_c / 100.0; memcpy(d, &f, 8); break;
        case L_DISCOUNT: f = (double)L.disc_c / 100.0; memcpy(d, &f, 8); break;
        case L_TAX: f = (double)L.tax_c / 100.0; memcpy(d, &f, 8); break;
        case L_RETURNFLAG: d[0] = (uint8_t)L.rflag; break;
        case L_LINESTATUS: d[0] = (uint8_t)L.lstatus; break;
        case L_SHIPDATE: memcpy(d, &L.sd, 4); break;
        case L_COMMITDATE: memcpy(d, &L.cd, 4); break;
        case L_RECEIPTDATE: memcpy(d, &L.rd, 4); break;
        case L_SHIPINSTRUCT: put_padded(d, INSTR[unif(g, F_INSTR, o * 8 + l, 0, 3)], 25); break;
        case L_SHIPMODE: put_padded(d, MODES[unif(g, F_MODE, o * 8 + l, 0, 6)], 10); break;
        default: return -1;
      }
      l++;
    }
    return 0;
  }
  if (table == T_PARTSUPP) {
    /* row r = part (r / 4) + 1, supplier slot i = r % 4; the supplier formula is dbgen's (4.2.3) */
    if (row0 + nrows > 4 * n_parts(g)) return -1;
    int64_t nsupp = (int64_t)(10000.0 * g->sf); if (nsupp < 4) nsupp = 4;
    for (uint64_t r = row0; r < row0 + nrows; r++) {
      uint8_t *d = dst + (r - row0) * (uint64_t)w;
      const int64_t part = (int64_t)(r / 4) + 1, i = (int64_t)(r % 4);
      int32_t i32; double f;
      switch (col) {
        case PS_PARTKEY: i32 = (int32_t)part; memcpy(d, &i32, 4); break;
        case PS_SUPPKEY: i32 = (int32_t)((part + i * (nsupp / 4 + (part - 1) / nsupp)) % nsupp + 1); memcpy(d, &i32, 4); break;
        case PS_AVAILQTY: i32 = (int32_t)unif(g, F_AVAILQTY, r, 1, 9999); memcpy(d, &i32, 4); break;
        case PS_SUPPLYCOST: f = (double)unif(g, F_SUPPLYCOST, r, 100, 100000) / 100.0; memcpy(d, &f, 8); break;
        default: return -1;
      }
    }
    return 0;
  }
  if (row0 + nrows > g->n_orders) return -1;
  int64_t ncust = (int64_t)(150000.0 * g->sf); if (ncust < 2) ncust = 2;
  int64_t nclerk = (int64_t)(1000.0 * g->sf); if (nclerk < 1) nclerk = 1;
  for (uint64_t r = 0; r < nrows; r++) {
    uint64_t o = row0 + r;
    uint8_t *d = dst + r * (uint64_t)w;
    int64_t i64; int32_t i32; double f;
    switch (col) {
      case O_ORDERKEY: i64 = orderkey_of(o); memcpy(d, &i64, 8); break;
      case O_CUSTKEY: {
        int64_t c = unif(g, F_CUST, o, 1, ncust);
        if (c % 3 == 0) c = (c == ncust) ? c - 1 : c + 1; /* dbgen: every third customer has no orders */
        i32 = (int32_t)c; memcpy(d, &i32, 4); break;
      }
      case O_ORDERDATE: i32 = (int32_t)unif(g, F_ODATE, o, STARTDATE, ENDDATE - 151); memcpy(d, &i32, 4); break;
      case O_ORDERPRIORITY: put_padded(d, PRIOS[unif(g, F_OPRIO, o, 0, 4)], 15); break;
      case O_CLERK: {
        char s[32];
        snprintf(s, sizeof s, "Clerk#%09lld", (long long)unif(g, F_CLERK, o, 1, nclerk));
        put_padded(d, s, 15); break;
      }
      case O_SHIPPRIORITY: i32 = 0; memcpy(d, &i32, 4); break;
      case O_ORDERSTATUS:
      case O_TOTALPRICE: {
        uint32_t nl = (uint32_t)(lp(g, o + 1) - lp(g, o));
        int nf = 0; int64_t tot = 0;
        for (uint32_t l = 0; l < nl; l++) {
          line_t L; make_line_fields(g, o, l, col == O_ORDERSTATUS ? N_LSTATUS : (N_EXT | N_TAX | N_DISC), &L);
          nf += (L.lstatus == 'F');
          /* cents * (100+tax) * (100-disc) / 10^4, rounded half up (integer, exact) */
          tot += (L.ext_c * (100 + L.tax_c) * (100 - L.disc_c) + 5000) / 10000;
        }
        if (col == O_ORDERSTATUS) d[0] = (uint8_t)(nf == (int)nl ? 'F' : (nf == 0 ? 'O' : 'P'));
        else { f = (double)tot / 100.0; memcpy(d, &f, 8); }
        break;
      }
      default: return -1;
    }
  }
  return 0;
}

/*
 * VARBYTES comment column, rows [row0, row0+nrows): offsets (nrows+1 int64, chunk-relative, exclusive
 * end) always written; bytes written to out when out != NULL.  *payload = total bytes.
 */
EXPORT int gen_varbytes(void *p, int table, int col, uint64_t row0, uint64_t nrows, int64_t *offsets,
                        void *out, uint64_t *payload) {
  gen_ctx *g = (gen_ctx *)p;
  if (!((table == T_LINEITEM && col == L_COMMENT) || (table == T_ORDERS && col == O_COMMENT) ||
        (table == T_PARTSUPP && col == PS_COMMENT))) return -1;
  uint64_t nrow_tab = gen_rows(p, table);
  if (row0 + nrows > nrow_tab) return -1;
  uint64_t o = 0; uint32_t l = 0;
  if (table == T_LINEITEM && nrows) { o = find_order(g, row0); l = (uint32_t)(row0 - lp(g, o)); }
  uint64_t pos = 0;
  uint8_t *dst = (uint8_t *)out;
  for (uint64_t r = 0; r < nrows; r++) {
    uint64_t id; int64_t len, off;
    if (table == T_LINEITEM) {
      while (lp(g, o) + l >= lp(g, o + 1)) { o++; l = 0; }
      id = o * 8 + l; l++;
      len = unif(g, F_LCOMLEN, id, 10, 43);
      off = unif(g, F_LCOMOFF, id, 0, POOL_BYTES - 1 - 43);
    } else if (table == T_PARTSUPP) {
      id = row0 + r;
      len = unif(g, F_PSCOMLEN, id, 49, 198);
      off = unif(g, F_PSCOMOFF, id, 0, POOL_BYTES - 1 - 198);
    } else {
      id = row0 + r;
      len = unif(g, F_OCOMLEN, id, 19, 78);
      off = unif(g, F_OCOMOFF, id, 0, POOL_BYTES - 1 - 78);
    }
    offsets[r] = (int64_t)pos;
    if (dst) memcpy(dst + pos, g->pool + off, (size_t)len);
    pos += (uint64_t)len;
  }
  offsets[nrows] = (int64_t)pos;
  if (payload) *payload = pos;
  return 0;
}
