/*
 * sxgen.h — counter-based, TPC-H-shaped data generator (value functions only).
 *
 * This is the ONE module shared by the CUDA product path and the CPU oracle
 * (task rule ③: "only the seeded input generators serve both, from a module
 * of their own that holds none of the method's arithmetic").  It defines what
 * the synthetic tables CONTAIN; it computes nothing the relational operators
 * compute (no predicates, joins, group-bys, sums over rows, sorts).
 *
 * Recipe: SURVEY.md Appendix A (TPC-H shapes [EXT-TPCH], exact values ours);
 * DESIGN.md §"Input recipe".  Every value is a pure function of
 * (seed, table, column, row counter), so CPU and GPU fills, and every shard
 * of a multi-GPU fill, produce identical bytes.
 *
 * Compiles as C99 (gcc, for gen_cpu.c and the oracle build) and as CUDA C++
 * (nvcc, for gen_gpu.cu) — functions are __host__ __device__ under nvcc.
 */
#ifndef SXGEN_H
#define SXGEN_H

#include <stdint.h>

#ifdef __CUDACC__
#define SXG_HD __host__ __device__ __forceinline__
#else
#define SXG_HD static inline
#endif

/* ---- table / column ids for the RNG counter (stable; part of the data definition) ---- */
enum {
  SXG_T_NATION = 0, SXG_T_REGION = 1, SXG_T_SUPPLIER = 2, SXG_T_CUSTOMER = 3,
  SXG_T_PART = 4, SXG_T_PARTSUPP = 5, SXG_T_ORDERS = 6, SXG_T_LINEITEM = 7
};
enum {
  /* supplier */ SXG_C_S_NATION = 1,
  /* customer */ SXG_C_C_SEGMENT = 1, SXG_C_C_NATION = 2,
  /* part     */ SXG_C_P_NAME0 = 1, /* ..5 */
  /* partsupp */ SXG_C_PS_COST = 1,
  /* orders   */ SXG_C_O_NLINES = 1, SXG_C_O_CUST = 2, SXG_C_O_DATE = 3,
  /* lineitem */ SXG_C_L_PART = 1, SXG_C_L_SUPPIDX = 2, SXG_C_L_QTY = 3, SXG_C_L_DISC = 4,
                 SXG_C_L_TAX = 5, SXG_C_L_SHIP = 6, SXG_C_L_RECEIPT = 7, SXG_C_L_RFLAG = 8,
                 SXG_C_L_COMMIT = 9
};

/* Dates are int32 days since 1970-01-01. */
#define SXG_DATE_1992_01_01 8035
#define SXG_DATE_1995_06_17 9298 /* TPC-H "current date" for returnflag/linestatus */
#define SXG_DATE_1998_08_02 10440

/* c_mktsegment dictionary (Arrow dictionary array, u8 codes) */
#define SXG_NSEGMENTS 5
#define SXG_SEGMENTS_INIT {"AUTOMOBILE", "BUILDING", "FURNITURE", "MACHINERY", "HOUSEHOLD"}

/* nation (25 rows, fixed; TPC-H [EXT-TPCH]) */
#define SXG_NNATIONS 25
#define SXG_NATIONS_INIT {                                                              \
  "ALGERIA", "ARGENTINA", "BRAZIL", "CANADA", "EGYPT", "ETHIOPIA", "FRANCE", "GERMANY", \
  "INDIA", "INDONESIA", "IRAN", "IRAQ", "JAPAN", "JORDAN", "KENYA", "MOROCCO",          \
  "MOZAMBIQUE", "PERU", "CHINA", "ROMANIA", "SAUDI ARABIA", "VIETNAM", "RUSSIA",        \
  "UNITED KINGDOM", "UNITED STATES"}

/* p_name colour words (92; TPC-H [EXT-TPCH]) */
#define SXG_NWORDS 92
#define SXG_WORD_MAXLEN 12
#define SXG_WORDS_INIT {                                                                  \
  "almond", "antique", "aquamarine", "azure", "beige", "bisque", "black", "blanched",    \
  "blue", "blush", "brown", "burlywood", "burnished", "chartreuse", "chiffon",           \
  "chocolate", "coral", "cornflower", "cornsilk", "cream", "cyan", "dark", "deep", "dim",\
  "dodger", "drab", "firebrick", "floral", "forest", "frosted", "gainsboro", "ghost",    \
  "goldenrod", "green", "grey", "honeydew", "hot", "indian", "ivory", "khaki", "lace",   \
  "lavender", "lawn", "lemon", "light", "lime", "linen", "magenta", "maroon", "medium",  \
  "metallic", "midnight", "mint", "misty", "moccasin", "navajo", "navy", "olive",        \
  "orange", "orchid", "pale", "papaya", "peach", "peru", "pink", "plum", "powder",       \
  "puff", "purple", "red", "rose", "rosy", "royal", "saddle", "salmon", "sandy",         \
  "seashell", "sienna", "sky", "slate", "smoke", "snow", "spring", "steel", "tan",       \
  "thistle", "tomato", "turquoise", "violet", "wheat", "white", "yellow"}
#define SXG_PNAME_MAXLEN 64

static const char sxg_words_host[SXG_NWORDS][SXG_WORD_MAXLEN] = SXG_WORDS_INIT;
#ifdef __CUDACC__
static __constant__ char sxg_words_dev[SXG_NWORDS][SXG_WORD_MAXLEN] = SXG_WORDS_INIT;
#endif

SXG_HD const char* sxg_word(int w) {
#ifdef __CUDA_ARCH__
  return sxg_words_dev[w];
#else
  return sxg_words_host[w];
#endif
}

/* ---- counter-based RNG ---- */

/* splitmix64 finalizer: a bijection on u64. */
SXG_HD uint64_t sxg_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

SXG_HD uint64_t sxg_rand(uint64_t seed, uint32_t table, uint32_t col, uint64_t row) {
  return sxg_mix64(seed ^ sxg_mix64(((uint64_t)table << 56) ^ ((uint64_t)col << 48) ^ row));
}

/* uniform integer in [a, b], b - a + 1 <= 2^32 (multiply-shift range reduction) */
SXG_HD int64_t sxg_uniform(uint64_t r, int64_t a, int64_t b) {
  return a + (int64_t)(((r >> 32) * (uint64_t)(b - a + 1)) >> 32);
}

/* ---- table sizes; sf_milli = scale factor x 1000 (SF 0.01 -> 10, SF 100 -> 100000) ---- */
SXG_HD int64_t sxg_n_supplier(int64_t sf_milli) { return 10 * sf_milli; }
SXG_HD int64_t sxg_n_customer(int64_t sf_milli) { return 150 * sf_milli; }
SXG_HD int64_t sxg_n_part(int64_t sf_milli) { return 200 * sf_milli; }
SXG_HD int64_t sxg_n_partsupp(int64_t sf_milli) { return 800 * sf_milli; }
SXG_HD int64_t sxg_n_orders(int64_t sf_milli) { return 1500 * sf_milli; }

/* ---- supplier (keys 1..S) ---- */
SXG_HD int32_t sxg_s_nationkey(uint64_t seed, int64_t suppkey) {
  return (int32_t)sxg_uniform(sxg_rand(seed, SXG_T_SUPPLIER, SXG_C_S_NATION, (uint64_t)suppkey), 0, 24);
}

/* ---- customer (keys 1..C) ---- */
SXG_HD uint8_t sxg_c_mktsegment(uint64_t seed, int64_t custkey) {
  return (uint8_t)sxg_uniform(sxg_rand(seed, SXG_T_CUSTOMER, SXG_C_C_SEGMENT, (uint64_t)custkey), 0, 4);
}
SXG_HD int32_t sxg_c_nationkey(uint64_t seed, int64_t custkey) {
  return (int32_t)sxg_uniform(sxg_rand(seed, SXG_T_CUSTOMER, SXG_C_C_NATION, (uint64_t)custkey), 0, 24);
}

/* ---- part (keys 1..P) ---- */
SXG_HD int64_t sxg_p_retailprice(int64_t partkey) { /* cents; TPC-H formula [EXT-TPCH] */
  return 90000 + ((partkey / 10) % 20001) + 100 * (partkey % 1000);
}

/* 5 distinct colour-word indices for part `partkey` (sequential draw without replacement). */
SXG_HD void sxg_p_name_words(uint64_t seed, int64_t partkey, int words[5]) {
  int used[5];
  for (int m = 0; m < 5; ++m) {
    int idx = (int)sxg_uniform(sxg_rand(seed, SXG_T_PART, SXG_C_P_NAME0 + m, (uint64_t)partkey), 0, SXG_NWORDS - 1 - m);
    /* idx-th word not yet used: walk the sorted used list */
    for (int u = 0; u < m; ++u)
      if (used[u] <= idx) ++idx;
    words[m] = idx;
    /* insert idx into sorted used[0..m] */
    int p = m;
    while (p > 0 && used[p - 1] > idx) { used[p] = used[p - 1]; --p; }
    used[p] = idx;
  }
}

/* Writes the space-joined name (no NUL) to out (>= SXG_PNAME_MAXLEN bytes), returns its length. */
SXG_HD int sxg_p_name(uint64_t seed, int64_t partkey, char* out) {
  int words[5];
  sxg_p_name_words(seed, partkey, words);
  int len = 0;
  for (int m = 0; m < 5; ++m) {
    if (m) out[len++] = ' ';
    const char* w = sxg_word(words[m]);
    for (int c = 0; c < SXG_WORD_MAXLEN && w[c]; ++c) out[len++] = w[c];
  }
  return len;
}

/* ---- partsupp (4 rows per part, i = 0..3) ---- */
SXG_HD int64_t sxg_ps_suppkey(int64_t partkey, int64_t i, int64_t n_supplier) { /* TPC-H formula */
  return ((partkey + i * (n_supplier / 4 + (partkey - 1) / n_supplier)) % n_supplier) + 1;
}
SXG_HD int64_t sxg_ps_supplycost(uint64_t seed, int64_t partkey, int64_t i) { /* cents */
  return sxg_uniform(sxg_rand(seed, SXG_T_PARTSUPP, SXG_C_PS_COST, (uint64_t)(partkey * 4 + i)), 100, 100000);
}

/* ---- orders (row index i = 1..O) ---- */
SXG_HD int64_t sxg_o_orderkey(int64_t i) { return ((i >> 3) << 5) | (i & 7); } /* sparse: 8 of 32 */
SXG_HD int32_t sxg_o_nlines(uint64_t seed, int64_t i) {
  return (int32_t)sxg_uniform(sxg_rand(seed, SXG_T_ORDERS, SXG_C_O_NLINES, (uint64_t)i), 1, 7);
}
SXG_HD int64_t sxg_o_custkey(uint64_t seed, int64_t i, int64_t n_customer) {
  int64_t u = sxg_uniform(sxg_rand(seed, SXG_T_ORDERS, SXG_C_O_CUST, (uint64_t)i), 0, (2 * n_customer) / 3 - 1);
  return u + u / 2 + 1; /* the u-th positive integer not divisible by 3 */
}
SXG_HD int32_t sxg_o_orderdate(uint64_t seed, int64_t i) {
  return (int32_t)sxg_uniform(sxg_rand(seed, SXG_T_ORDERS, SXG_C_O_DATE, (uint64_t)i), SXG_DATE_1992_01_01, SXG_DATE_1998_08_02);
}

/* ---- lineitem: line j (1..nlines) of order i; RNG row counter = i*8 + j ---- */
typedef struct {
  int32_t partkey, suppkey;
  int64_t quantity;      /* scale 2 (qty x 100) */
  int64_t extendedprice; /* cents */
  int64_t discount;      /* scale 2: 0..10 */
  int64_t tax;           /* scale 2: 0..8 */
  int32_t shipdate, commitdate, receiptdate;
  uint8_t returnflag, linestatus; /* ASCII */
} sxg_line;

SXG_HD void sxg_l_line(uint64_t seed, int64_t i, int32_t j, int32_t orderdate,
                       int64_t n_part, int64_t n_supplier, sxg_line* L) {
  uint64_t row = (uint64_t)i * 8 + (uint64_t)j;
  int64_t pk = sxg_uniform(sxg_rand(seed, SXG_T_LINEITEM, SXG_C_L_PART, row), 1, n_part);
  int64_t si = sxg_uniform(sxg_rand(seed, SXG_T_LINEITEM, SXG_C_L_SUPPIDX, row), 0, 3);
  int64_t q = sxg_uniform(sxg_rand(seed, SXG_T_LINEITEM, SXG_C_L_QTY, row), 1, 50);
  L->partkey = (int32_t)pk;
  L->suppkey = (int32_t)sxg_ps_suppkey(pk, si, n_supplier);
  L->quantity = q * 100;
  L->extendedprice = q * sxg_p_retailprice(pk);
  L->discount = sxg_uniform(sxg_rand(seed, SXG_T_LINEITEM, SXG_C_L_DISC, row), 0, 10);
  L->tax = sxg_uniform(sxg_rand(seed, SXG_T_LINEITEM, SXG_C_L_TAX, row), 0, 8);
  L->shipdate = orderdate + (int32_t)sxg_uniform(sxg_rand(seed, SXG_T_LINEITEM, SXG_C_L_SHIP, row), 1, 121);
  L->commitdate = orderdate + (int32_t)sxg_uniform(sxg_rand(seed, SXG_T_LINEITEM, SXG_C_L_COMMIT, row), 30, 90);
  L->receiptdate = L->shipdate + (int32_t)sxg_uniform(sxg_rand(seed, SXG_T_LINEITEM, SXG_C_L_RECEIPT, row), 1, 30);
  if (L->receiptdate <= SXG_DATE_1995_06_17)
    L->returnflag = sxg_uniform(sxg_rand(seed, SXG_T_LINEITEM, SXG_C_L_RFLAG, row), 0, 1) ? 'R' : 'A';
  else
    L->returnflag = 'N';
  L->linestatus = (L->shipdate > SXG_DATE_1995_06_17) ? 'O' : 'F';
}

/* o_totalprice term of one line (our definition):
 * floor(floor(ext*(100-disc)/100)*(100+tax)/100) — all operands non-negative. */
SXG_HD int64_t sxg_line_price_term(const sxg_line* L) {
  return ((L->extendedprice * (100 - L->discount)) / 100) * (100 + L->tax) / 100;
}

/* ---- operator micro-benchmarks (SURVEY.md §8(d) C5a/C5b and "(ours) sort µbench";
 *      readings R15-R17 in DESIGN.md).  Table ids 16.. are outside the TPC-H range. ---- */
enum { SXG_T_MB_PROBE = 16, SXG_T_MB_GB = 17, SXG_T_MB_SORT = 18, SXG_T_MB_PERM = 19 };

/* join build row i (0 <= i < nb): key mix64(i), payload i (R15: PK side, unique keys). */
SXG_HD uint64_t sxg_mb_build_key(int64_t i) { return sxg_mix64((uint64_t)i); }

/* affine permutation of [0, nb), nb a power of two: pi(r) = (a r + b) mod nb, a odd (R16: hot
 * ranks scatter over the table). */
SXG_HD int64_t sxg_mb_perm(uint64_t seed, int64_t r, int64_t nb) {
  uint64_t a = sxg_rand(seed, SXG_T_MB_PERM, 1, 0) | 1ull, b = sxg_rand(seed, SXG_T_MB_PERM, 2, 0);
  return (int64_t)((a * (uint64_t)r + b) & (uint64_t)(nb - 1));
}

/* 2^(m/16) in 16.16 fixed point, m = 0..16 (integer literals: identical on CPU and GPU). */
#define SXG_EXP2_16THS_INIT {65536, 68438, 71468, 74632, 77936, 81386, 84990, 88752, 92682, 96785, \
                             101070, 105545, 110218, 115098, 120194, 125515, 131072}

/* probe row j's rank in [0, nb): uniform, or Zipf(1.0) (R16) sampled as a log-uniform over
 * 16 x log2(nb) equal-probability cells (sub-octaves [2^(k+m/16), 2^(k+(m+1)/16)) of r+1), uniform
 * inside a cell: density of r+1 proportional to 1/(r+1) up to the cell discretisation.  Integer
 * arithmetic only, so CPU and GPU draw identical ranks.  nb a power of two, 2 <= nb <= 2^32. */
SXG_HD int64_t sxg_mb_probe_rank(uint64_t seed, int64_t j, int64_t nb, int zipf) {
  uint64_t r0 = sxg_rand(seed, SXG_T_MB_PROBE, 1, (uint64_t)j);
  if (!zipf) return sxg_uniform(r0, 0, nb - 1);
  const uint32_t B[17] = SXG_EXP2_16THS_INIT;
  int L = 0;
  while ((1ll << L) < nb) ++L;
  uint64_t c = ((r0 >> 32) * (uint64_t)(16 * L)) >> 32; /* cell in [0, 16L) */
  int k = (int)(c >> 4), m = (int)(c & 15);
  uint64_t lo = ((uint64_t)B[m] << k) >> 16, hi = ((uint64_t)B[m + 1] << k) >> 16;
  if (hi <= lo) hi = lo + 1;
  uint64_t r1 = sxg_rand(seed, SXG_T_MB_PROBE, 2, (uint64_t)j);
  int64_t v = (int64_t)lo + (int64_t)(((r1 >> 32) * (hi - lo)) >> 32); /* r + 1 in [lo, hi) */
  int64_t r = v - 1;
  return r < 0 ? 0 : (r >= nb ? nb - 1 : r);
}
/* probe row j: key = build key of pi(rank), payload j (every probe matches exactly one build row). */
SXG_HD uint64_t sxg_mb_probe_key(uint64_t seed, int64_t j, int64_t nb, int zipf) {
  return sxg_mb_build_key(sxg_mb_perm(seed, sxg_mb_probe_rank(seed, j, nb, zipf), nb));
}

/* group-by sweep row i (R17): group g ~ U[0, G), key mix64(g) (int64), value DEC64 scale 2
 * uniform in [1.00, 100000.00]. */
SXG_HD int64_t sxg_mb_gb_group(uint64_t seed, int64_t i, int64_t G) {
  return sxg_uniform(sxg_rand(seed, SXG_T_MB_GB, 1, (uint64_t)i), 0, G - 1);
}
SXG_HD int64_t sxg_mb_gb_value(uint64_t seed, int64_t i) {
  return sxg_uniform(sxg_rand(seed, SXG_T_MB_GB, 2, (uint64_t)i), 100, 10000000);
}

/* sort µbench row i: a uniform int64 key (all 64 bits), payload i. */
SXG_HD int64_t sxg_mb_sort_key(uint64_t seed, int64_t i) {
  return (int64_t)sxg_rand(seed, SXG_T_MB_SORT, 1, (uint64_t)i);
}

#endif /* SXGEN_H */
