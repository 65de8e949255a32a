/*
 * oracle.h — CPU ORACLE for the sx relational hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load, call or execute anything under oracle/.
 * The product (paper_2508_04701_b200/, include/sx.h, libsx.so) never links
 * or imports it, and shares no code with it (task rule ③); the one shared
 * module is the seeded generator gen/sxgen.h, which holds no operator
 * arithmetic.
 *
 * What it computes: the plain SQL definitions of TPC-H Q1/Q3/Q6/Q9/Q18
 * and of the operators the paper hands to
 * libcudf — "filters, joins, aggregations, sorting" (PAPER.md P:96, P:191,
 * P:254) — row at a time, single threaded, with std::unordered_map /
 * std::map / std::stable_sort as library steps and __int128 for every sum.
 * Readings of the paper where it is silent are listed in DESIGN.md
 * §"Readings" (R1..R21 = SURVEY §8(c) table rows 1..21).
 *
 * Integer layout: int128 values cross the ABI as {lo, hi} two's complement
 * (value = hi * 2^64 + (uint64)lo).
 */
#ifndef SX_ORACLE_H
#define SX_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { uint64_t lo; int64_t hi; } or_i128;

/* Host columns of the TPC-H-shaped tables (orderkeys widened to int64 by the caller). */
typedef struct {
  int64_t n_lineitem;
  const int64_t* l_orderkey; const int32_t* l_partkey; const int32_t* l_suppkey;
  const int64_t* l_quantity; const int64_t* l_extendedprice; const int64_t* l_discount; const int64_t* l_tax;
  const uint8_t* l_returnflag; const uint8_t* l_linestatus; const int32_t* l_shipdate;
  int64_t n_orders;
  const int64_t* o_orderkey; const int32_t* o_custkey; const int32_t* o_orderdate; const int32_t* o_shippriority;
  const int64_t* o_totalprice;
  int64_t n_customer; const int32_t* c_custkey; const uint8_t* c_mktsegment;
  int64_t n_part; const int32_t* p_partkey; const int64_t* p_name_offsets; const uint8_t* p_name_chars;
  int64_t n_partsupp; const int32_t* ps_partkey; const int32_t* ps_suppkey; const int64_t* ps_supplycost;
  int64_t n_supplier; const int32_t* s_suppkey; const int32_t* s_nationkey;
} or_tables;

/* Query substitution parameters (TPC-H validation values are the defaults, see or_default_params). */
typedef struct {
  int32_t q1_shipdate_max;  /* 1998-12-01 - 90 days = 10471 */
  int32_t q3_segment;       /* dictionary code of 'BUILDING' = 1 */
  int32_t q3_date;          /* 1995-03-15 = 9204 */
  int32_t q6_date_lo;       /* 1994-01-01 = 8766 (inclusive) */
  int32_t q6_date_hi;       /* 1995-01-01 = 9131 (exclusive) */
  int64_t q6_disc_lo;       /* 0.05 -> 5 (inclusive) */
  int64_t q6_disc_hi;       /* 0.07 -> 7 (inclusive) */
  int64_t q6_qty_lt;        /* 24 -> 2400 (exclusive) */
  char q9_color[16];        /* "green" */
  int64_t q18_qty_gt;       /* 300 -> 30000 (exclusive) */
} or_params;

void or_default_params(or_params* p);

typedef struct {
  uint8_t returnflag, linestatus;
  or_i128 sum_qty, sum_base_price, sum_disc_price, sum_charge, sum_disc;
  int64_t count_order;
  double avg_qty, avg_price, avg_disc;
} or_q1_row;
typedef struct { or_i128 revenue; int32_t is_null; } or_q6_row;
typedef struct { int64_t l_orderkey; or_i128 revenue; int32_t o_orderdate, o_shippriority; } or_q3_row;
typedef struct { int32_t nationkey, o_year; or_i128 sum_profit; } or_q9_row;
typedef struct { int32_t c_custkey; int32_t o_orderdate; int64_t o_orderkey; int64_t o_totalprice; or_i128 sum_qty; } or_q18_row;

/* Each returns the number of result rows written (<= cap), or -1 on error. */
int64_t or_q1(const or_tables* t, const or_params* p, or_q1_row* out, int64_t cap);
int64_t or_q6(const or_tables* t, const or_params* p, or_q6_row* out);
int64_t or_q3(const or_tables* t, const or_params* p, int64_t limit, or_q3_row* out, int64_t cap);
int64_t or_q9(const or_tables* t, const or_params* p, or_q9_row* out, int64_t cap);
int64_t or_q18(const or_tables* t, const or_params* p, int64_t limit, or_q18_row* out, int64_t cap);

/* ---- operator-level oracles (parity targets for the sx_* calls) ---- */
enum { OR_LT = 0, OR_LE, OR_GT, OR_GE, OR_EQ, OR_NE, OR_BETWEEN };
typedef struct { int32_t col; int32_t op; int64_t lo, hi; } or_pred;

/* filter: rows r (ascending) where every pred holds on cols[pred.col][r]; returns count. */
int64_t or_filter(int64_t n, const int64_t* const* cols, const or_pred* preds, int32_t npreds, int32_t* out_sel);
/* contains: rows r (ascending) whose string contains pattern as a byte substring; returns count. */
int64_t or_contains(int64_t n, const int64_t* offsets, const uint8_t* chars, const char* pattern, int32_t plen,
                    int32_t* out_sel);

/* value expression: sum over terms of coef * prod over factors of (mul * col[r] + add), exact in int128. */
typedef struct { int32_t col; int64_t mul, add; } or_factor;
typedef struct { int64_t coef; int32_t nf; or_factor f[3]; } or_term;
typedef struct { int32_t nterms; or_term t[2]; } or_expr;
void or_eval_expr(int64_t n, const int64_t* const* cols, const or_expr* e, or_i128* out);

/* join: 0 inner (pairs, probe-major, build index ascending within a probe row), 1 semi, 2 anti. */
int64_t or_join(int64_t nb, const int64_t* bkeys, int64_t np, const int64_t* pkeys, int32_t type,
                int32_t* out_probe, int32_t* out_build, int64_t cap);

/* group-by over nkeys (0..2) int64 key columns; aggs: 0 sum, 1 count, 2 min, 3 max, 4 avg (of expr values).
 * Output groups ascending by key tuple.  out_aggs[a][g] as int128; avg written to out_avg[a][g]
 * (double = (double)sum / (double)count / 10^avg_scale[a]).  Returns #groups. */
int64_t or_groupby(int64_t n, const int64_t* const* cols, int32_t nkeys, const int32_t* key_cols, int32_t naggs,
                   const int32_t* agg_ops, const or_expr* agg_exprs, const int32_t* avg_scale,
                   int64_t* const* out_keys, or_i128* const* out_aggs, double* const* out_avg, int64_t cap);

/* stable sort permutation over nkeys int128 key columns (desc[k] != 0 => descending); first k rows. */
int64_t or_sort(int64_t n, const or_i128* const* keys, int32_t nkeys, const int32_t* desc, int64_t k, int32_t* out_perm);


/* ---- operator µbenchmarks (SURVEY.md §8(c) "µbench join" / "µbench group-by", §8(d) C5a/C5b) ----
 * The generator's build keys are mix64(i) (splitmix64 finalizer, a bijection on u64), so a key's
 * build row is mix64^-1(key): the join's and the group-by's exact results reduce to plain loops
 * with no hash table ("a special case reducing to a plain loop"). */
typedef struct { int64_t count; or_i128 sum_build; or_i128 sum_probe; uint64_t pair_hash; } or_join_summary;
uint64_t or_unmix64(uint64_t z);                 /* inverse of the splitmix64 finalizer */
uint64_t or_pair_mix(int64_t b, int64_t p);      /* order-independent pair hash term (summed mod 2^64) */
/* closed form: the build side is rows (mix64(i), i), i < nb; probe row j (key, payload) matches row
 * mix64^-1(key) iff that is < nb.  Summary over all matching pairs. */
void or_mb_join_closed(int64_t nb, int64_t np, const int64_t* pkeys, const int64_t* ppay, or_join_summary* out);
/* brute force over arbitrary build rows: std::unordered_multimap (pins the closed form). */
void or_mb_join_hash(int64_t nb, const int64_t* bkeys, const int64_t* bpay, int64_t np, const int64_t* pkeys,
                     const int64_t* ppay, or_join_summary* out);
/* group-by sweep, direct array indexed by g = mix64^-1(key) (must be < G, else returns -1):
 * per g: sum (int128), count, min, max (count 0 = group absent).  Returns #groups present. */
int64_t or_mb_groupby_direct(int64_t n, const int64_t* keys, const int64_t* vals, int64_t G, or_i128* sum,
                             int64_t* cnt, int64_t* mn, int64_t* mx);

/* proleptic Gregorian year of a day number (days since 1970-01-01). */
int32_t or_civil_year(int32_t days);

#ifdef __cplusplus
}
#endif
#endif
