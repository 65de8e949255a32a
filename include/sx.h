/*
 * sx.h — C ABI of libsx.so: the data-parallel relational hot path of Sirius
 * (arXiv 2508.04701) re-built B200-native (sm_100a).
 *
 * The paper hands "relational operators like joins, filters, aggregations"
 * and "sorting" to libcudf, with custom CUDA
 * kernels for "predicate pushdown, and materialization", over
 * Arrow-derived columns passed by pointer with int32 kernel row
 * indices.  This header is that boundary: four operator families
 * (sx_filter, sx_hash_build/sx_hash_probe, sx_groupby_agg, sx_sort_topk)
 * plus a fixed-plan executor for TPC-H Q1/Q3/Q6/Q9/Q18 standing in for the
 * Substrait consumer (BASELINE.json north_star).
 *
 * Conventions (all calls):
 *  - Data pointers in sx_col / sx_sel are DEVICE pointers (current ctx device)
 *    unless a comment says "host".  Layouts are Arrow little-endian; column
 *    buffers must be dense and 16-byte aligned (cudaMalloc / torch allocations
 *    are; string offsets 8-byte aligned, string bytes unconstrained): a
 *    misaligned buffer -> SX_EINVAL.
 *  - Inputs are borrowed for the duration of the call.  Outputs (selection
 *    vectors, output columns) are allocated by the library from its
 *    stream-ordered pool and released with sx_free(); hash tables with
 *    sx_ht_destroy().
 *  - Every call is stream-ordered on the ctx stream.  A call whose output
 *    size is data-dependent performs ONE device->host read of that size and
 *    synchronises the stream once (noted per call).
 *  - Row ids are int32: more than INT32_MAX rows per call -> SX_EINDEX.
 *  - v1 is null-free: a non-NULL `validity` -> SX_EUNSUPPORTED (TPC-H base
 *    data has no NULLs; SURVEY §8(c) reading R18).
 *  - Return codes only; no C++ exception crosses the ABI.  On error, out-params
 *    are zeroed, nothing is left allocated, and sx_last_error() explains.
 *  - No CPU fallback exists: every step runs in libsx's CUDA kernels.
 */
#ifndef SX_H
#define SX_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SX_OK = 0,
  SX_EINVAL = 1,        /* bad argument (shape, index, null pointer) */
  SX_ETYPE = 2,         /* column type not accepted by this call */
  SX_ENOMEM = 3,        /* device pool exhausted (SPEC "ProcessingExhausted") */
  SX_EINDEX = 4,        /* > INT32_MAX rows in one call (SPEC "IndexOverflow") */
  SX_EOVERFLOW = 5,     /* a per-row value expression left int64 */
  SX_EUNSUPPORTED = 6,  /* e.g. validity bitmaps (null-free v1) */
  SX_ECUDA = 7,         /* CUDA runtime error (sticky errors included) */
  SX_ENCCL = 8          /* NCCL error */
} sx_status;

typedef enum {
  SX_U8 = 0,      /* uint8 (flags, dictionary codes) */
  SX_I32 = 1,     /* int32 keys */
  SX_I64 = 2,     /* int64 keys */
  SX_DATE32 = 3,  /* int32 days since 1970-01-01 */
  SX_DEC64 = 4,   /* scaled int64 decimal; value = data / 10^scale */
  SX_I128 = 5,    /* {uint64 lo; int64 hi} two's complement (aggregate outputs) */
  SX_F64 = 6,     /* double (avg outputs) */
  SX_STR = 7      /* Arrow large string: int64 offsets[len+1] + bytes in `data` */
} sx_type;

typedef struct {
  int32_t type;              /* sx_type */
  int32_t scale;             /* SX_DEC64 only */
  int64_t len;               /* rows */
  const void* data;          /* values (or string bytes) */
  const int64_t* offsets;    /* SX_STR only */
  const uint8_t* validity;   /* must be NULL in v1 */
} sx_col;

typedef struct {
  int64_t len;
  int32_t* idx;              /* device; ascending unless produced by a join or a sort */
} sx_sel;

typedef struct sx_ctx sx_ctx;
typedef struct sx_ht sx_ht;

/* ---- context ---------------------------------------------------------------
 * One ctx per host thread.  `stream` is a cudaStream_t (NULL = legacy default).
 * Device memory comes from a stream-ordered pool (cudaMallocAsync on the
 * device's default pool with its release threshold raised, so steady-state
 * queries do not call into the driver): the "processing region" of the
 * paper's buffer manager. */
sx_status sx_ctx_create(int device, void* stream, sx_ctx** out);
void sx_ctx_destroy(sx_ctx* ctx);
const char* sx_last_error(const sx_ctx* ctx);  /* host string, valid until the next call on ctx */
sx_status sx_free(sx_ctx* ctx, void* p);       /* stream-ordered free of any library-allocated buffer */
sx_status sx_sync(sx_ctx* ctx);                /* wait for the ctx stream */
/* Stream-ordered copy between any two pointers (cudaMemcpyDefault); binding helper. */
sx_status sx_memcpy(sx_ctx* ctx, void* dst, const void* src, size_t bytes);
/* Number of CUDA kernels libsx launched on this ctx since the last reset (reset != 0 zeroes it). */
int64_t sx_launch_count(sx_ctx* ctx, int reset);
/* Per-operator device timing (CUDA events around each sx_* call; Fig. 5 analog). */
sx_status sx_profile_enable(sx_ctx* ctx, int on);
/* Fills up to cap entries of (name, milliseconds, algorithmic bytes) for calls since the last read
 * (bytes: SURVEY §8(d) definition 1 — referenced input columns once at stored width + mandatory
 * outputs once; 0 where a call does not define it; `bytes` may be NULL); returns count in *n. */
sx_status sx_profile_read(sx_ctx* ctx, char (*names)[32], float* ms, double* bytes, int cap, int* n);

/* ---- value expressions ------------------------------------------------------
 * value(r) = sum over t < nterms of coef_t * prod over f < nf_t of (mul_f * cols[col_f][r] + add_f).
 * Evaluated exactly in integer arithmetic; every factor, partial product and
 * the result must fit in int64, else SX_EOVERFLOW.  Decimal scales add under
 * multiplication (SURVEY reading R2), e.g. l_extendedprice*(1-l_discount) with
 * both at scale 2 is {coef 1, f = {ext,1,0},{disc,-1,100}} at scale 4.
 * Accepted column types: U8, I32, DATE32, I64, DEC64. */
typedef struct { int32_t col; int32_t pad; int64_t mul, add; } sx_factor;
typedef struct { int64_t coef; int32_t nf; int32_t pad; sx_factor f[3]; } sx_term;
typedef struct { int32_t nterms; int32_t pad; sx_term t[2]; } sx_expr;

/* ---- predicates ------------------------------------------------------------
 * A conjunction of `col op constant` terms (predicate pushdown).
 * Fixed-width columns compare as int64 (U8/I32/DATE32/I64/DEC64 in stored
 * units).  SX_CONTAINS: byte-substring test on an SX_STR column
 * (LIKE '%pattern%', SURVEY reading R9); `pattern` is a HOST pointer. */
typedef enum { SX_LT = 0, SX_LE, SX_GT, SX_GE, SX_EQ, SX_NE, SX_BETWEEN /* lo <= x <= hi */, SX_CONTAINS } sx_cmp;
typedef struct {
  int32_t col;
  int32_t op;                /* sx_cmp */
  int64_t lo, hi;
  const char* pattern;       /* host; SX_CONTAINS only */
  int32_t pattern_len;
  int32_t pad;
} sx_pred;

#define SX_MAX_COLS 16
#define SX_MAX_PREDS 8
#define SX_MAX_AGGS 8

/* ---- H1/H2: filter + compaction (+ materialization) ---------------------------
 * Rows r (of in_sel if given, else 0..n-1, n = cols[conj[0].col].len) where
 * every predicate holds -> out_sel (ascending int32 row ids of the input
 * columns).  If ngather > 0, out_cols[i] receives the dense gathered column
 * cols[gather_cols[i]][out_sel] ("materialization").  At most one
 * SX_CONTAINS predicate, and it cannot be mixed with other predicates.
 * Syncs once (output length).  npred == 0 selects every row. */
sx_status sx_filter(sx_ctx* ctx, const sx_col* cols, int ncols, const sx_pred* conj, int npred, const sx_sel* in_sel,
                    const int32_t* gather_cols, int ngather, sx_sel* out_sel, sx_col* out_cols);

/* ---- H3/H7/H8: hash group-by aggregation --------------------------------------
 * Groups the selected rows (in_sel and/or the `where` conjunction) by up to two
 * key columns; each aggregate is over a value expression (sx_expr):
 *   SX_SUM   -> SX_I128 sum (exact; int128 cannot overflow: <= 2^31 rows x |v| < 2^63)
 *   SX_COUNT -> SX_I64 count(*)   (value ignored)
 *   SX_MIN / SX_MAX -> SX_I64
 *   SX_AVG   -> SX_F64 = (double)sum / (double)count / 10^scale   (reading R3)
 * Keys: U8 / I32 / DATE32 / I64; `key_fn` SX_KEY_YEAR maps a DATE32 key to its
 * proleptic Gregorian year (extract(year from ...)).  Two keys must each be
 * <= 32 bits wide.  nkeys == 0 is a keyless reduce: exactly one output row,
 * with count 0 and SUM/MIN/MAX/AVG undefined (NULL) when no row qualifies
 * — check the COUNT.
 * `having` (optional): keep only groups whose aggregate `having->agg` satisfies
 * op against lo/hi (SX_SUM compares the int128 sum; only LT..BETWEEN).
 * groups_hint sizes the table (<= 0: unknown); a too-small hint costs a retry.
 * Output group order is unspecified.  Syncs once (group count). */
typedef enum { SX_SUM = 0, SX_COUNT, SX_MIN, SX_MAX, SX_AVG } sx_aggop;
typedef struct { int32_t op; int32_t scale; sx_expr value; } sx_agg;
typedef enum { SX_KEY_IDENTITY = 0, SX_KEY_YEAR = 1 } sx_keyfn;
typedef struct { int32_t col; int32_t fn; } sx_key;
typedef struct { int32_t agg; int32_t op; int64_t lo, hi; } sx_having;
sx_status sx_groupby_agg(sx_ctx* ctx, const sx_col* cols, int ncols, const sx_key* keys, int nkeys,
                         const sx_sel* in_sel, const sx_pred* where, int nwhere, const sx_agg* aggs, int naggs,
                         const sx_having* having, int64_t groups_hint, sx_col* out_keys, sx_col* out_aggs,
                         int64_t* out_ngroups /* host */);

/* ---- H4/H6: hash join build / probe --------------------------------------------
 * Build: open-addressing table (linear probing, load <= 0.5) over the key
 * column(s) of the selected build rows; stores (key, build row id).  Keys:
 * one I32/I64/DATE32 column, or two <= 32-bit columns packed into 64 bits
 * (reading R11).  Duplicate keys are kept.  unique_hint != 0 lets probes stop
 * at the first match (PK side).  The table copies keys and row ids, so build
 * columns may be freed after the call, except those later gathered as payload.
 * Probe: for each selected probe row (in_sel and/or `where`):
 *   SX_INNER: every matching (probe row, build row) pair -> out_probe, out_build
 *             (order unspecified; a multiset, SPEC S:229 / reading R12)
 *   SX_SEMI:  each probe row with >= 1 match, once, ascending -> out_probe
 *   SX_ANTI:  each probe row with no match, once, ascending -> out_probe
 * Payload gather (fused materialization): out_payload[0..nbp) = build_cols[bp[i]]
 * at the matched build rows (INNER only), then out_payload[nbp..nbp+npp) =
 * probe_cols[pp[j]] at the output probe rows.  Syncs once (output length). *
 * unique_hint flags: SX_BUILD_UNIQUE (1) as above; SX_BUILD_MEMBERSHIP (2): only SEMI/ANTI probes
 * will follow, so when the exact key-range bitmap exists (one key column, key range <= 2^30) the
 * table itself is not built (probes answer from the bitmap); INNER probes of such a table return
 * SX_EINVAL. */
typedef enum { SX_INNER = 0, SX_SEMI = 1, SX_ANTI = 2 } sx_join;
#define SX_BUILD_UNIQUE 1
#define SX_BUILD_MEMBERSHIP 2
sx_status sx_hash_build(sx_ctx* ctx, const sx_col* cols, int ncols, const int32_t* key_cols, int nkeys,
                        const sx_sel* in_sel, const sx_pred* where, int nwhere, int unique_hint, sx_ht** out);
sx_status sx_hash_probe(sx_ctx* ctx, const sx_ht* ht, const sx_col* probe_cols, int nprobe_cols,
                        const int32_t* key_cols, int nkeys, const sx_sel* in_sel, const sx_pred* where, int nwhere,
                        int join_type, const sx_col* build_cols, int nbuild_cols, const int32_t* bp, int nbp,
                        const int32_t* pp, int npp, sx_sel* out_probe, sx_sel* out_build, sx_col* out_payload);
int64_t sx_ht_rows(const sx_ht* ht);  /* build rows inserted */
void sx_ht_destroy(sx_ctx* ctx, sx_ht* ht);

/* ---- H5: radix partitioning and the partitioned join ---------------------------------
 * (north_star: "radix-partitioned joins when the build side exceeds L2"; SURVEY §8(a) H5;
 * PAPER.md P:351 names GPU join algorithms as techniques Sirius can adopt.)
 * Partition of a key = (hash64(key) >> 48) & (2^bits - 1): hash bits 48..57, disjoint from the
 * table-slot bits (low) and the shard-rank bits (top; reading R14).  Two 32-bit key columns are
 * packed (k0 << 32) | k1 first (reading R11).  sx_radix_of is the host mirror. */
uint32_t sx_radix_of(uint64_t key, int bits);
/* Regroup the selected rows (in_sel, else all) of every column by partition, 1 <= bits <= 10:
 * out_cols[c] = cols[c] with rows partition-contiguous (partition p at rows
 * offsets[p] .. offsets[p+1]); order inside a partition is unspecified.  offsets: HOST array of
 * 2^bits + 1 entries.  out_rows (optional): the original row id of every output row.  Keys: one
 * I32/DATE32/I64 column or two 32-bit columns; carried columns: fixed-width, at most 12.
 * Syncs once (offsets). */
sx_status sx_radix_partition(sx_ctx* ctx, const sx_col* cols, int ncols, const int32_t* key_cols, int nkeys,
                             const sx_sel* in_sel, int bits, sx_col* out_cols, sx_sel* out_rows,
                             int64_t* offsets /* host */);
/* Build + probe in one call.  strategy 1 = flat (sx_hash_build + sx_hash_probe, semantics and
 * output order as there); 2 = radix-partitioned; 0 = automatic: partitioned when the flat table
 * (2^ceil(log2(2 n_build)) slots of 8/16 B) would exceed half the L2 and the join is INNER on a
 * unique build (unique_hint, the PK side), else flat.  Partitioned: both sides are partitioned
 * carrying their key and payload columns (sx_radix_partition), then the partitions are joined in
 * waves whose tables together fit half the L2.  Outputs as sx_hash_probe: out_payload[0..nbp) =
 * build_cols[bp[i]] at the matches, then out_payload[nbp..nbp+npp) = probe_cols[pp[j]];
 * out_probe / out_build (row ids; each may be NULL = not produced).  Partitioned output order is
 * unspecified (a multiset, reading R12).  *used_strategy (optional) = 1 or 2.  Syncs (counts). */
sx_status sx_hash_join(sx_ctx* ctx, const sx_col* build_cols, int nbuild_cols, const int32_t* build_keys,
                       const sx_sel* build_sel, int unique_hint, const sx_col* probe_cols, int nprobe_cols,
                       const int32_t* probe_keys, const sx_sel* probe_sel, int nkeys, int join_type,
                       const int32_t* bp, int nbp, const int32_t* pp, int npp, int strategy, sx_sel* out_probe,
                       sx_sel* out_build, sx_col* out_payload, int* used_strategy);

/* ---- H9: sort / top-k ---------------------------------------------------------
 * Stable sort of the selected rows by the keys (each ascending, or descending if
 * desc); out_perm = the first min(k, n) row ids (k < 0: all).  Ties keep input
 * order.  Key types: U8, I32, DATE32, I64, DEC64, I128.  Syncs once. */
typedef struct { int32_t col; int32_t desc; } sx_sortkey;
sx_status sx_sort_topk(sx_ctx* ctx, const sx_col* cols, int ncols, const sx_sortkey* keys, int nkeys,
                       const sx_sel* in_sel, int64_t k, sx_sel* out_perm);

/* ---- materialization helper: out[i] = col[sel[i]] (any fixed-width type) ---- */
sx_status sx_gather(sx_ctx* ctx, const sx_col* col, const sx_sel* sel, sx_col* out);

/* ---- FINAL phase of a distributed aggregation (avg carried as sum+count) ----
 * Groups partial rows (e.g. the allgathered outputs of sx_groupby_agg on every rank) by 1-2 key
 * columns and combines each partial column exactly: ops[j] = SX_SUM (SX_I128 partial sums, int128
 * add), SX_COUNT (SX_I64, add), SX_MIN / SX_MAX (SX_I64).  AVG: merge its SUM and COUNT, then sx_avg.
 * Output types = input types; optional HAVING on a merged column; order unspecified.  Syncs once. */
sx_status sx_groupby_merge(sx_ctx* ctx, const sx_col* keys, int nkeys, const sx_col* parts, const int32_t* ops,
                           int nparts, const sx_having* having, int64_t groups_hint, sx_col* out_keys,
                           sx_col* out_parts, int64_t* out_ngroups);
/* avg = (double)sum / (double)count / 10^scale, element-wise (reading R3). */
sx_status sx_avg(sx_ctx* ctx, const sx_col* sum /* SX_I128 */, const sx_col* count /* SX_I64 */, int scale,
                 sx_col* out /* SX_F64 */);

/* ---- H5/H10: partitioning and exchange across GPUs (NCCL over NVLink) ----------
 * Destination rank of a key = ((hash64(key) >> 32) * nranks) >> 32 — the high hash bits, disjoint
 * from the low bits that pick hash-table slots (reading R14); two 32-bit key columns are packed
 * (k0 << 32) | k1 first.  sx_dest_rank is the host mirror of that function. */
int sx_dest_rank(uint64_t key, int nranks);
/* Regroup the selected rows by destination rank: out_cols[c] holds rank 0's rows, then rank 1's,
 * ... (input order kept within each destination); counts[d] (host) = rows for rank d. */
sx_status sx_partition_by_rank(sx_ctx* ctx, const sx_col* cols, int ncols, const int32_t* key_cols, int nkeys,
                               const sx_sel* in_sel, int nranks, sx_col* out_cols, int64_t* counts /* host */);
typedef struct sx_comm sx_comm;
/* 128-byte NCCL unique id (host); create on one rank, distribute, then sx_comm_init on every rank. */
sx_status sx_comm_unique_id(void* out);
sx_status sx_comm_init(sx_ctx* ctx, const void* unique_id, int rank, int nranks, sx_comm** out);
void sx_comm_destroy(sx_comm* comm);
int sx_comm_rank(const sx_comm* comm);
int sx_comm_size(const sx_comm* comm);
/* Hash shuffle: every rank sends each selected row to sx_dest_rank(key) (partition + counts
 * allgather + grouped ncclSend/ncclRecv).  out_cols: received rows, ordered by source rank.
 * Syncs once (counts).  Collective: all ranks must call it. */
sx_status sx_shuffle(sx_ctx* ctx, sx_comm* comm, const sx_col* cols, int ncols, const int32_t* key_cols, int nkeys,
                     const sx_sel* in_sel, sx_col* out_cols, int64_t* out_rows /* host */);
/* Broadcast/merge exchange: concatenation of every rank's columns in rank order (variable
 * lengths).  Syncs once (lengths).  Collective. */
sx_status sx_allgather(sx_ctx* ctx, sx_comm* comm, const sx_col* cols, int ncols, sx_col* out_cols,
                       int64_t* out_rows /* host */);

/* ---- fixed-plan executor: TPC-H Q1/Q3/Q6/Q9/Q18 ---------------------------------
 * Stands in for the Substrait consumer (north_star).  Columns are device
 * buffers as produced by gen/ (orderkey I32 or I64; decimals DEC64 scale 2;
 * dates DATE32; flags U8 ASCII; c_mktsegment U8 dictionary codes; p_name SX_STR).
 * Results are written to HOST row buffers in query order (the final D2H is
 * inside the call).  Semantics and readings: SURVEY §8(c), DESIGN.md. */
typedef struct {
  sx_col l_orderkey, l_partkey, l_suppkey, l_quantity, l_extendedprice, l_discount, l_tax, l_returnflag,
      l_linestatus, l_shipdate;
  sx_col o_orderkey, o_custkey, o_orderdate, o_shippriority, o_totalprice;
  sx_col c_custkey, c_mktsegment;
  sx_col p_partkey, p_name;
  sx_col ps_partkey, ps_suppkey, ps_supplycost;
  sx_col s_suppkey, s_nationkey;
} sx_tpch_tables;

typedef struct {
  int32_t q1_shipdate_max;  /* 10471 */
  int32_t q3_segment;       /* 1 (BUILDING) */
  int32_t q3_date;          /* 9204 */
  int32_t q6_date_lo, q6_date_hi;   /* 8766, 9131 */
  int64_t q6_disc_lo, q6_disc_hi;   /* 5, 7 */
  int64_t q6_qty_lt;        /* 2400 */
  char q9_color[16];        /* "green" */
  int64_t q18_qty_gt;       /* 30000 */
  int64_t q3_limit;         /* 10 */
  int64_t q18_limit;        /* 100 */
} sx_tpch_params;
void sx_tpch_default_params(sx_tpch_params* p);

/* End-to-end entry: `host` describes the same tables in HOST memory (pinned for full PCIe speed;
 * SX_STR offsets are host too).  Every non-empty column is copied into a library-allocated device
 * buffer (stream-ordered H2D copies, no sync) and `dev` receives the device description, to be
 * passed to sx_tpch_q* and released with sx_tpch_tables_free. */
sx_status sx_tpch_upload(sx_ctx* ctx, const sx_tpch_tables* host, sx_tpch_tables* dev);
void sx_tpch_tables_free(sx_ctx* ctx, sx_tpch_tables* dev);

typedef struct { uint64_t lo; int64_t hi; } sx_i128;
typedef struct {
  uint8_t returnflag, linestatus, pad[6];
  sx_i128 sum_qty, sum_base_price, sum_disc_price, sum_charge;
  double avg_qty, avg_price, avg_disc;
  int64_t count_order;
} sx_q1_row;
typedef struct { sx_i128 revenue; int32_t is_null; int32_t pad; } sx_q6_row;
typedef struct { int64_t l_orderkey; sx_i128 revenue; int32_t o_orderdate, o_shippriority; } sx_q3_row;
typedef struct { int32_t nationkey, o_year; sx_i128 sum_profit; } sx_q9_row;
typedef struct { int32_t c_custkey, o_orderdate; int64_t o_orderkey, o_totalprice; sx_i128 sum_qty; } sx_q18_row;

/* Each writes <= cap rows to host `out` and the row count to *nrows (host). */
sx_status sx_tpch_q1(sx_ctx* ctx, const sx_tpch_tables* t, const sx_tpch_params* p, sx_q1_row* out, int64_t cap,
                     int64_t* nrows);
sx_status sx_tpch_q6(sx_ctx* ctx, const sx_tpch_tables* t, const sx_tpch_params* p, sx_q6_row* out, int64_t* nrows);
sx_status sx_tpch_q3(sx_ctx* ctx, const sx_tpch_tables* t, const sx_tpch_params* p, sx_q3_row* out, int64_t cap,
                     int64_t* nrows);
sx_status sx_tpch_q9(sx_ctx* ctx, const sx_tpch_tables* t, const sx_tpch_params* p, sx_q9_row* out, int64_t cap,
                     int64_t* nrows);
sx_status sx_tpch_q18(sx_ctx* ctx, const sx_tpch_tables* t, const sx_tpch_params* p, sx_q18_row* out, int64_t cap,
                      int64_t* nrows);

#ifdef __cplusplus
}
#endif
#endif /* SX_H */
