/*
 * gen_cpu.c — host fill functions over gen/sxgen.h (libsxgen.so, C99).
 * Used by the oracle CLI, by tests (ctypes) and by bench.py's host-buffer
 * e2e leg.  Holds no relational arithmetic; see sxgen.h header comment.
 *
 * Ranges are half-open and 1-based in key/order-index space: [k0, k1).
 * Any output pointer may be NULL (column skipped).
 */
#include "sxgen.h"
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

EXPORT void sxg_cpu_sizes(int64_t sf_milli, int64_t out[5]) {
  out[0] = sxg_n_supplier(sf_milli);
  out[1] = sxg_n_customer(sf_milli);
  out[2] = sxg_n_part(sf_milli);
  out[3] = sxg_n_partsupp(sf_milli);
  out[4] = sxg_n_orders(sf_milli);
}

EXPORT void sxg_cpu_fill_supplier(uint64_t seed, int64_t k0, int64_t k1, int32_t* suppkey, int32_t* nationkey) {
  for (int64_t k = k0; k < k1; ++k) {
    if (suppkey) suppkey[k - k0] = (int32_t)k;
    if (nationkey) nationkey[k - k0] = sxg_s_nationkey(seed, k);
  }
}

EXPORT void sxg_cpu_fill_customer(uint64_t seed, int64_t k0, int64_t k1, int32_t* custkey, uint8_t* mktsegment,
                                  int32_t* nationkey) {
  for (int64_t k = k0; k < k1; ++k) {
    if (custkey) custkey[k - k0] = (int32_t)k;
    if (mktsegment) mktsegment[k - k0] = sxg_c_mktsegment(seed, k);
    if (nationkey) nationkey[k - k0] = sxg_c_nationkey(seed, k);
  }
}

/* total p_name bytes for parts [k0, k1) */
EXPORT int64_t sxg_cpu_part_name_bytes(uint64_t seed, int64_t k0, int64_t k1) {
  char buf[SXG_PNAME_MAXLEN];
  int64_t total = 0;
  for (int64_t k = k0; k < k1; ++k) total += sxg_p_name(seed, k, buf);
  return total;
}

/* offsets: int64[k1-k0+1] (Arrow large-string, offsets[0] = 0); chars may be NULL */
EXPORT void sxg_cpu_fill_part(uint64_t seed, int64_t k0, int64_t k1, int32_t* partkey, int64_t* offsets, char* chars,
                              int64_t* retailprice) {
  char buf[SXG_PNAME_MAXLEN];
  int64_t off = 0;
  if (offsets) offsets[0] = 0;
  for (int64_t k = k0; k < k1; ++k) {
    if (partkey) partkey[k - k0] = (int32_t)k;
    if (retailprice) retailprice[k - k0] = sxg_p_retailprice(k);
    if (offsets || chars) {
      int len = sxg_p_name(seed, k, buf);
      if (chars) memcpy(chars + off, buf, (size_t)len);
      off += len;
      if (offsets) offsets[k - k0 + 1] = off;
    }
  }
}

/* partsupp rows for parts [p0, p1): 4 rows per part */
EXPORT void sxg_cpu_fill_partsupp(uint64_t seed, int64_t sf_milli, int64_t p0, int64_t p1, int32_t* partkey,
                                  int32_t* suppkey, int64_t* supplycost) {
  int64_t S = sxg_n_supplier(sf_milli);
  int64_t r = 0;
  for (int64_t p = p0; p < p1; ++p)
    for (int64_t i = 0; i < 4; ++i, ++r) {
      if (partkey) partkey[r] = (int32_t)p;
      if (suppkey) suppkey[r] = (int32_t)sxg_ps_suppkey(p, i, S);
      if (supplycost) supplycost[r] = sxg_ps_supplycost(seed, p, i);
    }
}

EXPORT int64_t sxg_cpu_lineitem_count(uint64_t seed, int64_t i0, int64_t i1) {
  int64_t n = 0;
  for (int64_t i = i0; i < i1; ++i) n += sxg_o_nlines(seed, i);
  return n;
}

static inline void put_key(void* col, int key_bytes, int64_t r, int64_t v) {
  if (!col) return;
  if (key_bytes == 8) ((int64_t*)col)[r] = v;
  else ((int32_t*)col)[r] = (int32_t)v;
}

/* orders [i0, i1) and their lineitems (rows clustered by order, line order). key_bytes = 4 | 8 for orderkeys. */
EXPORT void sxg_cpu_fill_orders_lineitem(
    uint64_t seed, int64_t sf_milli, int64_t i0, int64_t i1, int key_bytes,
    void* o_orderkey, int32_t* o_custkey, int32_t* o_orderdate, int32_t* o_shippriority, int64_t* o_totalprice,
    void* l_orderkey, int32_t* l_partkey, int32_t* l_suppkey, int64_t* l_quantity, int64_t* l_extendedprice,
    int64_t* l_discount, int64_t* l_tax, uint8_t* l_returnflag, uint8_t* l_linestatus, int32_t* l_shipdate) {
  int64_t P = sxg_n_part(sf_milli), S = sxg_n_supplier(sf_milli), C = sxg_n_customer(sf_milli);
  int64_t r = 0;
  for (int64_t i = i0; i < i1; ++i) {
    int64_t o = i - i0;
    int64_t ok = sxg_o_orderkey(i);
    int32_t od = sxg_o_orderdate(seed, i);
    int32_t n = sxg_o_nlines(seed, i);
    put_key(o_orderkey, key_bytes, o, ok);
    if (o_custkey) o_custkey[o] = (int32_t)sxg_o_custkey(seed, i, C);
    if (o_orderdate) o_orderdate[o] = od;
    if (o_shippriority) o_shippriority[o] = 0;
    int64_t total = 0;
    for (int32_t j = 1; j <= n; ++j, ++r) {
      sxg_line L;
      sxg_l_line(seed, i, j, od, P, S, &L);
      total += sxg_line_price_term(&L);
      put_key(l_orderkey, key_bytes, r, ok);
      if (l_partkey) l_partkey[r] = L.partkey;
      if (l_suppkey) l_suppkey[r] = L.suppkey;
      if (l_quantity) l_quantity[r] = L.quantity;
      if (l_extendedprice) l_extendedprice[r] = L.extendedprice;
      if (l_discount) l_discount[r] = L.discount;
      if (l_tax) l_tax[r] = L.tax;
      if (l_returnflag) l_returnflag[r] = L.returnflag;
      if (l_linestatus) l_linestatus[r] = L.linestatus;
      if (l_shipdate) l_shipdate[r] = L.shipdate;
    }
    if (o_totalprice) o_totalprice[o] = total;
  }
}

/* For generator tests: the nation/segment dictionaries and the word list. */
EXPORT const char* sxg_cpu_word(int w) { return sxg_word(w); }

/* ---- operator micro-benchmarks (rows [r0, r1)) ---- */
EXPORT void sxg_cpu_fill_mb_build(int64_t r0, int64_t r1, int64_t* key, int64_t* payload) {
  for (int64_t i = r0; i < r1; ++i) {
    if (key) key[i - r0] = (int64_t)sxg_mb_build_key(i);
    if (payload) payload[i - r0] = i;
  }
}
EXPORT void sxg_cpu_fill_mb_probe(uint64_t seed, int64_t nb, int zipf, int64_t r0, int64_t r1, int64_t* key,
                                  int64_t* payload) {
  for (int64_t j = r0; j < r1; ++j) {
    if (key) key[j - r0] = (int64_t)sxg_mb_probe_key(seed, j, nb, zipf);
    if (payload) payload[j - r0] = j;
  }
}
EXPORT void sxg_cpu_fill_mb_groupby(uint64_t seed, int64_t G, int64_t r0, int64_t r1, int64_t* key, int64_t* value) {
  for (int64_t i = r0; i < r1; ++i) {
    if (key) key[i - r0] = (int64_t)sxg_mix64((uint64_t)sxg_mb_gb_group(seed, i, G));
    if (value) value[i - r0] = sxg_mb_gb_value(seed, i);
  }
}
EXPORT void sxg_cpu_fill_mb_sort(uint64_t seed, int64_t r0, int64_t r1, int64_t* key, int32_t* payload) {
  for (int64_t i = r0; i < r1; ++i) {
    if (key) key[i - r0] = sxg_mb_sort_key(seed, i);
    if (payload) payload[i - r0] = (int32_t)i;
  }
}
EXPORT int64_t sxg_cpu_mb_probe_rank(uint64_t seed, int64_t j, int64_t nb, int zipf) {
  return sxg_mb_probe_rank(seed, j, nb, zipf);
}
