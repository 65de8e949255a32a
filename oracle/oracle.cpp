// oracle.cpp — CPU ORACLE (test infrastructure only; see oracle.h header).
//
// Plain, slow, single-threaded, row at a time.  Every function follows the
// SQL definition it cites; library containers (std::map, std::unordered_map,
// std::stable_sort) are used as whole steps, with no blocking, fusion or
// reordering.  All sums are __int128 (SURVEY §8(c) reading R2).
#include "oracle.h"
#include "../gen/sxgen.h"  // nation names only (data definition, not operator arithmetic)

#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <unordered_map>
#include <unordered_set>
#include <vector>

typedef __int128 i128;

static or_i128 pack(i128 v) {
  or_i128 r;
  r.lo = (uint64_t)v;
  r.hi = (int64_t)(v >> 64);
  return r;
}
static i128 unpack(or_i128 v) { return (i128)(((unsigned __int128)(uint64_t)v.hi << 64) | v.lo); }

static const char* kNationNames[SXG_NNATIONS] = SXG_NATIONS_INIT;

extern "C" {

void or_default_params(or_params* p) {
  // TPC-H validation substitution parameters, days since 1970-01-01 (App. C),
  // decimals scaled by 100 (reading R1), Q6 BETWEEN bounds exact (reading R5).
  p->q1_shipdate_max = 10471;  // date '1998-12-01' - interval '90' day
  p->q3_segment = 1;           // dictionary index of 'BUILDING' (reading R10)
  p->q3_date = 9204;           // 1995-03-15
  p->q6_date_lo = 8766;        // 1994-01-01
  p->q6_date_hi = 9131;        // 1994-01-01 + 1 year
  p->q6_disc_lo = 5;           // 0.06 - 0.01
  p->q6_disc_hi = 7;           // 0.06 + 0.01
  p->q6_qty_lt = 2400;         // 24
  std::memset(p->q9_color, 0, sizeof(p->q9_color));
  std::strcpy(p->q9_color, "green");
  p->q18_qty_gt = 30000;       // 300
}

// Year of a day number by counting whole years from 1970 (Gregorian leap rule).
// Deliberately the naive definition; the GPU path uses a closed-form civil-from-days.
int32_t or_civil_year(int32_t days) {
  auto leap = [](int32_t y) { return (y % 4 == 0 && y % 100 != 0) || (y % 400 == 0); };
  int32_t y = 1970;
  if (days >= 0) {
    while (days >= (leap(y) ? 366 : 365)) { days -= leap(y) ? 366 : 365; ++y; }
  } else {
    while (days < 0) { --y; days += leap(y) ? 366 : 365; }
  }
  return y;
}

// ---------------------------------------------------------------- Q1
// TPC-H Q1 (SURVEY §8(c) "Q1", App. B): lineitem rows with l_shipdate <= date '1998-12-01' - 90 days,
// grouped by (l_returnflag, l_linestatus), ordered by the same.  avg = (double)sum/(double)count/100 (R3).
int64_t or_q1(const or_tables* t, const or_params* p, or_q1_row* out, int64_t cap) {
  struct Acc { i128 qty = 0, base = 0, disc_price = 0, charge = 0, disc = 0; int64_t count = 0; };
  std::map<std::pair<uint8_t, uint8_t>, Acc> groups;
  for (int64_t r = 0; r < t->n_lineitem; ++r) {
    if (!(t->l_shipdate[r] <= p->q1_shipdate_max)) continue;
    Acc& a = groups[{t->l_returnflag[r], t->l_linestatus[r]}];
    i128 ext = t->l_extendedprice[r], disc = t->l_discount[r], tax = t->l_tax[r];
    a.qty += t->l_quantity[r];                        // sum(l_quantity)                 scale 2
    a.base += ext;                                    // sum(l_extendedprice)            scale 2
    a.disc_price += ext * (100 - disc);               // sum(l_extendedprice*(1-l_discount))           scale 4
    a.charge += ext * (100 - disc) * (100 + tax);     // sum(l_extendedprice*(1-l_discount)*(1+l_tax)) scale 6
    a.disc += disc;                                   // for avg(l_discount)             scale 2
    a.count += 1;                                     // count(*)
  }
  int64_t g = 0;
  for (auto& kv : groups) {
    if (g >= cap) return -1;
    or_q1_row& o = out[g++];
    const Acc& a = kv.second;
    o.returnflag = kv.first.first;
    o.linestatus = kv.first.second;
    o.sum_qty = pack(a.qty);
    o.sum_base_price = pack(a.base);
    o.sum_disc_price = pack(a.disc_price);
    o.sum_charge = pack(a.charge);
    o.sum_disc = pack(a.disc);
    o.count_order = a.count;
    o.avg_qty = (double)a.qty / (double)a.count / 100.0;
    o.avg_price = (double)a.base / (double)a.count / 100.0;
    o.avg_disc = (double)a.disc / (double)a.count / 100.0;
  }
  return g;
}

// ---------------------------------------------------------------- Q6
// TPC-H Q6: sum(l_extendedprice*l_discount) over shipdate in [1994-01-01, 1995-01-01),
// discount between 0.05 and 0.07 (inclusive, exact decimals; R5), quantity < 24.  NULL if no row (R20).
int64_t or_q6(const or_tables* t, const or_params* p, or_q6_row* out) {
  i128 sum = 0;
  int64_t n = 0;
  for (int64_t r = 0; r < t->n_lineitem; ++r) {
    if (t->l_shipdate[r] >= p->q6_date_lo && t->l_shipdate[r] < p->q6_date_hi &&
        t->l_discount[r] >= p->q6_disc_lo && t->l_discount[r] <= p->q6_disc_hi && t->l_quantity[r] < p->q6_qty_lt) {
      sum += (i128)t->l_extendedprice[r] * t->l_discount[r];  // scale 4
      ++n;
    }
  }
  out->revenue = pack(sum);
  out->is_null = n == 0;
  return 1;
}

// ---------------------------------------------------------------- Q3
// TPC-H Q3: customer(c_mktsegment = SEGMENT) ⋈ orders(o_orderdate < DATE) ⋈ lineitem(l_shipdate > DATE),
// group by (l_orderkey, o_orderdate, o_shippriority), revenue = sum(ext*(100-disc)) [scale 4],
// order by revenue desc, o_orderdate asc, then l_orderkey asc (tie-break reading R6), limit.
int64_t or_q3(const or_tables* t, const or_params* p, int64_t limit, or_q3_row* out, int64_t cap) {
  std::unordered_set<int64_t> cust;  // C = {custkey | mktsegment = SEGMENT}
  for (int64_t r = 0; r < t->n_customer; ++r)
    if (t->c_mktsegment[r] == p->q3_segment) cust.insert(t->c_custkey[r]);
  std::unordered_map<int64_t, int64_t> ord;  // orderkey -> orders row, for orders of C before DATE
  for (int64_t r = 0; r < t->n_orders; ++r)
    if (t->o_orderdate[r] < p->q3_date && cust.count(t->o_custkey[r])) ord.emplace(t->o_orderkey[r], r);
  std::map<std::tuple<int64_t, int32_t, int32_t>, i128> groups;
  for (int64_t r = 0; r < t->n_lineitem; ++r) {
    if (!(t->l_shipdate[r] > p->q3_date)) continue;
    auto it = ord.find(t->l_orderkey[r]);
    if (it == ord.end()) continue;
    int64_t o = it->second;
    groups[{t->l_orderkey[r], t->o_orderdate[o], t->o_shippriority[o]}] +=
        (i128)t->l_extendedprice[r] * (100 - t->l_discount[r]);
  }
  std::vector<or_q3_row> rows;
  for (auto& kv : groups) {
    or_q3_row x;
    x.l_orderkey = std::get<0>(kv.first);
    x.o_orderdate = std::get<1>(kv.first);
    x.o_shippriority = std::get<2>(kv.first);
    x.revenue = pack(kv.second);
    rows.push_back(x);
  }
  std::sort(rows.begin(), rows.end(), [](const or_q3_row& a, const or_q3_row& b) {
    i128 ra = unpack(a.revenue), rb = unpack(b.revenue);
    if (ra != rb) return ra > rb;
    if (a.o_orderdate != b.o_orderdate) return a.o_orderdate < b.o_orderdate;
    return a.l_orderkey < b.l_orderkey;
  });
  int64_t n = std::min<int64_t>((int64_t)rows.size(), limit < 0 ? (int64_t)rows.size() : limit);
  if (n > cap) return -1;
  for (int64_t i = 0; i < n; ++i) out[i] = rows[i];
  return n;
}

// ---------------------------------------------------------------- Q9
// TPC-H Q9: part(p_name like '%COLOR%') ⋈ lineitem ⋈ partsupp(ps_partkey, ps_suppkey) ⋈ supplier ⋈ orders ⋈ nation;
// amount = l_extendedprice*(1-l_discount) - ps_supplycost*l_quantity [scale 4]; group by (n_name, year(o_orderdate));
// order by n_name asc, o_year desc.  LIKE is a case-sensitive byte substring test (R9).
int64_t or_q9(const or_tables* t, const or_params* p, or_q9_row* out, int64_t cap) {
  std::string color(p->q9_color);
  std::unordered_set<int64_t> green;
  for (int64_t r = 0; r < t->n_part; ++r) {
    std::string name((const char*)t->p_name_chars + t->p_name_offsets[r],
                     (size_t)(t->p_name_offsets[r + 1] - t->p_name_offsets[r]));
    if (name.find(color) != std::string::npos) green.insert(t->p_partkey[r]);
  }
  std::map<std::pair<int64_t, int64_t>, int64_t> ps_cost;  // (partkey, suppkey) -> supplycost
  for (int64_t r = 0; r < t->n_partsupp; ++r) ps_cost[{t->ps_partkey[r], t->ps_suppkey[r]}] = t->ps_supplycost[r];
  std::unordered_map<int64_t, int32_t> s_nation;
  for (int64_t r = 0; r < t->n_supplier; ++r) s_nation[t->s_suppkey[r]] = t->s_nationkey[r];
  std::unordered_map<int64_t, int32_t> o_date;
  for (int64_t r = 0; r < t->n_orders; ++r) o_date[t->o_orderkey[r]] = t->o_orderdate[r];
  // group key: (n_name, o_year) -> profit; n_name ascending (string order), o_year descending
  std::map<std::pair<std::string, int32_t>, std::pair<int32_t, i128>> groups;  // value: (nationkey, sum)
  for (int64_t r = 0; r < t->n_lineitem; ++r) {
    if (!green.count(t->l_partkey[r])) continue;
    auto ps = ps_cost.find({t->l_partkey[r], t->l_suppkey[r]});
    auto s = s_nation.find(t->l_suppkey[r]);
    auto o = o_date.find(t->l_orderkey[r]);
    if (ps == ps_cost.end() || s == s_nation.end() || o == o_date.end()) continue;  // inner joins
    int32_t year = or_civil_year(o->second);
    i128 amount = (i128)t->l_extendedprice[r] * (100 - t->l_discount[r]) - (i128)ps->second * t->l_quantity[r];
    auto& g = groups[{std::string(kNationNames[s->second]), -year}];  // -year: descending
    g.first = s->second;
    g.second += amount;
  }
  int64_t n = 0;
  for (auto& kv : groups) {
    if (n >= cap) return -1;
    out[n].nationkey = kv.second.first;
    out[n].o_year = -kv.first.second;
    out[n].sum_profit = pack(kv.second.second);
    ++n;
  }
  return n;
}

// ---------------------------------------------------------------- Q18
// TPC-H Q18: orders whose lineitems' sum(l_quantity) > QUANTITY, joined with customer and lineitem,
// group by (c_name, c_custkey, o_orderkey, o_orderdate, o_totalprice) sum(l_quantity),
// order by o_totalprice desc, o_orderdate asc, then o_orderkey asc (R6), limit 100.
// c_name is derived from c_custkey ("Customer#%09d", R8), so grouping by c_custkey is the same grouping.
int64_t or_q18(const or_tables* t, const or_params* p, int64_t limit, or_q18_row* out, int64_t cap) {
  std::unordered_map<int64_t, i128> s;  // subquery: l_orderkey -> sum(l_quantity)
  for (int64_t r = 0; r < t->n_lineitem; ++r) s[t->l_orderkey[r]] += t->l_quantity[r];
  std::unordered_set<int64_t> big;
  for (auto& kv : s)
    if (kv.second > p->q18_qty_gt) big.insert(kv.first);
  std::unordered_set<int64_t> custs;
  for (int64_t r = 0; r < t->n_customer; ++r) custs.insert(t->c_custkey[r]);
  std::unordered_map<int64_t, int64_t> ord;  // orderkey -> orders row (o_orderkey in big, customer exists)
  for (int64_t r = 0; r < t->n_orders; ++r)
    if (big.count(t->o_orderkey[r]) && custs.count(t->o_custkey[r])) ord.emplace(t->o_orderkey[r], r);
  std::map<int64_t, i128> sums;  // per joined order: sum(l_quantity) over its lineitems (recomputed literally)
  for (int64_t r = 0; r < t->n_lineitem; ++r)
    if (ord.count(t->l_orderkey[r])) sums[t->l_orderkey[r]] += t->l_quantity[r];
  std::vector<or_q18_row> rows;
  for (auto& kv : sums) {
    int64_t o = ord[kv.first];
    or_q18_row x;
    x.c_custkey = t->o_custkey[o];
    x.o_orderkey = kv.first;
    x.o_orderdate = t->o_orderdate[o];
    x.o_totalprice = t->o_totalprice[o];
    x.sum_qty = pack(kv.second);
    rows.push_back(x);
  }
  std::sort(rows.begin(), rows.end(), [](const or_q18_row& a, const or_q18_row& b) {
    if (a.o_totalprice != b.o_totalprice) return a.o_totalprice > b.o_totalprice;
    if (a.o_orderdate != b.o_orderdate) return a.o_orderdate < b.o_orderdate;
    return a.o_orderkey < b.o_orderkey;
  });
  int64_t n = std::min<int64_t>((int64_t)rows.size(), limit < 0 ? (int64_t)rows.size() : limit);
  if (n > cap) return -1;
  for (int64_t i = 0; i < n; ++i) out[i] = rows[i];
  return n;
}

// ---------------------------------------------------------------- operators
// filter (SPEC S:208-216 shape; P:254 predicate pushdown): ascending row ids where the conjunction holds.
static bool pred_holds(const or_pred& q, int64_t v) {
  switch (q.op) {
    case OR_LT: return v < q.lo;
    case OR_LE: return v <= q.lo;
    case OR_GT: return v > q.lo;
    case OR_GE: return v >= q.lo;
    case OR_EQ: return v == q.lo;
    case OR_NE: return v != q.lo;
    case OR_BETWEEN: return q.lo <= v && v <= q.hi;
  }
  return false;
}

int64_t or_filter(int64_t n, const int64_t* const* cols, const or_pred* preds, int32_t npreds, int32_t* out_sel) {
  int64_t k = 0;
  for (int64_t r = 0; r < n; ++r) {
    bool ok = true;
    for (int32_t i = 0; i < npreds; ++i) ok = ok && pred_holds(preds[i], cols[preds[i].col][r]);
    if (ok) out_sel[k++] = (int32_t)r;
  }
  return k;
}

int64_t or_contains(int64_t n, const int64_t* offsets, const uint8_t* chars, const char* pattern, int32_t plen,
                    int32_t* out_sel) {
  std::string pat(pattern, (size_t)plen);
  int64_t k = 0;
  for (int64_t r = 0; r < n; ++r) {
    std::string s((const char*)chars + offsets[r], (size_t)(offsets[r + 1] - offsets[r]));
    if (s.find(pat) != std::string::npos) out_sel[k++] = (int32_t)r;
  }
  return k;
}

static i128 eval_row(const int64_t* const* cols, const or_expr* e, int64_t r) {
  i128 v = 0;
  for (int32_t ti = 0; ti < e->nterms; ++ti) {
    const or_term& tm = e->t[ti];
    i128 prod = tm.coef;
    for (int32_t f = 0; f < tm.nf; ++f) prod *= (i128)tm.f[f].mul * cols[tm.f[f].col][r] + tm.f[f].add;
    v += prod;
  }
  return v;
}

void or_eval_expr(int64_t n, const int64_t* const* cols, const or_expr* e, or_i128* out) {
  for (int64_t r = 0; r < n; ++r) out[r] = pack(eval_row(cols, e, r));
}

// join: inner = all matching (probe, build) pairs, probe-major; semi = probe rows with a
// match; anti = probe rows without one.  Library step: std::unordered_multimap-like map of key -> build rows.
int64_t or_join(int64_t nb, const int64_t* bkeys, int64_t np, const int64_t* pkeys, int32_t type,
                int32_t* out_probe, int32_t* out_build, int64_t cap) {
  std::unordered_map<int64_t, std::vector<int32_t>> ht;
  for (int64_t b = 0; b < nb; ++b) ht[bkeys[b]].push_back((int32_t)b);
  int64_t k = 0;
  for (int64_t q = 0; q < np; ++q) {
    auto it = ht.find(pkeys[q]);
    bool hit = it != ht.end();
    if (type == 0 && hit) {
      for (int32_t b : it->second) {
        if (k >= cap) return -1;
        out_probe[k] = (int32_t)q;
        out_build[k] = b;
        ++k;
      }
    } else if ((type == 1 && hit) || (type == 2 && !hit)) {
      if (k >= cap) return -1;
      out_probe[k++] = (int32_t)q;
    }
  }
  return k;
}

// group-by: one row per distinct key tuple, ascending; sum/min/max of exact int128 expression
// values, count(*), avg = (double)sum/(double)count/10^scale (R3).
int64_t or_groupby(int64_t n, const int64_t* const* cols, int32_t nkeys, const int32_t* key_cols, int32_t naggs,
                   const int32_t* agg_ops, const or_expr* agg_exprs, const int32_t* avg_scale,
                   int64_t* const* out_keys, or_i128* const* out_aggs, double* const* out_avg, int64_t cap) {
  struct Acc { std::vector<i128> sum, mn, mx; int64_t count = 0; };
  std::map<std::vector<int64_t>, Acc> groups;
  if (nkeys == 0 && n == 0) return 0;  // keyless: caller handles the empty-input NULL row
  for (int64_t r = 0; r < n; ++r) {
    std::vector<int64_t> key;
    for (int32_t k = 0; k < nkeys; ++k) key.push_back(cols[key_cols[k]][r]);
    Acc& a = groups[key];
    if (a.sum.empty()) { a.sum.assign(naggs, 0); a.mn.assign(naggs, 0); a.mx.assign(naggs, 0); }
    for (int32_t i = 0; i < naggs; ++i) {
      i128 v = eval_row(cols, &agg_exprs[i], r);
      a.sum[i] += v;
      if (a.count == 0 || v < a.mn[i]) a.mn[i] = v;
      if (a.count == 0 || v > a.mx[i]) a.mx[i] = v;
    }
    a.count += 1;
  }
  int64_t g = 0;
  for (auto& kv : groups) {
    if (g >= cap) return -1;
    for (int32_t k = 0; k < nkeys; ++k) out_keys[k][g] = kv.first[k];
    for (int32_t i = 0; i < naggs; ++i) {
      const Acc& a = kv.second;
      i128 v = 0;
      switch (agg_ops[i]) {
        case 0: v = a.sum[i]; break;
        case 1: v = a.count; break;
        case 2: v = a.mn[i]; break;
        case 3: v = a.mx[i]; break;
        case 4: {
          v = a.sum[i];
          double sc = 1.0;
          for (int32_t s = 0; s < avg_scale[i]; ++s) sc *= 10.0;
          out_avg[i][g] = (double)a.sum[i] / (double)a.count / sc;
          break;
        }
      }
      out_aggs[i][g] = pack(v);
    }
    ++g;
  }
  return g;
}

// sort: stable permutation by the key columns (each asc or desc); top-k = its prefix.
int64_t or_sort(int64_t n, const or_i128* const* keys, int32_t nkeys, const int32_t* desc, int64_t k, int32_t* out_perm) {
  std::vector<int32_t> perm((size_t)n);
  for (int64_t i = 0; i < n; ++i) perm[(size_t)i] = (int32_t)i;
  std::stable_sort(perm.begin(), perm.end(), [&](int32_t a, int32_t b) {
    for (int32_t c = 0; c < nkeys; ++c) {
      i128 x = unpack(keys[c][a]), y = unpack(keys[c][b]);
      if (x != y) return desc[c] ? x > y : x < y;
    }
    return false;
  });
  int64_t m = (k < 0 || k > n) ? n : k;
  for (int64_t i = 0; i < m; ++i) out_perm[i] = perm[(size_t)i];
  return m;
}

// ---- operator µbenchmarks (SURVEY §8(c) "µbench join" / "µbench group-by") -----------------------
// splitmix64 finalizer z -> (z ^ z>>30) * C1 -> (. ^ .>>27) * C2 -> . ^ .>>31 is a bijection; its
// inverse undoes each step: x ^ x>>s is inverted by x ^ x>>s ^ x>>2s ^ ..., multiplication by an
// odd constant by its inverse mod 2^64.
uint64_t or_unmix64(uint64_t z) {
  z = z ^ (z >> 31) ^ (z >> 62);
  z *= 0x319642b2d24d8ec3ULL;  // C2^-1 mod 2^64
  z = z ^ (z >> 27) ^ (z >> 54);
  z *= 0x96de1b173f119089ULL;  // C1^-1 mod 2^64
  z = z ^ (z >> 30) ^ (z >> 60);
  return z;
}

uint64_t or_pair_mix(int64_t b, int64_t p) {
  uint64_t z = (uint64_t)b * 0x9e3779b97f4a7c15ULL ^ (uint64_t)p;
  z = (z ^ (z >> 32)) * 0xd6e8feb86659fd93ULL;
  return z ^ (z >> 32);
}

static void summary_add(or_join_summary* s, i128& sb, i128& sp, int64_t b, int64_t p) {
  s->count += 1;
  sb += b;
  sp += p;
  s->pair_hash += or_pair_mix(b, p);
}

void or_mb_join_closed(int64_t nb, int64_t np, const int64_t* pkeys, const int64_t* ppay, or_join_summary* out) {
  std::memset(out, 0, sizeof *out);
  i128 sb = 0, sp = 0;
  for (int64_t j = 0; j < np; ++j) {
    uint64_t i = or_unmix64((uint64_t)pkeys[j]);
    if (i < (uint64_t)nb) summary_add(out, sb, sp, (int64_t)i, ppay[j]);
  }
  out->sum_build = pack(sb);
  out->sum_probe = pack(sp);
}

void or_mb_join_hash(int64_t nb, const int64_t* bkeys, const int64_t* bpay, int64_t np, const int64_t* pkeys,
                     const int64_t* ppay, or_join_summary* out) {
  std::memset(out, 0, sizeof *out);
  std::unordered_multimap<int64_t, int64_t> m;
  m.reserve((size_t)nb);
  for (int64_t i = 0; i < nb; ++i) m.emplace(bkeys[i], bpay[i]);
  i128 sb = 0, sp = 0;
  for (int64_t j = 0; j < np; ++j) {
    auto r = m.equal_range(pkeys[j]);
    for (auto it = r.first; it != r.second; ++it) summary_add(out, sb, sp, it->second, ppay[j]);
  }
  out->sum_build = pack(sb);
  out->sum_probe = pack(sp);
}

int64_t or_mb_groupby_direct(int64_t n, const int64_t* keys, const int64_t* vals, int64_t G, or_i128* sum,
                             int64_t* cnt, int64_t* mn, int64_t* mx) {
  std::vector<i128> s((size_t)G, 0);
  for (int64_t g = 0; g < G; ++g) { cnt[g] = 0; mn[g] = INT64_MAX; mx[g] = INT64_MIN; }
  for (int64_t r = 0; r < n; ++r) {
    uint64_t g = or_unmix64((uint64_t)keys[r]);
    if (g >= (uint64_t)G) return -1;
    s[g] += vals[r];
    cnt[g] += 1;
    mn[g] = std::min(mn[g], vals[r]);
    mx[g] = std::max(mx[g], vals[r]);
  }
  int64_t present = 0;
  for (int64_t g = 0; g < G; ++g) {
    sum[g] = pack(s[(size_t)g]);
    present += cnt[g] > 0;
  }
  return present;
}

}  // extern "C"
