// sx_oracle — CLI around the CPU oracle (test infrastructure only).
//
//   sx_oracle --query q1|q3|q6|q9|q18|all --sf-milli N [--seed S] [--q18-qty Q] [--reps R]
//
// Generates the needed columns on the host (gen/gen_cpu.c), runs the query
// single-threaded and prints one JSON object per query:
//   {"query": "q1", "sf_milli": N, "seed": S, "rows": [...], "seconds": [...]}
// "seconds" times the query only (generation excluded; hot run).
// int128 values print as JSON integers.
#include "oracle.h"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

extern "C" {
void sxg_cpu_sizes(int64_t sf_milli, int64_t out[5]);
void sxg_cpu_fill_supplier(uint64_t, int64_t, int64_t, int32_t*, int32_t*);
void sxg_cpu_fill_customer(uint64_t, int64_t, int64_t, int32_t*, uint8_t*, int32_t*);
int64_t sxg_cpu_part_name_bytes(uint64_t, int64_t, int64_t);
void sxg_cpu_fill_part(uint64_t, int64_t, int64_t, int32_t*, int64_t*, char*, int64_t*);
void sxg_cpu_fill_partsupp(uint64_t, int64_t, int64_t, int64_t, int32_t*, int32_t*, int64_t*);
int64_t sxg_cpu_lineitem_count(uint64_t, int64_t, int64_t);
void sxg_cpu_fill_orders_lineitem(uint64_t, int64_t, int64_t, int64_t, int, void*, int32_t*, int32_t*, int32_t*,
                                  int64_t*, void*, int32_t*, int32_t*, int64_t*, int64_t*, int64_t*, int64_t*,
                                  uint8_t*, uint8_t*, int32_t*);
}

static std::string i128s(or_i128 v) {
  __int128 x = (__int128)(((unsigned __int128)(uint64_t)v.hi << 64) | v.lo);
  if (x == 0) return "0";
  bool neg = x < 0;
  unsigned __int128 u = neg ? -(unsigned __int128)x : (unsigned __int128)x;
  std::string s;
  while (u) { s.push_back((char)('0' + (int)(u % 10))); u /= 10; }
  if (neg) s.push_back('-');
  return std::string(s.rbegin(), s.rend());
}

struct Data {
  std::vector<int64_t> l_orderkey, l_quantity, l_ext, l_disc, l_tax;
  std::vector<int32_t> l_partkey, l_suppkey, l_ship;
  std::vector<uint8_t> l_rf, l_ls;
  std::vector<int64_t> o_orderkey, o_totalprice;
  std::vector<int32_t> o_custkey, o_orderdate, o_shippriority;
  std::vector<int32_t> c_custkey; std::vector<uint8_t> c_seg;
  std::vector<int32_t> p_partkey; std::vector<int64_t> p_off; std::vector<char> p_chars;
  std::vector<int32_t> ps_partkey, ps_suppkey; std::vector<int64_t> ps_cost;
  std::vector<int32_t> s_suppkey, s_nation;
};

template <class T> static T* P(std::vector<T>& v, bool need) { return need ? v.data() : nullptr; }

static void generate(const std::string& q, int64_t sfm, uint64_t seed, Data& d, or_tables& t) {
  int64_t sz[5];
  sxg_cpu_sizes(sfm, sz);
  bool all = q == "all";
  bool need_l = true;
  bool need_o = all || q == "q3" || q == "q9" || q == "q18";
  bool need_c = all || q == "q3" || q == "q18";
  bool need_p = all || q == "q9";
  std::memset(&t, 0, sizeof(t));
  int64_t O = sz[4];
  if (need_l || need_o) {
    int64_t nl = sxg_cpu_lineitem_count(seed, 1, O + 1);
    bool q1 = all || q == "q1", q3 = all || q == "q3", q6 = all || q == "q6", q9 = all || q == "q9",
         q18 = all || q == "q18";
    auto rs = [&](auto& v, bool need, int64_t n) { if (need) v.resize((size_t)n); };
    rs(d.l_orderkey, q3 || q9 || q18, nl); rs(d.l_partkey, q9, nl); rs(d.l_suppkey, q9, nl);
    rs(d.l_quantity, q1 || q6 || q9 || q18, nl); rs(d.l_ext, q1 || q3 || q6 || q9, nl);
    rs(d.l_disc, q1 || q3 || q6 || q9, nl); rs(d.l_tax, q1, nl); rs(d.l_rf, q1, nl); rs(d.l_ls, q1, nl);
    rs(d.l_ship, q1 || q3 || q6, nl);
    rs(d.o_orderkey, need_o, O); rs(d.o_custkey, q3 || q18, O); rs(d.o_orderdate, need_o, O);
    rs(d.o_shippriority, q3, O); rs(d.o_totalprice, q18, O);
    auto p = [](auto& v) { return v.empty() ? nullptr : v.data(); };
    sxg_cpu_fill_orders_lineitem(seed, sfm, 1, O + 1, 8, p(d.o_orderkey), p(d.o_custkey), p(d.o_orderdate),
                                 p(d.o_shippriority), p(d.o_totalprice), p(d.l_orderkey), p(d.l_partkey),
                                 p(d.l_suppkey), p(d.l_quantity), p(d.l_ext), p(d.l_disc), p(d.l_tax), p(d.l_rf),
                                 p(d.l_ls), p(d.l_ship));
    t.n_lineitem = nl;
    t.l_orderkey = p(d.l_orderkey); t.l_partkey = p(d.l_partkey); t.l_suppkey = p(d.l_suppkey);
    t.l_quantity = p(d.l_quantity); t.l_extendedprice = p(d.l_ext); t.l_discount = p(d.l_disc);
    t.l_tax = p(d.l_tax); t.l_returnflag = p(d.l_rf); t.l_linestatus = p(d.l_ls); t.l_shipdate = p(d.l_ship);
    t.n_orders = O;
    t.o_orderkey = p(d.o_orderkey); t.o_custkey = p(d.o_custkey); t.o_orderdate = p(d.o_orderdate);
    t.o_shippriority = p(d.o_shippriority); t.o_totalprice = p(d.o_totalprice);
  }
  if (need_c) {
    int64_t C = sz[1];
    d.c_custkey.resize((size_t)C); d.c_seg.resize((size_t)C);
    sxg_cpu_fill_customer(seed, 1, C + 1, d.c_custkey.data(), d.c_seg.data(), nullptr);
    t.n_customer = C; t.c_custkey = d.c_custkey.data(); t.c_mktsegment = d.c_seg.data();
  }
  if (need_p) {
    int64_t Pn = sz[2], S = sz[0];
    int64_t nb = sxg_cpu_part_name_bytes(seed, 1, Pn + 1);
    d.p_partkey.resize((size_t)Pn); d.p_off.resize((size_t)Pn + 1); d.p_chars.resize((size_t)nb + 1);
    sxg_cpu_fill_part(seed, 1, Pn + 1, d.p_partkey.data(), d.p_off.data(), d.p_chars.data(), nullptr);
    d.ps_partkey.resize((size_t)(4 * Pn)); d.ps_suppkey.resize((size_t)(4 * Pn)); d.ps_cost.resize((size_t)(4 * Pn));
    sxg_cpu_fill_partsupp(seed, sfm, 1, Pn + 1, d.ps_partkey.data(), d.ps_suppkey.data(), d.ps_cost.data());
    d.s_suppkey.resize((size_t)S); d.s_nation.resize((size_t)S);
    sxg_cpu_fill_supplier(seed, 1, S + 1, d.s_suppkey.data(), d.s_nation.data());
    t.n_part = Pn; t.p_partkey = d.p_partkey.data(); t.p_name_offsets = d.p_off.data();
    t.p_name_chars = (const uint8_t*)d.p_chars.data();
    t.n_partsupp = 4 * Pn; t.ps_partkey = d.ps_partkey.data(); t.ps_suppkey = d.ps_suppkey.data();
    t.ps_supplycost = d.ps_cost.data();
    t.n_supplier = S; t.s_suppkey = d.s_suppkey.data(); t.s_nationkey = d.s_nation.data();
  }
}

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  std::string query = "all";
  int64_t sfm = 10, reps = 1, q18 = -1;
  uint64_t seed = 42;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    auto next = [&]() { if (i + 1 >= argc) { std::fprintf(stderr, "missing value for %s\n", a.c_str()); std::exit(2); } return std::string(argv[++i]); };
    if (a == "--query") query = next();
    else if (a == "--sf-milli") sfm = std::atoll(next().c_str());
    else if (a == "--seed") seed = std::strtoull(next().c_str(), nullptr, 10);
    else if (a == "--reps") reps = std::atoll(next().c_str());
    else if (a == "--q18-qty") q18 = std::atoll(next().c_str());
    else { std::fprintf(stderr, "unknown arg %s\n", a.c_str()); return 2; }
  }
  Data d;
  or_tables t;
  generate(query, sfm, seed, d, t);
  or_params prm;
  or_default_params(&prm);
  if (q18 >= 0) prm.q18_qty_gt = q18;
  std::vector<std::string> qs;
  if (query == "all") qs = {"q1", "q6", "q3", "q9", "q18"}; else qs = {query};
  for (auto& q : qs) {
    std::vector<double> secs;
    std::string rows;
    for (int64_t rep = 0; rep < reps; ++rep) {
      rows.clear();
      double t0 = now();
      if (q == "q1") {
        std::vector<or_q1_row> r(64);
        int64_t n = or_q1(&t, &prm, r.data(), 64);
        secs.push_back(now() - t0);
        for (int64_t i = 0; i < n; ++i) {
          char buf[512];
          std::snprintf(buf, sizeof buf, "%s[\"%c\", \"%c\", %s, %s, %s, %s, %.17g, %.17g, %.17g, %lld]", i ? ", " : "",
                        r[i].returnflag, r[i].linestatus, i128s(r[i].sum_qty).c_str(), i128s(r[i].sum_base_price).c_str(),
                        i128s(r[i].sum_disc_price).c_str(), i128s(r[i].sum_charge).c_str(), r[i].avg_qty, r[i].avg_price,
                        r[i].avg_disc, (long long)r[i].count_order);
          rows += buf;
        }
      } else if (q == "q6") {
        or_q6_row r;
        or_q6(&t, &prm, &r);
        secs.push_back(now() - t0);
        rows = "[" + (r.is_null ? std::string("null") : i128s(r.revenue)) + "]";
      } else if (q == "q3") {
        std::vector<or_q3_row> r(10);
        int64_t n = or_q3(&t, &prm, 10, r.data(), 10);
        secs.push_back(now() - t0);
        for (int64_t i = 0; i < n; ++i)
          rows += (i ? ", [" : "[") + std::to_string(r[i].l_orderkey) + ", " + i128s(r[i].revenue) + ", " +
                  std::to_string(r[i].o_orderdate) + ", " + std::to_string(r[i].o_shippriority) + "]";
      } else if (q == "q9") {
        std::vector<or_q9_row> r(1024);
        int64_t n = or_q9(&t, &prm, r.data(), 1024);
        secs.push_back(now() - t0);
        for (int64_t i = 0; i < n; ++i)
          rows += (i ? ", [" : "[") + std::to_string(r[i].nationkey) + ", " + std::to_string(r[i].o_year) + ", " +
                  i128s(r[i].sum_profit) + "]";
      } else if (q == "q18") {
        std::vector<or_q18_row> r(100);
        int64_t n = or_q18(&t, &prm, 100, r.data(), 100);
        secs.push_back(now() - t0);
        for (int64_t i = 0; i < n; ++i)
          rows += (i ? ", [" : "[") + std::to_string(r[i].c_custkey) + ", " + std::to_string(r[i].o_orderkey) + ", " +
                  std::to_string(r[i].o_orderdate) + ", " + std::to_string(r[i].o_totalprice) + ", " +
                  i128s(r[i].sum_qty) + "]";
      } else {
        std::fprintf(stderr, "unknown query %s\n", q.c_str());
        return 2;
      }
    }
    std::string s;
    for (size_t i = 0; i < secs.size(); ++i) s += (i ? ", " : "") + std::to_string(secs[i]);
    std::printf("{\"query\": \"%s\", \"sf_milli\": %lld, \"seed\": %llu, \"q18_qty\": %lld, \"n_lineitem\": %lld, "
                "\"rows\": [%s], \"seconds\": [%s]}\n",
                q.c_str(), (long long)sfm, (unsigned long long)seed, (long long)prm.q18_qty_gt,
                (long long)t.n_lineitem, rows.c_str(), s.c_str());
    std::fflush(stdout);
  }
  return 0;
}
