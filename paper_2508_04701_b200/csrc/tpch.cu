// tpch.cu — fixed-plan executor for TPC-H Q1/Q3/Q6/Q9/Q18 (stands in for the Substrait
// consumer, BASELINE.json north_star).  Each plan is a sequence of sx_* operator calls
// (SURVEY.md §8(a) "Per-query fixed plans"); every step runs in libsx kernels; the only
// host work is argument marshalling and the final device->host copy of the (tiny) result.
// Semantics: SURVEY §8(c) "Definitions"; readings R1..R21 in DESIGN.md.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "gb_host.cuh"
#include "join.cuh"

using namespace sx;

namespace {

// ------------------------------------------------------------------------------------------
// Compile-time row programs for the plans' dominant group-bys (see groupby.cuh "row programs").
// Same kernels and table layout as sx_groupby_agg; the expressions are compiled instead of
// interpreted, so each column is loaded once per row and shared subexpressions are reused.
// State order = the order gb_plan() derives from the plan's aggregate list (checked on the host).
__device__ __forceinline__ int64_t sub_ck(int64_t a, int64_t b, bool& ovf) {
  int64_t s = (int64_t)((uint64_t)a - (uint64_t)b);
  ovf |= ((a ^ b) & (a ^ s)) < 0;
  return s;
}

// Q1: where l_shipdate <= X; key (l_returnflag, l_linestatus);
// states: 0 sum(qty) 1 sum(ext) 2 sum(ext*(100-disc)) 3 sum(ext*(100-disc)*(100+tax)) 4 count 5 sum(disc)
struct Q1Prog {
  const int32_t* ship;
  const uint8_t *rf, *ls;
  const long long *qty, *ext, *disc, *tax;
  int32_t ship_max;
  int* ovf_flag;
  static constexpr int kMaxNst = 6;
  static constexpr int kUnrollStates = 6;
  static constexpr bool kSortedOK = false;
  bool no_filter() const { return false; }
  template <int I>
  __device__ __forceinline__ void keys_only(const int32_t (&)[I], const bool (&)[I], uint64_t (&)[I]) const {}
  template <int I>
  struct Cache { int64_t qty[I], ext[I], disc[I], tax[I]; };
  __device__ __forceinline__ int kind(int a, const Layout&) const { return a == 4 ? ST_COUNT : ST_SUM; }
  template <int I>
  __device__ __forceinline__ void where_keys(const int32_t (&row)[I], bool (&alive)[I], uint64_t (&key)[I],
                                             Cache<I>& c) const {
    int32_t sd[I];
#pragma unroll
    for (int i = 0; i < I; ++i) sd[i] = alive[i] ? __ldg(ship + row[i]) : 0;
#pragma unroll
    for (int i = 0; i < I; ++i) alive[i] = alive[i] && sd[i] <= ship_max;
#pragma unroll
    for (int i = 0; i < I; ++i) {
      uint32_t r = alive[i] ? __ldg(rf + row[i]) : 0, l = alive[i] ? __ldg(ls + row[i]) : 0;
      key[i] = ((uint64_t)r << 32) | l;
      c.qty[i] = alive[i] ? __ldg(qty + row[i]) : 0;
      c.ext[i] = alive[i] ? __ldg(ext + row[i]) : 0;
      c.disc[i] = alive[i] ? __ldg(disc + row[i]) : 0;
      c.tax[i] = alive[i] ? __ldg(tax + row[i]) : 0;
    }
  }
  // Dense interface (k_gb_dense): 4 consecutive rows with 128-bit loads.  Guard: qty, ext < 2^26 and
  // 0 <= disc, tax < 2^7 make every state |v| < 2^41 and the products exact as 32x32->64 multiplies
  // (|ext*(100-disc)| < 2^33, |.. *(100+tax)| < 2^41); a group failing it takes the checked path.
  static constexpr int kDenseNst = 6;
  static constexpr int kDenseRows = 4;  // (3 CTAs/SM measured 5.0 vs 4.35 ms: register spills)
  template <int R>
  __device__ __forceinline__ void compute(const int32_t (&sd)[R], const uint32_t (&f)[R], const uint32_t (&s)[R],
                                          const long long (&q)[R], const long long (&e)[R], const long long (&d)[R],
                                          const long long (&x)[R], bool (&alive)[R], uint64_t (&key)[R],
                                          int64_t (&v)[R][kDenseNst], bool& fast) const {
    unsigned long long u = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      alive[i] = alive[i] && sd[i] <= ship_max;
      key[i] = ((uint64_t)f[i] << 32) | s[i];
      u |= (((unsigned long long)q[i] | (unsigned long long)e[i]) >> 26) |
           (((unsigned long long)d[i] | (unsigned long long)x[i]) >> 7);
    }
    fast = u == 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const long long dp = (long long)(int32_t)e[i] * (long long)(100 - (int32_t)d[i]);
      v[i][0] = q[i];
      v[i][1] = e[i];
      v[i][2] = dp;
      v[i][3] = dp * (long long)(100 + (int32_t)x[i]);
      v[i][4] = 1;
      v[i][5] = d[i];
    }
  }
  // 4 rows at row r0 from columns at (global or shared) base pointers; vector loads when `vec`
  template <int R, bool GLOBAL>
  __device__ __forceinline__ void load4(const int32_t* sp, const uint8_t* fp, const uint8_t* lp, const long long* qp,
                                        const long long* ep, const long long* dp, const long long* xp, int32_t (&sd)[R],
                                        uint32_t (&f)[R], uint32_t (&s)[R], long long (&q)[R], long long (&e)[R],
                                        long long (&d)[R], long long (&x)[R]) const {
    static_assert(R == 4, "4 rows");
    int4 a;
    uint32_t fr, lv;
    longlong2 vq[2], ve[2], vd[2], vx[2];
    if (GLOBAL) {
      a = __ldcs((const int4*)sp);
      fr = __ldcs((const unsigned int*)fp);
      lv = __ldcs((const unsigned int*)lp);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        vq[j] = __ldcs((const longlong2*)qp + j);
        ve[j] = __ldcs((const longlong2*)ep + j);
        vd[j] = __ldcs((const longlong2*)dp + j);
        vx[j] = __ldcs((const longlong2*)xp + j);
      }
    } else {
      a = *(const int4*)sp;
      fr = *(const unsigned int*)fp;
      lv = *(const unsigned int*)lp;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        vq[j] = ((const longlong2*)qp)[j];
        ve[j] = ((const longlong2*)ep)[j];
        vd[j] = ((const longlong2*)dp)[j];
        vx[j] = ((const longlong2*)xp)[j];
      }
    }
    sd[0] = a.x; sd[1] = a.y; sd[2] = a.z; sd[3] = a.w;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[i] = (fr >> (8 * i)) & 0xffu;
      s[i] = (lv >> (8 * i)) & 0xffu;
      q[i] = (i & 1) ? vq[i >> 1].y : vq[i >> 1].x;
      e[i] = (i & 1) ? ve[i >> 1].y : ve[i >> 1].x;
      d[i] = (i & 1) ? vd[i >> 1].y : vd[i >> 1].x;
      x[i] = (i & 1) ? vx[i >> 1].y : vx[i >> 1].x;
    }
  }
  template <int R>
  __device__ __forceinline__ void dense(int64_t r0, int64_t n, bool (&alive)[R], uint64_t (&key)[R],
                                        int64_t (&v)[R][kDenseNst], bool& fast) const {
    static_assert(R == 4, "Q1Prog::dense loads 4 rows");
    int32_t sd[4];
    uint32_t f[4], s[4];
    long long q[4], e[4], d[4], x[4];
    if (r0 + 4 <= n) {
      load4<4, true>(ship + r0, rf + r0, ls + r0, qty + r0, ext + r0, disc + r0, tax + r0, sd, f, s, q, e, d, x);
#pragma unroll
      for (int i = 0; i < 4; ++i) alive[i] = true;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        alive[i] = r0 + i < n;
        const int64_t r = alive[i] ? r0 + i : r0;
        sd[i] = alive[i] ? __ldg(ship + r) : 0;
        f[i] = alive[i] ? __ldg(rf + r) : 0;
        s[i] = alive[i] ? __ldg(ls + r) : 0;
        q[i] = alive[i] ? __ldg(qty + r) : 0;
        e[i] = alive[i] ? __ldg(ext + r) : 0;
        d[i] = alive[i] ? __ldg(disc + r) : 0;
        x[i] = alive[i] ? __ldg(tax + r) : 0;
      }
    }
    compute<4>(sd, f, s, q, e, d, x, alive, key, v, fast);
  }
  // Staged interface (k_gb_dense<P, true>): whole tiles of the 7 columns are copied into shared
  // memory by bulk asynchronous copies (cp.async.bulk, the TMA engine); rows are read from there.
  static constexpr int kBulkCols = 7;
  __host__ __device__ static constexpr int bulk_width(int c) { return c == 0 ? 4 : (c <= 2 ? 1 : 8); }
  __host__ __device__ const void* bulk_col(int c) const {
    switch (c) {
      case 0: return ship;
      case 1: return rf;
      case 2: return ls;
      case 3: return qty;
      case 4: return ext;
      case 5: return disc;
      default: return tax;
    }
  }
  template <int R>
  __device__ __forceinline__ void staged(const uint8_t* const (&b)[kBulkCols], int j, bool (&alive)[R],
                                         uint64_t (&key)[R], int64_t (&v)[R][kDenseNst], bool& fast) const {
    int32_t sd[4];
    uint32_t f[4], s[4];
    long long q[4], e[4], d[4], x[4];
    load4<4, false>((const int32_t*)b[0] + j, b[1] + j, b[2] + j, (const long long*)b[3] + j,
                    (const long long*)b[4] + j, (const long long*)b[5] + j, (const long long*)b[6] + j, sd, f, s, q,
                    e, d, x);
#pragma unroll
    for (int i = 0; i < 4; ++i) alive[i] = true;
    compute<4>(sd, f, s, q, e, d, x, alive, key, v, fast);
  }
  // Ring interface (K9r, ring.cuh): 1024-row tiles of the 7 columns (38.9 KB per stage), 3 stages,
  // 16 consumer warps taking 2 consecutive rows per lane.  Exact per-thread accumulators live in
  // lane-private shared memory cells indexed by the row's group, so the group choice is an address,
  // not a branch: the 6 (returnflag, linestatus) combinations {A,N,R} x {F,O}, 4 sums per group in
  // two 16-byte cells: {pk, sum(ext)} and {sum(dp), sum(charge)}, where
  //   pk = sum(qty) | sum(disc) << 24 | count << 39  (packed).
  // Fast-path guard per row: 0 <= qty < 2^13, 0 <= ext < 2^24, 0 <= disc, tax < 2^4.  Then dp =
  // ext*(100-disc) < 2^31 and charge = dp*(100+tax) < 2^38 are exact 32x32->64 products, and over
  // kRingFlush = 2048 rows per thread the packed fields (< 2^24, 2^15, 2^12) and the other sums
  // (< 2^35, 2^42, 2^49) cannot overflow; every 2048 rows a warp-collective flush adds them into a
  // per-CTA shared state (96-bit sums), merged into the global table once per CTA.  A row failing
  // the guard, or with another flag value, goes to a per-CTA list for the exact per-row path
  // (gb_dense_slow_row) after the stream; if that list overflows the host reruns K9d.
  static constexpr int kRingCols = 7;
  static constexpr int kRingTile = 1024;
  static constexpr int kRingStages = 3;
  static constexpr int kRingConsumers = 16;
  static constexpr int kRingThreads = kRingConsumers * 32;
  static constexpr int kRingLane = kRingTile / kRingThreads;
  static constexpr int kRingFlush = 2048;
  static constexpr size_t kRingExtraBytes = (size_t)6 * 2 * kRingThreads * sizeof(ulonglong2);  // 96 KB
  static_assert(kRingLane == 2, "ring_consume reads 2 rows per lane");
  __host__ __device__ static constexpr int ring_width(int c) { return bulk_width(c); }
  __host__ __device__ const void* ring_col(int c) const { return bulk_col(c); }
  struct RingAcc {
    int since;
  };
  static constexpr int kRingSlowCap = 2048;  // rows per CTA for the exact path (else the host reruns K9d)
  struct RingShared {
    unsigned long long lo[6][6];
    int hi[6][6];
    int nslow;
    int32_t slow[kRingSlowCap];
  };
  __device__ __forceinline__ static ulonglong2* ring_cell(uint8_t* xs, int slot, int ct) {
    return (ulonglong2*)xs + (slot * 2 * kRingThreads + ct);  // second cell at + kRingThreads
  }
  __device__ __forceinline__ void ring_init(RingAcc& acc) const { acc.since = 0; }
  __device__ __forceinline__ void ring_shared_init(RingShared& sh, uint8_t* xs, int tid, int nt) const {
    for (int j = tid; j < 36; j += nt) {
      sh.lo[j / 6][j % 6] = 0;
      sh.hi[j / 6][j % 6] = 0;
    }
    if (tid == 0) sh.nslow = 0;
    for (int j = tid; j < 6 * 2 * kRingThreads; j += nt) ((ulonglong2*)xs)[j] = make_ulonglong2(0, 0);
  }
  __device__ __forceinline__ void ring_row(int32_t sd, uint32_t f, uint32_t s, long long q, long long e, long long d,
                                           long long x, int64_t row, int ct, RingShared& sh, uint8_t* xs) const {
    const bool fN = f == 'N', fR = f == 'R', sO = s == 'O';
    const bool flags_ok = (f == 'A' || fN || fR) && (s == 'F' || sO);
    const unsigned long long g = ((unsigned long long)q >> 13) | ((unsigned long long)e >> 24) |
                                 ((unsigned long long)d >> 4) | ((unsigned long long)x >> 4);
    const bool alive = sd <= ship_max, fast = flags_ok && g == 0;
    if (alive && !fast) {  // exact path after the stream (no call in the hot loop)
      const int pos = atomicAdd(&sh.nslow, 1);
      if (pos < kRingSlowCap) sh.slow[pos] = (int32_t)row;
      else atomicExch(ovf_flag + 3, 1);
    }
    if (alive && fast) {
      const int slot = ((int)fN + 2 * (int)fR) * 2 + (int)sO;
      const uint32_t qq = (uint32_t)q, ee = (uint32_t)e, dd = (uint32_t)d, xx = (uint32_t)x;
      const uint32_t dp = ee * (100u - dd);  // < 2^31
      ulonglong2* c = ring_cell(xs, slot, ct);
      ulonglong2 a = c[0], b = c[kRingThreads];
      a.x += (unsigned long long)(qq | (dd << 24)) + (1ull << 39);
      a.y += ee;
      b.x += dp;
      b.y += (unsigned long long)dp * (100u + xx);
      c[0] = a;
      c[kRingThreads] = b;
    }
  }
  // warp-collective (every lane of the warp calls it at the same point)
  __device__ __forceinline__ void ring_flush(RingAcc& acc, int cw, int lane, RingShared& sh, uint8_t* xs) const {
    const int ct = cw * 32 + lane;
#pragma unroll 1
    for (int k = 0; k < 6; ++k) {
      ulonglong2* c = ring_cell(xs, k, ct);
      const ulonglong2 a = c[0], b = c[kRingThreads];
      unsigned long long v[6];
      v[0] = a.x & ((1ull << 24) - 1);          // sum(qty)
      v[5] = (a.x >> 24) & ((1ull << 15) - 1);  // sum(disc)
      v[4] = a.x >> 39;                         // count
      v[1] = a.y;
      v[2] = b.x;
      v[3] = b.y;
      if (!__any_sync(kFull, v[4] != 0)) continue;
      c[0] = make_ulonglong2(0, 0);
      c[kRingThreads] = make_ulonglong2(0, 0);
#pragma unroll
      for (int j = 0; j < 6; ++j)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_xor_sync(kFull, v[j], o);
      if (lane == 0) {
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          const unsigned long long old = atomicAdd(&sh.lo[k][j], v[j]);
          if (old + v[j] < old) atomicAdd(&sh.hi[k][j], 1);
        }
      }
    }
    acc.since = 0;
  }
  __device__ __forceinline__ void ring_consume(const uint8_t* const* b, int64_t row0, int cw, int lane,
                                               RingAcc& acc, RingShared& sh, uint8_t* xs) const {
    if (acc.since + kRingLane > kRingFlush) ring_flush(acc, cw, lane, sh, xs);
    acc.since += kRingLane;
    const int ct = cw * 32 + lane, j = ct * kRingLane;
    const int2 sd = *(const int2*)(b[0] + 4 * j);
    const uint32_t f = *(const uint16_t*)(b[1] + j), sv = *(const uint16_t*)(b[2] + j);
    const longlong2 q = *(const longlong2*)(b[3] + 8 * j), e = *(const longlong2*)(b[4] + 8 * j);
    const longlong2 d = *(const longlong2*)(b[5] + 8 * j), x = *(const longlong2*)(b[6] + 8 * j);
    ring_row(sd.x, f & 0xffu, sv & 0xffu, q.x, e.x, d.x, x.x, row0 + j, ct, sh, xs);
    ring_row(sd.y, f >> 8, sv >> 8, q.y, e.y, d.y, x.y, row0 + j + 1, ct, sh, xs);
  }
  __device__ __forceinline__ void ring_tail(int64_t r0, int64_t n, int cw, int lane, RingAcc& acc, RingShared& sh,
                                            uint8_t* xs) const {
    ring_flush(acc, cw, lane, sh, xs);  // <= kRingLane tail rows per lane follow
    const int ct = cw * 32 + lane;
    for (int64_t r = r0 + ct; r < n; r += kRingThreads)
      ring_row(__ldg(ship + r), __ldg(rf + r), __ldg(ls + r), __ldg(qty + r), __ldg(ext + r), __ldg(disc + r),
               __ldg(tax + r), r, ct, sh, xs);
  }
  __device__ __forceinline__ void ring_finish(RingShared& sh, int tid, int nt, const Layout& L, const Table& t) const {
    bool ovf = false;
    const int ns = min(sh.nslow, kRingSlowCap);
    for (int i = tid; i < ns; i += nt) gb_dense_slow_row(*this, t, L, sh.slow[i], ovf);
    if (ovf) atomicExch(ovf_flag, 1);
    if (tid >= 6) return;
    const int k = tid;
    if (sh.lo[k][4] == 0 && sh.hi[k][4] == 0) return;  // no row of this group in the CTA
    const uint64_t key = ((uint64_t)(k < 2 ? 'A' : (k < 4 ? 'N' : 'R')) << 32) | (uint64_t)((k & 1) ? 'O' : 'F');
    uint8_t* p = find_or_insert(t, L, key);
    if (!p) return;
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      if (L.kind[a] == ST_SUM)
        atomic_add_sum96((unsigned long long*)(p + L.off8[a]), (int*)(p + L.off4[a]), (int64_t)sh.lo[k][a], sh.hi[k][a]);
      else
        atomicAdd((unsigned long long*)(p + L.off8[a]), sh.lo[k][a]);
    }
  }
  template <int I>
  __device__ __forceinline__ void state(int a, const int32_t (&)[I], const bool (&)[I], const Cache<I>& c,
                                        int64_t (&v)[I], bool& ovf) const {
#pragma unroll
    for (int i = 0; i < I; ++i) {
      switch (a) {
        case 0: v[i] = c.qty[i]; break;
        case 1: v[i] = c.ext[i]; break;
        case 2: v[i] = mul_ck(c.ext[i], sub_ck(100, c.disc[i], ovf), ovf); break;
        case 3: v[i] = mul_ck(mul_ck(c.ext[i], sub_ck(100, c.disc[i], ovf), ovf), add_ck(c.tax[i], 100, ovf), ovf); break;
        case 4: v[i] = 1; break;
        default: v[i] = c.disc[i]; break;
      }
    }
  }
};

// Q6: keyless; where date in [lo, hi), disc in [dlo, dhi], qty < qlt (each column loaded only for
// rows still alive); states: 0 sum(ext*disc) 1 count
struct Q6Prog {
  const int32_t* ship;
  const long long *disc, *qty, *ext;
  int32_t date_lo, date_hi;
  int64_t disc_lo, disc_hi, qty_lt;
  int* ovf_flag;
  int lazy3;  // 1: discount first, quantity/price only where the discount qualifies (3 levels)
  static constexpr int kMaxNst = 2;
  static constexpr int kUnrollStates = 2;
  static constexpr bool kSortedOK = false;
  bool no_filter() const { return false; }
  template <int I>
  __device__ __forceinline__ void keys_only(const int32_t (&)[I], const bool (&)[I], uint64_t (&)[I]) const {}
  template <int I>
  struct Cache { int64_t ext[I], disc[I]; };
  __device__ __forceinline__ int kind(int a, const Layout&) const { return a == 1 ? ST_COUNT : ST_SUM; }
  template <int I>
  __device__ __forceinline__ void where_keys(const int32_t (&row)[I], bool (&alive)[I], uint64_t (&key)[I],
                                             Cache<I>& c) const {
    int32_t sd[I];
#pragma unroll
    for (int i = 0; i < I; ++i) sd[i] = alive[i] ? __ldg(ship + row[i]) : 0;
#pragma unroll
    for (int i = 0; i < I; ++i) alive[i] = alive[i] && sd[i] >= date_lo && sd[i] < date_hi;
#pragma unroll
    for (int i = 0; i < I; ++i) c.disc[i] = alive[i] ? __ldg(disc + row[i]) : 0;
#pragma unroll
    for (int i = 0; i < I; ++i) alive[i] = alive[i] && c.disc[i] >= disc_lo && c.disc[i] <= disc_hi;
    int64_t q[I];
#pragma unroll
    for (int i = 0; i < I; ++i) q[i] = alive[i] ? __ldg(qty + row[i]) : 0;
#pragma unroll
    for (int i = 0; i < I; ++i) {
      alive[i] = alive[i] && q[i] < qty_lt;
      c.ext[i] = alive[i] ? __ldg(ext + row[i]) : 0;
      key[i] = 0;
    }
  }
  template <int I>
  __device__ __forceinline__ void state(int a, const int32_t (&)[I], const bool (&)[I], const Cache<I>& c,
                                        int64_t (&v)[I], bool& ovf) const {
#pragma unroll
    for (int i = 0; i < I; ++i) v[i] = a == 0 ? mul_ck(c.ext[i], c.disc[i], ovf) : 1;
  }
  // Dense interface (k_gb_dense): shipdate for 8 rows first (2 x 128-bit); discount, quantity and
  // extendedprice are then loaded per row pair only where a shipdate qualifies (one dependent
  // level; ~15% of rows pass the date range).  Guard: ext < 2^26, 0 <= disc < 2^14 on qualifying
  // rows make ext*disc < 2^40 an exact 32x32->64 product.
  static constexpr int kDenseNst = 2;
  static constexpr int kDenseRows = 8;
  static constexpr int kDenseMinBlocks = 4;  // more rows in flight for the lazy (dependent) loads
  template <int R>
  __device__ __forceinline__ void dense(int64_t r0, int64_t n, bool (&alive)[R], uint64_t (&key)[R],
                                        int64_t (&v)[R][kDenseNst], bool& fast) const {
    static_assert(R == 8, "Q6Prog::dense loads 8 rows");
    int32_t sd[8];
    long long q[8], e[8], d[8];
    const bool full = r0 + 8 <= n;
    if (full) {
      const int4 a = __ldg((const int4*)(ship + r0)), b = __ldg((const int4*)(ship + r0 + 4));
      sd[0] = a.x; sd[1] = a.y; sd[2] = a.z; sd[3] = a.w;
      sd[4] = b.x; sd[5] = b.y; sd[6] = b.z; sd[7] = b.w;
#pragma unroll
      for (int i = 0; i < 8; ++i) alive[i] = sd[i] >= date_lo && sd[i] < date_hi;
      if (lazy3) {
        // discount pairs where a shipdate qualifies (~28% of pairs), then quantity / price pairs
        // only where date and discount qualify (~8%): fewer sectors than loading all three
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const bool need = alive[2 * j] || alive[2 * j + 1];
          const longlong2 dd = need ? __ldg((const longlong2*)(disc + r0) + j) : make_longlong2(0, 0);
          d[2 * j] = dd.x; d[2 * j + 1] = dd.y;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) alive[i] = alive[i] && d[i] >= disc_lo && d[i] <= disc_hi;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const bool need = alive[2 * j] || alive[2 * j + 1];
          const longlong2 z = make_longlong2(0, 0);
          const longlong2 qq = need ? __ldg((const longlong2*)(qty + r0) + j) : z;
          const longlong2 ee = need ? __ldg((const longlong2*)(ext + r0) + j) : z;
          q[2 * j] = qq.x; q[2 * j + 1] = qq.y;
          e[2 * j] = ee.x; e[2 * j + 1] = ee.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const bool need = alive[2 * j] || alive[2 * j + 1];
          const longlong2 z = make_longlong2(0, 0);
          const longlong2 dd = need ? __ldg((const longlong2*)(disc + r0) + j) : z;
          const longlong2 qq = need ? __ldg((const longlong2*)(qty + r0) + j) : z;
          const longlong2 ee = need ? __ldg((const longlong2*)(ext + r0) + j) : z;
          d[2 * j] = dd.x; d[2 * j + 1] = dd.y;
          q[2 * j] = qq.x; q[2 * j + 1] = qq.y;
          e[2 * j] = ee.x; e[2 * j + 1] = ee.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const bool in = r0 + i < n;
        const int64_t r = in ? r0 + i : r0;
        sd[i] = in ? __ldg(ship + r) : 0;
        alive[i] = in && sd[i] >= date_lo && sd[i] < date_hi;
        d[i] = alive[i] ? __ldg(disc + r) : 0;
        q[i] = alive[i] ? __ldg(qty + r) : 0;
        e[i] = alive[i] ? __ldg(ext + r) : 0;
      }
    }
    unsigned long long u = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      alive[i] = alive[i] && d[i] >= disc_lo && d[i] <= disc_hi && q[i] < qty_lt;
      key[i] = 0;
      u |= alive[i] ? ((unsigned long long)e[i] >> 26) | ((unsigned long long)d[i] >> 14) : 0ull;
    }
    fast = u == 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i][0] = (long long)(int32_t)e[i] * (long long)(int32_t)d[i];
      v[i][1] = 1;
    }
  }
};

// Q18 subquery: group lineitem by l_orderkey; state 0 sum(l_quantity)
template <typename KT>
struct Q18Prog {
  const KT* okey;
  const long long* qty;
  int* ovf_flag;
  static constexpr int kMaxNst = 1;
  static constexpr int kUnrollStates = 1;
  static constexpr bool kSortedOK = true;
  bool no_filter() const { return true; }
  template <int I>
  __device__ __forceinline__ void keys_only(const int32_t (&row)[I], const bool (&valid)[I], uint64_t (&key)[I]) const {
#pragma unroll
    for (int i = 0; i < I; ++i) key[i] = valid[i] ? (uint64_t)(int64_t)__ldg(okey + row[i]) : 0;
  }
  template <int I>
  struct Cache { int64_t q[I]; };
  __device__ __forceinline__ int kind(int, const Layout&) const { return ST_SUM; }
  template <int I>
  __device__ __forceinline__ void where_keys(const int32_t (&row)[I], bool (&alive)[I], uint64_t (&key)[I],
                                             Cache<I>& c) const {
#pragma unroll
    for (int i = 0; i < I; ++i) {
      key[i] = alive[i] ? (uint64_t)(int64_t)__ldg(okey + row[i]) : 0;
      c.q[i] = alive[i] ? __ldg(qty + row[i]) : 0;
    }
  }
  template <int I>
  __device__ __forceinline__ void state(int, const int32_t (&)[I], const bool (&)[I], const Cache<I>& c,
                                        int64_t (&v)[I], bool&) const {
#pragma unroll
    for (int i = 0; i < I; ++i) v[i] = c.q[i];
  }
  // K10l (k_runs_lean): 32-bit keys; 8 rows per thread with 128-bit streaming loads
  static constexpr bool kLeanRuns = sizeof(KT) == 4;
  __device__ __forceinline__ void lean_load(int64_t r0, int64_t n, int32_t (&k)[8], long long (&v)[8]) const {
    if (r0 + 8 <= n) {
      const int4 a = __ldcs((const int4*)(okey + r0)), b = __ldcs((const int4*)(okey + r0) + 1);
      k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w; k[4] = b.x; k[5] = b.y; k[6] = b.z; k[7] = b.w;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const longlong2 q = __ldcs((const longlong2*)(qty + r0) + j);
        v[2 * j] = q.x;
        v[2 * j + 1] = q.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const bool in = r0 + i < n;
        k[i] = in ? (int32_t)__ldg(okey + r0 + i) : 0;
        v[i] = in ? __ldg(qty + r0 + i) : 0;
      }
    }
  }
  __device__ __forceinline__ int32_t lean_key(int64_t r) const { return (int32_t)__ldg(okey + r); }
  __device__ __forceinline__ long long lean_val(int64_t r) const { return __ldg(qty + r); }
  // the key / value columns themselves (K10l's cp.async double buffer copies whole 8-row chunks)
  __device__ __forceinline__ const int32_t* lean_kp() const { return (const int32_t*)okey; }
  __device__ __forceinline__ const long long* lean_vp() const { return qty; }
  // Dense rows for k_runs_own: R consecutive rows (r0 % R == 0) with 128-bit streaming loads.
  static constexpr bool kDenseRuns = true;
  template <int R>
  __device__ __forceinline__ void runs_dense(int64_t r0, int64_t n, uint64_t (&key)[R], int64_t (&v)[R]) const {
    static_assert(R % 4 == 0, "groups of 4 rows");
    if (r0 + R <= n) {
      if constexpr (sizeof(KT) == 4) {
#pragma unroll
        for (int j = 0; j < R / 4; ++j) {
          const int4 k = __ldcs((const int4*)(okey + r0) + j);
          key[4 * j] = (uint64_t)(int64_t)k.x; key[4 * j + 1] = (uint64_t)(int64_t)k.y;
          key[4 * j + 2] = (uint64_t)(int64_t)k.z; key[4 * j + 3] = (uint64_t)(int64_t)k.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < R / 2; ++j) {
          const longlong2 k = __ldcs((const longlong2*)(okey + r0) + j);
          key[2 * j] = (uint64_t)k.x; key[2 * j + 1] = (uint64_t)k.y;
        }
      }
#pragma unroll
      for (int j = 0; j < R / 2; ++j) {
        const longlong2 q = __ldcs((const longlong2*)(qty + r0) + j);
        v[2 * j] = q.x; v[2 * j + 1] = q.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const bool in = r0 + i < n;
        key[i] = in ? (uint64_t)(int64_t)__ldg(okey + r0 + i) : 0;
        v[i] = in ? __ldg(qty + r0 + i) : 0;
      }
    }
  }
};

// Q9: key (nationkey, year(o_orderdate)); state 0 sum(ext*(100-disc) - supplycost*qty)
struct Q9Prog {
  const int32_t* nation;
  const long long *cost, *qty, *ext, *disc;
  const int32_t* odate;
  int* ovf_flag;
  static constexpr int kMaxNst = 1;
  static constexpr int kUnrollStates = 1;
  static constexpr bool kSortedOK = false;
  bool no_filter() const { return true; }
  template <int I>
  __device__ __forceinline__ void keys_only(const int32_t (&)[I], const bool (&)[I], uint64_t (&)[I]) const {}
  template <int I>
  struct Cache {};
  __device__ __forceinline__ int kind(int, const Layout&) const { return ST_SUM; }
  template <int I>
  __device__ __forceinline__ void where_keys(const int32_t (&row)[I], bool (&alive)[I], uint64_t (&key)[I],
                                             Cache<I>&) const {
#pragma unroll
    for (int i = 0; i < I; ++i) {
      uint32_t nk = alive[i] ? (uint32_t)__ldg(nation + row[i]) : 0u;
      int32_t d = alive[i] ? __ldg(odate + row[i]) : 0;
      key[i] = ((uint64_t)nk << 32) | (uint32_t)civil_year(d);
    }
  }
  template <int I>
  __device__ __forceinline__ void state(int, const int32_t (&row)[I], const bool (&alive)[I], const Cache<I>&,
                                        int64_t (&v)[I], bool& ovf) const {
#pragma unroll
    for (int i = 0; i < I; ++i) {
      int64_t e = alive[i] ? __ldg(ext + row[i]) : 0, d = alive[i] ? __ldg(disc + row[i]) : 0;
      int64_t c = alive[i] ? __ldg(cost + row[i]) : 0, q = alive[i] ? __ldg(qty + row[i]) : 0;
      v[i] = sub_ck(mul_ck(e, sub_ck(100, d, ovf), ovf), mul_ck(c, q, ovf), ovf);
    }
  }
};

// Unique-key lookup in an sx_hash_build table (the layouts of join.cu): the build row id, or -1.
template <int KB>
__device__ __forceinline__ int32_t ht_find(const void* slots, uint32_t mask, uint64_t key) {
  if (KB == 4) {
    const unsigned long long* s = (const unsigned long long*)slots;
    uint32_t h = hash32((uint32_t)key) & mask;
    for (;;) {
      const unsigned long long v = __ldg(s + h);
      if ((uint32_t)(v >> 32) == 0xffffffffu) return -1;
      if ((uint32_t)v == (uint32_t)key) return (int32_t)(v >> 32);
      h = (h + 1) & mask;
    }
  } else {
    const longlong2* s = (const longlong2*)slots;
    uint32_t h = (uint32_t)hash64(key) & mask;
    for (;;) {
      const longlong2 v = __ldg(s + h);
      const uint32_t rw = (uint32_t)(unsigned long long)v.y;
      if (rw == 0xffffffffu) return -1;
      if ((uint64_t)v.x == key) return (int32_t)rw;
      h = (h + 1) & mask;
    }
  }
}

// Q9 as one pass over lineitem (the plan's probe chain fused into its group-by, SURVEY §8(a) "the
// executor may fuse adjacent steps"): green-part membership from the part build's exact key-range
// bitmap; partsupp (partkey, suppkey) -> ps_supplycost, supplier suppkey -> s_nationkey and orders
// orderkey -> o_orderdate through unique-key tables (PK sides); key (nationkey, year(o_orderdate));
// state 0 sum(ext*(100-disc) - supplycost*qty).  Rows whose lookups miss drop out (inner joins).
// Several rows per thread (kSharedItems) so their independent lookups overlap.
template <typename V>
__device__ __forceinline__ bool direct_get(const uint32_t* __restrict__ bm, long long mn, unsigned long long nbits,
                                           const V* __restrict__ val, long long key, int64_t& out) {
  const unsigned long long off = (unsigned long long)(key - mn);
  if (!bm || off >= nbits || !((__ldg(bm + (off >> 5)) >> (off & 31)) & 1u)) return false;
  out = __ldg(val + off);
  return true;
}

// Q9 needs only year(o_orderdate): the orders lookup array holds the year as one byte,
// year - kYear0 in 0..127, with 0x80 = "no order" (the memset / 16-byte sentinel fill value); a
// date whose year falls outside [kYear0, kYear0 + 127] makes the fill report it (the plan then
// takes its operator-at-a-time fallback).  (int16 days before: twice the fill writes, and a
// warp's sorted lookups touched twice the lines.)
constexpr uint8_t kNoYear = 0x80;
constexpr int32_t kYear0 = 1900;
// year(days since 1970-01-01) - kYear0: 1901..2099 keep every fourth year a leap year, so there
// year = 1901 + (4d + 3) / 1461 with d = days since 1901-01-01 (checked against the calendar for
// every day of the range); civil_year's ~8 divisions only outside it.  (Computing civil_year for
// each of the 1.5e8 orders made the fill 0.74 instead of 0.54 ms.)
__device__ __forceinline__ int32_t year_byte(int32_t days) {
  const int32_t d = days + 25202;
  if ((uint32_t)d < 72684u) return 1901 + (4 * d + 3) / 1461 - kYear0;
  return civil_year(days) - kYear0;
}

// [min, max] of a key column (d_mm preset to {LLONG_MAX, LLONG_MIN})
template <typename KT>
__global__ void k_key_range(const KT* __restrict__ keys, int64_t n, long long* d_mm) {
  long long mn = LLONG_MAX, mx = LLONG_MIN;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const long long k = (long long)__ldcs(keys + r);
    mn = min(mn, k);
    mx = max(mx, k);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0 && mn <= mx) {
    atomicMin(d_mm, mn);
    atomicMax(d_mm + 1, mx);
  }
}

// val[key - min] = pay[r] for the rows whose key is in the bitmap (a PK side: one row per key;
// bm == nullptr: every key of the column is in range, the bitmap was built from this column).
// A narrower value type V sets *bad for a value it cannot hold (the plan then falls back).
template <typename KT, typename V>
__global__ void k_direct_fill(const KT* __restrict__ keys, const int32_t* __restrict__ pay, int64_t n,
                              const uint32_t* __restrict__ bm, long long mn, unsigned long long nbits,
                              V* __restrict__ val, long long* bad) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long off = (unsigned long long)((long long)__ldg(keys + r) - mn);
    if (off < nbits && (!bm || ((__ldg(bm + (off >> 5)) >> (off & 31)) & 1u))) {
      int32_t x = __ldg(pay + r);
      if constexpr (sizeof(V) == 1) {  // the Q9 year byte of a date
        x = year_byte(x);
        if ((unsigned)x >= (unsigned)kNoYear) *bad = 1;
      } else if (sizeof(V) < 4 && (int32_t)(V)x != x) {
        *bad = 1;
      }
      val[off] = (V)x;
    }
  }
}

// Orders stored in strictly increasing orderkey order (checked here; TPC-H's orders are): ONE pass
// writes the whole year-byte array over [min, max].  A warp takes 256 consecutive orders and owns
// the array entries from their first key up to the next warp's first key: it fills them with the
// "no order" sentinel using 16-byte stores, then (after __syncwarp) writes each order's date at its
// key.  This replaces a sentinel memset followed by scattered writes into the (then
// DRAM-resident) array — read-modify-write of every sector — and a per-thread gap-filling
// version (stores 32 sectors apart per warp instruction: 4.2 ms).  bad[0]: a year outside the
// byte's range (plan falls back); bad[1]: keys not strictly increasing (host reruns the scatter fill).
template <typename KT>
__global__ void k_date_fill_sorted(const KT* __restrict__ keys, const int32_t* __restrict__ dates, int64_t n,
                                   long long mn, unsigned long long nbits, uint8_t* __restrict__ val, long long* bad) {
  constexpr int K = 8, W = 32 * K;
  const int lane = threadIdx.x & 31;
  bool wide = false, unsorted = false;
  const long long nb = (long long)nbits;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c * W < n; c += warps) {
    const int64_t o0 = c * W, o1 = min(n, o0 + W);
    const long long p0 = o0 > 0 ? (long long)__ldg(keys + o0) - mn : 0;
    const long long p1 = o1 < n ? (long long)__ldg(keys + o1) - mn : nb;
    if (p0 < 0 || p1 > nb || p1 < p0) {
      unsorted = true;
      continue;
    }
    // 1. sentinel over [p0, p1): scalar head and tail, 16 entries per 16-byte store between
    const long long a = min(p1, (p0 + 15) & ~15ll), b = max(a, p1 & ~15ll);
    if (p0 + lane < a) val[p0 + lane] = kNoYear;
    if (b + lane < p1) val[b + lane] = kNoYear;
    const uint4 sent = make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
    for (long long u = a / 16 + lane; u < b / 16; u += 32) __stcs((uint4*)val + u, sent);
    __syncwarp();
    // 2. the dates at the keys (and the order check); every key and date load of the chunk is
    //    issued together, the previous key comes from the neighbouring lane
    long long kk[K];
    int32_t dd[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t o = o0 + k * 32 + lane;
      kk[k] = o < o1 ? (long long)__ldg(keys + o) : LLONG_MAX;
      dd[k] = o < o1 ? __ldg(dates + o) : 0;
    }
    const long long before = o0 > 0 ? (long long)__ldg(keys + o0 - 1) : mn - 1;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t o = o0 + k * 32 + lane;
      long long prev = __shfl_up_sync(kFull, kk[k], 1);
      const long long last_prev = __shfl_sync(kFull, k > 0 ? kk[k > 0 ? k - 1 : 0] : before, 31);
      if (lane == 0) prev = k == 0 ? before : last_prev;
      if (o >= o1) continue;
      const long long key = kk[k];
      const long long off = key - mn;
      if (key <= prev || off < p0 || off >= p1) {
        unsorted = true;
        continue;
      }
      const int32_t y = year_byte(dd[k]);
      wide |= (unsigned)y >= (unsigned)kNoYear;
      val[off] = (uint8_t)y;
    }
  }
  if (wide) atomicExch((unsigned long long*)bad, 1ull);
  if (unsorted) atomicExch((unsigned long long*)bad + 1, 1ull);
}

template <typename KT, int OKB>
struct Q9FusedProg {
  const int32_t *partkey, *suppkey;
  const KT* orderkey;
  const long long *qty, *ext, *disc;
  const uint32_t* pbm;
  long long pbm_min;
  unsigned long long pbm_bits;
  const ulonglong2* ps;   // (partkey, suppkey) -> ps_supplycost
  uint32_t ps_mask;
  int ps_bits;
  // suppkey -> s_nationkey and orderkey -> o_orderdate: direct-address arrays over each key range,
  // valid where the build's exact bitmap has the key (entries elsewhere are never read)
  const uint32_t* sup_bm;
  long long sup_min;
  unsigned long long sup_n;
  const int32_t* sup_val;
  const uint32_t* ord_bm;
  long long ord_min;
  unsigned long long ord_n;
  const uint8_t* ord_val;  // year(o_orderdate) - kYear0 (kNoYear: no order; the fill checks the range)
  int* ovf_flag;
  static constexpr int kMaxNst = 1;
  static constexpr int kUnrollStates = 1;
  static constexpr bool kSortedOK = false;
  static constexpr int kSharedItems = 4;
  // orderkey -> o_orderdate: bitmap-guarded (ord_bm) or, without a bitmap, the sentinel-initialised
  // array itself tells which keys exist
  __device__ __forceinline__ bool ord_get(long long key, int64_t& out) const {
    if (ord_bm) return direct_get(ord_bm, ord_min, ord_n, ord_val, key, out);
    const unsigned long long off = (unsigned long long)(key - ord_min);
    if (off >= ord_n) return false;
    const uint8_t v = __ldg(ord_val + off);
    if (v == kNoYear) return false;
    out = v;
    return true;
  }
  bool no_filter() const { return false; }
  template <int I>
  __device__ __forceinline__ void keys_only(const int32_t (&)[I], const bool (&)[I], uint64_t (&)[I]) const {}
  template <int I>
  struct Cache { int64_t cost[I], qty[I], ext[I], disc[I]; };
  __device__ __forceinline__ int kind(int, const Layout&) const { return ST_SUM; }
  template <int I>
  __device__ __forceinline__ void where_keys(const int32_t (&row)[I], bool (&alive)[I], uint64_t (&key)[I],
                                             Cache<I>& c) const {
    int32_t pk[I], sk[I];
    KT ok[I];
    if (pbm) {
      // dense scan of every lineitem row: all six columns are loaded together (one latency level,
      // streaming; ~5% of rows survive, too sparse for partial sector reads to save traffic), then
      // the green-part membership test
#pragma unroll
      for (int i = 0; i < I; ++i) {
        pk[i] = alive[i] ? __ldcs(partkey + row[i]) : 0;
        sk[i] = alive[i] ? __ldcs(suppkey + row[i]) : 0;
        ok[i] = alive[i] ? __ldcs(orderkey + row[i]) : (KT)0;
        c.qty[i] = alive[i] ? __ldcs(qty + row[i]) : 0;
        c.ext[i] = alive[i] ? __ldcs(ext + row[i]) : 0;
        c.disc[i] = alive[i] ? __ldcs(disc + row[i]) : 0;
      }
#pragma unroll
      for (int i = 0; i < I; ++i) {
        const unsigned long long off = (unsigned long long)((long long)pk[i] - pbm_min);
        const bool in = alive[i] && off < pbm_bits;
        const uint32_t w = in ? __ldg(pbm + (off >> 5)) : 0u;
        alive[i] = in && ((w >> (off & 31)) & 1u);
      }
    } else {  // rows pre-selected by the semi-join (gathers)
#pragma unroll
      for (int i = 0; i < I; ++i) pk[i] = alive[i] ? __ldg(partkey + row[i]) : 0;
#pragma unroll
      for (int i = 0; i < I; ++i) {
        sk[i] = alive[i] ? __ldg(suppkey + row[i]) : 0;
        ok[i] = alive[i] ? __ldg(orderkey + row[i]) : (KT)0;
        c.qty[i] = alive[i] ? __ldg(qty + row[i]) : 0;
        c.ext[i] = alive[i] ? __ldg(ext + row[i]) : 0;
        c.disc[i] = alive[i] ? __ldg(disc + row[i]) : 0;
      }
    }
    int64_t nk[I], d[I];
#pragma unroll
    for (int i = 0; i < I; ++i) {
      bool f = alive[i];
      c.cost[i] = 0;
      nk[i] = 0;
      d[i] = 0;
      if (f) f = direct_get(sup_bm, sup_min, sup_n, sup_val, (long long)sk[i], nk[i]);
      if (f) f = ord_get((long long)ok[i], d[i]);
      if (f) f = pt_find<8>(ps, ps_mask, ps_bits, ((uint64_t)(uint32_t)pk[i] << 32) | (uint32_t)sk[i], c.cost[i]);
      alive[i] = f;
      key[i] = ((uint64_t)(uint32_t)nk[i] << 32) | (uint32_t)((int32_t)d[i] + kYear0);
    }
  }
  template <int I>
  __device__ __forceinline__ void state(int, const int32_t (&)[I], const bool (&)[I], const Cache<I>& c,
                                        int64_t (&v)[I], bool& ovf) const {
#pragma unroll
    for (int i = 0; i < I; ++i)
      v[i] = sub_ck(mul_ck(c.ext[i], sub_ck(100, c.disc[i], ovf), ovf), mul_ck(c.cost[i], c.qty[i], ovf), ovf);
  }
  // Dense interface (K10d): 8 consecutive lineitem rows, all six columns with 128-bit streaming
  // loads (every sector is read once: cheaper than gathering 5.4% of the rows' sectors), the
  // green-part bitmap, then the three lookups for the green rows only.
  static constexpr int kDenseNst = 1;
  static constexpr int kDenseRows = 8;
  static constexpr bool kDenseShared = true;
  int wscan = 0;  // 1: K10w (warp-compacted scan) instead of K10d for the full lineitem scan
  bool dense_ok() const { return pbm != nullptr && !wscan; }  // K10d only for the dense lineitem scan
  // K10w interface: the streaming green-part test of 8 rows (returns the passing mask and the
  // partkeys), then the rest of the program for U compacted rows with every load of one level
  // issued together: five column gathers, then the supplier and orders direct arrays (bitmap word
  // and value read speculatively, both inside the key range) and the partsupp table's first slot.
  static constexpr int kWChunks = 2;
  static constexpr int kWRows = 2;  // (3 rows per lane: 4.58 vs 4.25 ms for Q9 at SF100)
  // K10wr interface (gb_host.cuh): the six lineitem columns through the tile ring
  static constexpr bool kWRing = true;
  using KeyT = KT;
  struct RingCols {
    const void* col[6];  // partkey, suppkey, orderkey, quantity, extendedprice, discount
    static constexpr int kRingCols = 6, kRingTile = 1024, kRingStages = 3, kRingConsumers = 16;
    __host__ __device__ static constexpr int ring_width(int c) { return c == 2 ? (int)sizeof(KT) : (c < 2 ? 4 : 8); }
    __host__ __device__ const void* ring_col(int c) const { return col[c]; }
  };
  RingCols ring_cols() const { return RingCols{{partkey, suppkey, orderkey, qty, ext, disc}}; }
  __device__ __forceinline__ bool wring_green(int32_t pk) const {
    const unsigned long long off = (unsigned long long)((long long)pk - pbm_min);
    return off < pbm_bits && ((__ldg(pbm + (off >> 5)) >> (off & 31)) & 1u);
  }
  bool wscan_ok() const { return pbm != nullptr && wscan; }
  __device__ __forceinline__ uint32_t wscan_select(int64_t r0, int64_t n, int32_t (&pk)[8]) const {
    dense_load32<8>(partkey, r0, n, r0 + 8 <= n, pk);
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const unsigned long long off = (unsigned long long)((long long)pk[i] - pbm_min);
      const bool in = r0 + i < n && off < pbm_bits;
      const uint32_t w = in ? __ldg(pbm + (off >> 5)) : 0u;
      m |= (in && ((w >> (off & 31)) & 1u)) ? (1u << i) : 0u;
    }
    return m;
  }
  template <int U>
  __device__ __forceinline__ void wscan_rows(const int32_t (&row)[U], const int32_t (&pk)[U], bool (&alive)[U],
                                             uint64_t (&key)[U], int64_t (&v)[U], bool& ovf) const {
    int32_t sk[U];
    KT ok[U];
    int64_t q[U], e[U], d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      sk[u] = alive[u] ? __ldg(suppkey + row[u]) : 0;
      ok[u] = alive[u] ? __ldg(orderkey + row[u]) : (KT)0;
      q[u] = alive[u] ? __ldg(qty + row[u]) : 0;
      e[u] = alive[u] ? __ldg(ext + row[u]) : 0;
      d[u] = alive[u] ? __ldg(disc + row[u]) : 0;
    }
    lookups<U>(pk, sk, ok, q, e, d, alive, key, v, ovf);
  }
  // the three lookups (supplier nation, order date, partsupp cost) and the profit of U green rows,
  // every load of one level issued together
  template <int U>
  __device__ __forceinline__ void lookups(const int32_t (&pk)[U], const int32_t (&sk)[U], const KT (&ok)[U],
                                          const int64_t (&q)[U], const int64_t (&e)[U], const int64_t (&d)[U],
                                          bool (&alive)[U], uint64_t (&key)[U], int64_t (&v)[U], bool& ovf) const {
    uint32_t sw[U], ow[U];
    int32_t sv[U], ov[U];
    ulonglong2 p0[U];
    uint32_t h[U];
    const ulonglong2* reg[U];
    uint64_t pkey[U];
    unsigned long long soff[U], ooff[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      soff[u] = (unsigned long long)((long long)sk[u] - sup_min);
      ooff[u] = (unsigned long long)((long long)ok[u] - ord_min);
      const bool si = alive[u] && sup_bm && soff[u] < sup_n, oi = alive[u] && ooff[u] < ord_n;
      sw[u] = si ? __ldg(sup_bm + (soff[u] >> 5)) : 0u;
      sv[u] = si ? __ldg(sup_val + soff[u]) : 0;
      ow[u] = (oi && ord_bm) ? __ldg(ord_bm + (ooff[u] >> 5)) : 0u;
      ov[u] = oi ? (int32_t)__ldg(ord_val + ooff[u]) : (int32_t)kNoYear;
      pkey[u] = ((uint64_t)(uint32_t)pk[u] << 32) | (uint32_t)sk[u];
      reg[u] = ps + pt_region_base(pkey[u], ps_bits, ps_mask);
      h[u] = (uint32_t)hash64(pkey[u]) & ps_mask;
      p0[u] = alive[u] ? __ldg(reg[u] + h[u]) : make_ulonglong2(~0ull, 0ull);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool of = ord_bm ? ((ow[u] >> (ooff[u] & 31)) & 1u) != 0 : ov[u] != (int32_t)kNoYear;
      bool f = alive[u] && ((sw[u] >> (soff[u] & 31)) & 1u) && of;
      int64_t cost = 0;
      if (f) {
        ulonglong2 s = p0[u];
        uint32_t hh = h[u];
        for (;;) {
          if (s.x == ~0ull) { f = false; break; }
          if (s.x == pkey[u]) { cost = (int64_t)s.y; break; }
          hh = (hh + 1) & ps_mask;
          s = __ldg(reg[u] + hh);
        }
      }
      alive[u] = f;
      key[u] = ((uint64_t)(uint32_t)sv[u] << 32) | (uint32_t)(ov[u] + kYear0);
      v[u] = f ? sub_ck(mul_ck(e[u], sub_ck(100, d[u], ovf), ovf), mul_ck(cost, q[u], ovf), ovf) : 0;
    }
  }
  template <int R>
  __device__ __forceinline__ void dense(int64_t r0, int64_t n, bool (&alive)[R], uint64_t (&key)[R],
                                        int64_t (&v)[R][kDenseNst], bool& fast) const {
    static_assert(R == 8, "8 rows");
    int64_t pk[R], sk[R], ok[R], q[R], e[R], d[R];
    const bool full = r0 + R <= n;
    dense_load<R>(DCol{partkey, SX_I32, 0}, r0, n, full, pk);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const unsigned long long off = (unsigned long long)(pk[i] - pbm_min);
      const bool in = r0 + i < n && off < pbm_bits;
      const uint32_t w = in ? __ldg(pbm + (off >> 5)) : 0u;
      alive[i] = in && ((w >> (off & 31)) & 1u);
    }
    dense_load<R>(DCol{suppkey, SX_I32, 0}, r0, n, full, sk);
    dense_load<R>(DCol{orderkey, sizeof(KT) == 4 ? SX_I32 : SX_I64, 0}, r0, n, full, ok);
    dense_load<R>(DCol{qty, SX_I64, 0}, r0, n, full, q);
    dense_load<R>(DCol{ext, SX_I64, 0}, r0, n, full, e);
    dense_load<R>(DCol{disc, SX_I64, 0}, r0, n, full, d);
    bool ovf = false;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      bool f = alive[i];
      int64_t cost = 0, nk = 0, dt = 0;
      if (f) f = direct_get(sup_bm, sup_min, sup_n, sup_val, sk[i], nk);
      if (f) f = ord_get((long long)ok[i], dt);
      if (f) f = pt_find<8>(ps, ps_mask, ps_bits, ((uint64_t)(uint32_t)pk[i] << 32) | (uint32_t)sk[i], cost);
      alive[i] = f;
      key[i] = ((uint64_t)(uint32_t)nk << 32) | (uint32_t)((int32_t)dt + kYear0);
      v[i][0] = f ? sub_ck(mul_ck(e[i], sub_ck(100, d[i], ovf), ovf), mul_ck(cost, q[i], ovf), ovf) : 0;
    }
    fast = !ovf;
  }
};

// Column width checks for the compiled plans (other layouts take the interpreted operator path).
bool w1(const sx_col& c) { return c.type == SX_U8 && !c.validity; }
bool w4(const sx_col& c) { return (c.type == SX_I32 || c.type == SX_DATE32) && !c.validity; }
bool w8(const sx_col& c) { return (c.type == SX_I64 || c.type == SX_DEC64) && !c.validity; }
sx_status to_dcols_check(sx_ctx* ctx, const sx_col* cols, int n) {
  DCol d[SX_MAX_COLS];
  return to_dcols(ctx, cols, n, d);
}

// The compiled program must see exactly the states gb_plan() derived from the aggregate list.
sx_status check_states(sx_ctx* ctx, const GbPlan& P, std::initializer_list<int> kinds) {
  int a = 0;
  for (int k : kinds) {
    if (a >= P.L.nst || P.L.kind[a] != k) return set_err(ctx, SX_EINVAL, "compiled plan/state layout mismatch");
    ++a;
  }
  if (a != P.L.nst) return set_err(ctx, SX_EINVAL, "compiled plan/state count mismatch");
  return SX_OK;
}

// Owns intermediate device buffers and hash tables of one query.
struct Bag {
  sx_ctx* ctx;
  std::vector<void*> bufs;
  std::vector<sx_ht*> hts;
  explicit Bag(sx_ctx* c) : ctx(c) {}
  ~Bag() {
    for (void* p : bufs) sx_free(ctx, p);
    for (sx_ht* h : hts) sx_ht_destroy(ctx, h);
  }
  void keep(const sx_sel& s) { if (s.idx) bufs.push_back(s.idx); }
  void keep(const sx_col& c) { if (c.data) bufs.push_back((void*)c.data); }
  void keep(const sx_col* c, int n) { for (int i = 0; i < n; ++i) keep(c[i]); }
  void keep(sx_ht* h) { if (h) hts.push_back(h); }
};

sx_factor F(int col, int64_t mul = 1, int64_t add = 0) { return sx_factor{col, 0, mul, add}; }

sx_expr E1(int64_t coef, std::initializer_list<sx_factor> fs) {
  sx_expr e;
  std::memset(&e, 0, sizeof e);
  e.nterms = 1;
  e.t[0].coef = coef;
  e.t[0].nf = (int32_t)fs.size();
  int i = 0;
  for (auto& f : fs) e.t[0].f[i++] = f;
  return e;
}

sx_agg A(int op, sx_expr e, int scale = 0) { return sx_agg{op, scale, e}; }
sx_agg Count() { sx_agg a; std::memset(&a, 0, sizeof a); a.op = SX_COUNT; return a; }

sx_pred P(int col, int op, int64_t lo, int64_t hi = 0) { return sx_pred{col, op, lo, hi, nullptr, 0, 0}; }

// Copy a device column to host (caller syncs).
sx_status d2h(sx_ctx* ctx, const sx_col& c, std::vector<uint8_t>& out) {
  size_t bytes = (size_t)c.len * type_width(c.type);
  out.resize(bytes + 16);
  if (bytes) SX_CUDA(cudaMemcpyAsync(out.data(), c.data, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return SX_OK;
}

template <class T>
T at(const std::vector<uint8_t>& v, int64_t i) {
  T x;
  std::memcpy(&x, v.data() + i * sizeof(T), sizeof(T));
  return x;
}

int64_t key_at(const std::vector<uint8_t>& v, int type, int64_t i) {
  switch (type) {
    case SX_U8: return v[i];
    case SX_I32: case SX_DATE32: return at<int32_t>(v, i);
    default: return at<int64_t>(v, i);
  }
}

sx_i128 i128_at(const std::vector<uint8_t>& v, int64_t i) {
  sx_i128 r;
  std::memcpy(&r, v.data() + 16 * i, 16);
  return r;
}

// Gather `cols` by the permutation and copy them to host (one sync at the end).
// The result rows: every output column gathered at the final permutation by ONE kernel into one
// device buffer, then ONE copy into pinned host memory and one synchronisation.
sx_status fetch_rows(sx_ctx* ctx, Bag& bag, const sx_col* cols, int n, const sx_sel& perm,
                     std::vector<std::vector<uint8_t>>& host) {
  host.assign(n, {});
  if (n > kMaxGather) return set_err(ctx, SX_EINVAL, "fetch_rows: %d columns", n);
  GatherSpec gs;
  gs.n = n;
  size_t off[kMaxGather + 1];
  off[0] = 0;
  for (int i = 0; i < n; ++i) {
    const int w = type_width(cols[i].type);
    if (!w) return set_err(ctx, SX_ETYPE, "fetch_rows: column %d is not fixed-width", i);
    gs.g[i].src = DCol{cols[i].data, cols[i].type, 0};
    gs.g[i].by_aux = 0;
    gs.g[i].width = w;
    off[i + 1] = off[i] + (((size_t)perm.len * w + 15) & ~(size_t)15);
  }
  uint8_t* dbuf;
  SX_TRY(alloc(ctx, &dbuf, off[n] > 0 ? off[n] : 16));
  bag.bufs.push_back(dbuf);
  for (int i = 0; i < n; ++i) gs.g[i].dst = dbuf + off[i];
  if (perm.len > 0) {
    k_gather_multi<<<persistent_grid(ctx, 8, (perm.len + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
        perm.idx, nullptr, perm.len, gs);
    SX_CHECK_LAUNCH();
  }
  if (ctx->h_stage_bytes < off[n]) {
    if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
    ctx->h_stage = nullptr;
    ctx->h_stage_bytes = 0;
    SX_CUDA(cudaMallocHost(&ctx->h_stage, off[n] + (1 << 16)));
    ctx->h_stage_bytes = off[n] + (1 << 16);
  }
  if (off[n]) SX_CUDA(cudaMemcpyAsync(ctx->h_stage, dbuf, off[n], cudaMemcpyDeviceToHost, ctx->stream));
  SX_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < n; ++i) {
    const size_t bytes = (size_t)perm.len * gs.g[i].width;
    host[i].resize(bytes + 16);
    std::memcpy(host[i].data(), (const uint8_t*)ctx->h_stage + off[i], bytes);
  }
  return SX_OK;
}

__global__ void k_lookup_rank(const int32_t* __restrict__ keys, int64_t n, const int32_t* __restrict__ rank_of,
                              int32_t nrank, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t k = keys[i];
    out[i] = (k >= 0 && k < nrank) ? rank_of[k] : nrank + k;
  }
}

// Q3 fused lineitem pass (K10q; SURVEY §8(a) Q3 steps 3 + 4, adjacent steps fused by the
// executor): lineitem is read once — l_shipdate and l_orderkey streamed with 128-bit loads, 8
// consecutive rows per lane — rows with shipdate > DATE are tested against the exact key-range
// bitmap of the qualifying orders (the orders build; two bitmap words serve a lane's 8 sorted
// keys), and only the ~0.5% rows that join load l_extendedprice / l_discount.  Each warp owns a
// CONTIGUOUS range of rows and the orderkey groups that start in it: it merges its joining rows'
// revenue terms in row order (warp-uniform state, lanes taken in order), skips the leading rows
// of the group begun before its range (the previous warp's), and reads past its range end while
// the last group continues.  One (orderkey, revenue) per order with >= 1 joining row is appended
// through a per-warp shared buffer; no group-by table.  Earlier versions: owned runs per THREAD
// (~100 instructions per row: 3.1 ms), and join records + sx_groupby_agg (1.06 + 0.76 ms).
// flags: [0] l_orderkey decreases (the plan takes the operator steps), [1] a product or a group
// sum left int64.
struct Q3Fused {
  const int32_t* okey;
  const int32_t* ship;
  const long long* ext;
  const long long* disc;
  int32_t date;
  const uint32_t* bm;
  long long bm_min;
  unsigned long long bm_bits;
  int32_t* out_key;
  longlong2* out_rev;
  int64_t cap;
  unsigned long long* cursor;
  int* flags;
  __device__ __forceinline__ bool joins1(int32_t k, int32_t sd) const {
    const uint32_t off = (uint32_t)k - (uint32_t)bm_min;
    return sd > date && off < (uint32_t)bm_bits && ((__ldg(bm + (off >> 5)) >> (off & 31)) & 1u);
  }
};

constexpr int kQ3Buf = 96, kQ3Flush = 64;  // a chunk closes <= 8 * 32 groups... flushed per group (see emit)
__global__ void __launch_bounds__(kBlock, 4) k_q3_fused(const __grid_constant__ Q3Fused a, int64_t n, int64_t per) {
  constexpr int R = 8;
  __shared__ int32_t s_key[kBlock / 32][kQ3Buf];
  __shared__ long long s_val[kBlock / 32][kQ3Buf];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t R0 = gw * per, R1 = min(n, R0 + per);
  if (R0 >= n) return;  // (warp-uniform)
  const uint32_t kmin = (uint32_t)a.bm_min, bits = (uint32_t)a.bm_bits;  // (bm_bits <= 2^30)
  bool ovf = false, bad = false;
  int cnt = 0;  // buffered groups (warp-uniform)
  auto flush = [&]() {  // warp-collective
    unsigned long long base = 0;
    if (lane == 0 && cnt) base = atomicAdd(a.cursor, (unsigned long long)cnt);
    base = __shfl_sync(kFull, base, 0);
    __syncwarp();
    for (int i = lane; i < cnt; i += 32) {
      const int64_t pos = (int64_t)base + i;
      if (pos < a.cap) {
        a.out_key[pos] = s_key[w][i];
        const long long v = s_val[w][i];
        a.out_rev[pos] = make_longlong2(v, v < 0 ? -1 : 0);
      }
    }
    __syncwarp();
    cnt = 0;
  };
  // warp-uniform current group
  bool cur = false;
  int32_t cur_key = 0;
  long long cur_sum = 0;
  auto add = [&](int32_t key, long long term) {  // warp-uniform call
    if (cur && key == cur_key) {
      cur_sum = add_ck(cur_sum, term, ovf);
      return;
    }
    if (cur) {
      if (lane == 0) {
        s_key[w][cnt] = cur_key;
        s_val[w][cnt] = cur_sum;
      }
      if (++cnt == kQ3Buf) flush();
    }
    cur = true;
    cur_key = key;
    cur_sum = term;
  };
  const bool has_prev = R0 > 0;
  const int32_t kprev = has_prev ? __ldg(a.okey + R0 - 1) : 0;  // rows of this group: the previous warp's
  int32_t lastk = kprev;  // last key seen (sortedness check across chunks)
  // (prefetching the next chunk into registers measured slower: 2.05 vs 1.87 ms at 3 CTAs/SM)
  for (int64_t base = R0; base < R1; base += 32 * R) {
    const int64_t r0 = base + (int64_t)lane * R;
    const int m = (int)max((int64_t)0, min((int64_t)R, R1 - r0));
    int32_t k[R], sd[R];
    if (m == R) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int4 x = __ldcs((const int4*)(a.okey + r0) + j), y = __ldcs((const int4*)(a.ship + r0) + j);
        k[4 * j] = x.x; k[4 * j + 1] = x.y; k[4 * j + 2] = x.z; k[4 * j + 3] = x.w;
        sd[4 * j] = y.x; sd[4 * j + 1] = y.y; sd[4 * j + 2] = y.z; sd[4 * j + 3] = y.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        k[i] = i < m ? __ldg(a.okey + r0 + i) : INT32_MAX;
        sd[i] = i < m ? __ldg(a.ship + r0 + i) : INT32_MIN;
      }
    }
    // keys non-decreasing across the chunk (lane order) and from the previous chunk
    {
      int32_t pk = __shfl_up_sync(kFull, k[R - 1], 1);
      if (lane == 0) pk = lastk;
      bool dec = (has_prev || base > R0 || lane > 0) && m > 0 && k[0] < pk;
#pragma unroll
      for (int i = 1; i < R; ++i) dec |= i < m && k[i] < k[i - 1];
      bad |= __any_sync(kFull, dec);
      int32_t lk = k[0];  // my last valid key (selects: no dynamic register indexing)
#pragma unroll
      for (int i = 1; i < R; ++i) lk = i < m ? k[i] : lk;
      const int lastlane = (int)min((int64_t)31, (R1 - 1 - base) / R);
      lastk = __shfl_sync(kFull, lk, lastlane);
    }
    uint32_t off[R];
    bool cand[R], anyc = false;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      off[i] = (uint32_t)k[i] - kmin;
      cand[i] = i < m && sd[i] > a.date && off[i] < bits && !(has_prev && k[i] == kprev);
      anyc |= cand[i];
    }
    unsigned qmask = 0;
    if (anyc) {
      const uint32_t w0 = off[0] >> 5, w1 = off[R - 1] >> 5;
      if (m == R && off[0] < bits && off[R - 1] < bits && w1 - w0 <= 1) {
        const uint32_t b0 = __ldg(a.bm + w0), b1 = __ldg(a.bm + w1);
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const uint32_t wd = (off[i] >> 5) == w0 ? b0 : b1;
          qmask |= (cand[i] && ((wd >> (off[i] & 31)) & 1u)) ? 1u << i : 0u;
        }
      } else {
#pragma unroll
        for (int i = 0; i < R; ++i)
          qmask |= (cand[i] && ((__ldg(a.bm + (off[i] >> 5)) >> (off[i] & 31)) & 1u)) ? 1u << i : 0u;
      }
    }
    unsigned lanes = __ballot_sync(kFull, qmask != 0);
    if (!lanes) continue;
    long long t[R];
#pragma unroll
    for (int i = 0; i < R; ++i)
      t[i] = ((qmask >> i) & 1u) ? mul_ck(__ldg(a.ext + r0 + i), 100 - __ldg(a.disc + r0 + i), ovf) : 0;
    // the joining rows in row order: lanes ascending, a lane's rows ascending
    while (lanes) {
      const int L = __ffs(lanes) - 1;
      lanes &= lanes - 1;
      const unsigned qm = __shfl_sync(kFull, qmask, L);
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int32_t key = __shfl_sync(kFull, k[i], L);
        const long long term = __shfl_sync(kFull, t[i], L);
        if ((qm >> i) & 1u) add(key, term);
      }
    }
  }
  // the range's last group continues past R1 (its owner is this warp)
  if (R1 < n) {
    const int32_t klast = __ldg(a.okey + R1 - 1);
    for (int64_t r = R1;; r += 32) {
      const int64_t rr = r + lane;
      const int32_t kr = rr < n ? __ldg(a.okey + rr) : INT32_MIN;
      const bool same = rr < n && kr == klast;
      const bool q = same && a.joins1(kr, __ldg(a.ship + rr)) && !(has_prev && kr == kprev);
      const long long term = q ? mul_ck(__ldg(a.ext + rr), 100 - __ldg(a.disc + rr), ovf) : 0;
      unsigned ql = __ballot_sync(kFull, q);
      while (ql) {
        const int L = __ffs(ql) - 1;
        ql &= ql - 1;
        add(klast, __shfl_sync(kFull, term, L));
      }
      if (__ballot_sync(kFull, same) != kFull) break;
    }
  }
  if (cur) {
    if (lane == 0) {
      s_key[w][cnt] = cur_key;
      s_val[w][cnt] = cur_sum;
    }
    ++cnt;
  }
  flush();
  if (bad) atomicExch(a.flags, 1);
  if (ovf) atomicExch(a.flags + 1, 1);
}

// Q3 step 2 for the fused plan: one pass over orders applies o_orderdate < DATE and the customer
// semi-join (the customer build's exact custkey bitmap) and sets the qualifying orderkeys' bits in
// an exact bitmap over [first key, last key] of o_orderkey — the join filter the lineitem pass
// probes (predicate transfer).  No selection vector and no separate build pass.  The
// bitmap is exact in any row order as long as every key lies in the range (else *flag: the plan
// takes the operator steps).  8 consecutive orders per thread: their keys share 1-2 bitmap words.
__global__ void __launch_bounds__(kBlock) k_q3_orders(const int32_t* __restrict__ okey, const int32_t* __restrict__ ocust,
                                                      const int32_t* __restrict__ odate, int64_t n, int32_t date,
                                                      const uint32_t* __restrict__ cbm, long long cbm_min,
                                                      unsigned long long cbm_bits, uint32_t* obm, long long omin,
                                                      unsigned long long obits, unsigned long long* count, int* flag) {
  constexpr int R = 8;
  unsigned long long c = 0;
  bool bad = false;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t * R < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r0 = t * R;
    int32_t k[R], cu[R], d[R];
    if (r0 + R <= n) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int4 x = __ldcs((const int4*)(okey + r0) + j), y = __ldcs((const int4*)(ocust + r0) + j),
                   z = __ldcs((const int4*)(odate + r0) + j);
        k[4 * j] = x.x; k[4 * j + 1] = x.y; k[4 * j + 2] = x.z; k[4 * j + 3] = x.w;
        cu[4 * j] = y.x; cu[4 * j + 1] = y.y; cu[4 * j + 2] = y.z; cu[4 * j + 3] = y.w;
        d[4 * j] = z.x; d[4 * j + 1] = z.y; d[4 * j + 2] = z.z; d[4 * j + 3] = z.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const bool in = r0 + i < n;
        k[i] = in ? __ldg(okey + r0 + i) : 0;
        cu[i] = in ? __ldg(ocust + r0 + i) : 0;
        d[i] = in ? __ldg(odate + r0 + i) : INT32_MAX;
      }
    }
    uint32_t w0 = 0xffffffffu, m0 = 0, w1 = 0xffffffffu, m1 = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const unsigned long long coff = (unsigned long long)((long long)cu[i] - cbm_min);
      const bool dq = d[i] < date && coff < cbm_bits;
      const bool q = dq && ((__ldg(cbm + (coff >> 5)) >> (coff & 31)) & 1u);
      if (!q) continue;
      const unsigned long long off = (unsigned long long)((long long)k[i] - omin);
      if (off >= obits) {
        bad = true;
        continue;
      }
      ++c;
      const uint32_t w = (uint32_t)(off >> 5), b = 1u << (off & 31);
      if (w == w0) m0 |= b;
      else if (w == w1) m1 |= b;
      else if (w0 == 0xffffffffu) { w0 = w; m0 = b; }
      else if (w1 == 0xffffffffu) { w1 = w; m1 = b; }
      else atomicOr(obm + w, b);
    }
    if (m0) atomicOr(obm + w0, m0);
    if (m1) atomicOr(obm + w1, m1);
  }
  c = __reduce_add_sync(kFull, (unsigned)c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
  if (bad) atomicExch(flag, 1);
}

// Q3 carries of each group: the order with that key, searched in o_orderkey (orders in strictly
// increasing key order) from an interpolated guess — TPC-H orderkeys are spread evenly, so the
// guess lands within a few rows — with an exponential then binary search around it; any key not
// found sets *notfound and the plan takes the operator steps.
__global__ void k_q3_carry(const int32_t* __restrict__ gk, int64_t ng, const int32_t* __restrict__ okey, int64_t no,
                           const int32_t* __restrict__ odate, const int32_t* __restrict__ oprio, int32_t* out_date,
                           int32_t* out_prio, int* notfound) {
  const long long kmin = __ldg(okey), kmax = __ldg(okey + no - 1);
  const double scale = kmax > kmin ? (double)(no - 1) / (double)(kmax - kmin) : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ng; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = gk[i];
    int64_t g = (int64_t)((double)((long long)k - kmin) * scale);
    g = g < 0 ? 0 : (g >= no ? no - 1 : g);
    // bracket [lo, hi) containing the first position with okey >= k
    int64_t lo, hi;  // the answer is the first position of [lo, hi) with okey >= k, else hi
    if (__ldg(okey + g) < k) {  // answer > g: probe g + 1, g + 2, g + 4, ...
      int64_t prev = g, step = 1, c = g + 1;  // okey[prev] < k
      while (c < no && __ldg(okey + c) < k) {
        prev = c;
        step <<= 1;
        c = g + step;
      }
      lo = prev + 1;
      hi = c < no ? c : no;  // okey[c] >= k, or the end
    } else {  // answer <= g: probe g - 1, g - 2, g - 4, ...
      int64_t prev = g, step = 1, c = g - 1;  // okey[prev] >= k
      while (c >= 0 && __ldg(okey + c) >= k) {
        prev = c;
        step <<= 1;
        c = g - step;
      }
      lo = c >= 0 ? c + 1 : 0;  // okey[c] < k, or the start
      hi = prev;
    }
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(okey + mid) < k) lo = mid + 1;
      else hi = mid;
    }
    if (lo < no && __ldg(okey + lo) == k) {
      out_date[i] = __ldg(odate + lo);
      out_prio[i] = __ldg(oprio + lo);
    } else {
      atomicExch(notfound, 1);
    }
  }
}

// Row of each probe key in a PK column stored in strictly increasing order (the executor's
// "sorted primary key" lookup; TPC-H's orders and customer are stored in key order): search from
// an interpolated guess, exponential then binary; a key not found sets *notfound (the plan then
// takes its hash-join steps, which decide inner-join semantics and unsorted tables).
template <typename KT>
__global__ void k_sorted_lookup(const KT* __restrict__ probe, int64_t np, const KT* __restrict__ sorted, int64_t ns,
                                int32_t* __restrict__ out_row, int* notfound) {
  if (ns <= 0) {
    if (np > 0 && blockIdx.x == 0 && threadIdx.x == 0) atomicExch(notfound, 1);
    return;
  }
  const long long kmin = (long long)__ldg(sorted), kmax = (long long)__ldg(sorted + ns - 1);
  const double scale = kmax > kmin ? (double)(ns - 1) / ((double)kmax - (double)kmin) : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
    const KT k = probe[i];
    double gd = ((double)k - (double)kmin) * scale;
    int64_t g = gd < 0 ? 0 : (gd >= (double)(ns - 1) ? ns - 1 : (int64_t)gd);
    int64_t lo, hi;  // the answer is the first position of [lo, hi) with key >= k, else hi
    if (__ldg(sorted + g) < k) {
      int64_t prev = g, step = 1, c = g + 1;
      while (c < ns && __ldg(sorted + c) < k) {
        prev = c;
        step <<= 1;
        c = g + step;
      }
      lo = prev + 1;
      hi = c < ns ? c : ns;
    } else {
      int64_t prev = g, step = 1, c = g - 1;
      while (c >= 0 && __ldg(sorted + c) >= k) {
        prev = c;
        step <<= 1;
        c = g - step;
      }
      lo = c >= 0 ? c + 1 : 0;
      hi = prev;
    }
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(sorted + mid) < k) lo = mid + 1;
      else hi = mid;
    }
    if (lo < ns && __ldg(sorted + lo) == k) out_row[i] = (int32_t)lo;
    else atomicExch(notfound, 1);
  }
}

// rows of `keys` (len n) in the sorted PK column pk; false when a key is missing (or pk unsorted)
sx_status sorted_lookup(sx_ctx* ctx, Bag& bag, const sx_col& pk, const sx_col& keys, int32_t** rows, bool* ok) {
  *ok = false;
  *rows = nullptr;
  if (pk.type != keys.type || !(w4(pk) || w8(pk)) || pk.len > INT32_MAX) return SX_OK;
  int32_t* r;
  SX_TRY(alloc(ctx, &r, (size_t)std::max<int64_t>(keys.len, 1)));
  bag.bufs.push_back(r);
  int* nf = ctx->d_flags + 8;
  SX_CUDA(cudaMemsetAsync(nf, 0, sizeof(int), ctx->stream));
  if (keys.len > 0) {
    const unsigned grid = persistent_grid(ctx, 8, (keys.len + kBlock - 1) / kBlock);
    if (w4(pk))
      k_sorted_lookup<int32_t><<<grid, kBlock, 0, SX_STREAM(ctx)>>>((const int32_t*)keys.data, keys.len,
                                                                   (const int32_t*)pk.data, pk.len, r, nf);
    else
      k_sorted_lookup<long long><<<grid, kBlock, 0, SX_STREAM(ctx)>>>((const long long*)keys.data, keys.len,
                                                                     (const long long*)pk.data, pk.len, r, nf);
    SX_CHECK_LAUNCH();
  }
  int h = 0;
  SX_CUDA(cudaMemcpy(&h, nf, sizeof(int), cudaMemcpyDeviceToHost));
  *ok = h == 0;
  *rows = r;
  return SX_OK;
}

// Q18's joins of the ~6.4e3 qualifying orderkeys in ONE kernel: each
// key's orders row by interpolated search of o_orderkey (as k_sorted_lookup), its o_custkey /
// o_orderdate / o_totalprice gathered, and the customer's existence checked by the same search of
// c_custkey (Q18 outputs c_custkey; an order without its customer would drop out of the inner
// join: *notfound sends the plan to the hash joins).  Replaces two lookups with a host sync each
// plus four gathers (0.29 ms at SF100, mostly launch and sync latency).
template <typename KT>
__device__ __forceinline__ int64_t sorted_pos(const KT* __restrict__ sorted, int64_t ns, KT k) {
  if (ns <= 0) return -1;
  const long long kmin = (long long)__ldg(sorted), kmax = (long long)__ldg(sorted + ns - 1);
  const double scale = kmax > kmin ? (double)(ns - 1) / ((double)kmax - (double)kmin) : 0.0;
  const double gd = ((double)k - (double)kmin) * scale;
  const int64_t g = gd < 0 ? 0 : (gd >= (double)(ns - 1) ? ns - 1 : (int64_t)gd);
  int64_t lo, hi;  // the answer is the first position of [lo, hi) with key >= k, else hi
  if (__ldg(sorted + g) < k) {
    int64_t prev = g, step = 1, c = g + 1;
    while (c < ns && __ldg(sorted + c) < k) {
      prev = c;
      step <<= 1;
      c = g + step;
    }
    lo = prev + 1;
    hi = c < ns ? c : ns;
  } else {
    int64_t prev = g, step = 1, c = g - 1;
    while (c >= 0 && __ldg(sorted + c) >= k) {
      prev = c;
      step <<= 1;
      c = g - step;
    }
    lo = c >= 0 ? c + 1 : 0;
    hi = prev;
  }
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(sorted + mid) < k) lo = mid + 1;
    else hi = mid;
  }
  return (lo < ns && __ldg(sorted + lo) == k) ? lo : -1;
}

template <typename KT>
__global__ void k_q18_join(const KT* __restrict__ gkey, int64_t ng, const KT* __restrict__ okey, int64_t no,
                           const int32_t* __restrict__ ocust, const int32_t* __restrict__ odate,
                           const long long* __restrict__ oprice, const int32_t* __restrict__ ckey, int64_t nc,
                           KT* r_key, int32_t* r_cust, int32_t* r_date, long long* r_price, int* notfound) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ng; i += (int64_t)gridDim.x * blockDim.x) {
    const KT k = gkey[i];
    const int64_t o = sorted_pos(okey, no, k);
    if (o < 0) {
      atomicExch(notfound, 1);
      continue;
    }
    const int32_t cu = __ldg(ocust + o);
    r_key[i] = k;
    r_cust[i] = cu;
    r_date[i] = __ldg(odate + o);
    r_price[i] = __ldg(oprice + o);
    if (sorted_pos(ckey, nc, cu) < 0) atomicExch(notfound, 1);
  }
}

// -> R[1..4] = o_orderkey, o_custkey, o_orderdate, o_totalprice of the keys; *ok = false when a key
// or a customer is missing, or the layouts do not fit (the caller takes the hash joins)
sx_status q18_join(sx_ctx* ctx, Bag& bag, const sx_tpch_tables* t, const sx_col& keys, sx_col* R, bool* ok) {
  *ok = false;
  const bool k4 = w4(t->o_orderkey) && keys.type == t->o_orderkey.type;
  const bool k8 = w8(t->o_orderkey) && keys.type == t->o_orderkey.type;
  if (!(k4 || k8) || !w4(t->o_custkey) || !w4(t->o_orderdate) || !w8(t->o_totalprice) || !w4(t->c_custkey) ||
      t->o_orderkey.len > INT32_MAX)
    return SX_OK;
  const int64_t ng = keys.len, kw = type_width(keys.type);
  void *rk, *rc, *rd, *rp;
  SX_TRY(alloc(ctx, (char**)&rk, (size_t)std::max<int64_t>(ng, 1) * kw));
  bag.bufs.push_back(rk);
  SX_TRY(alloc(ctx, (char**)&rc, (size_t)std::max<int64_t>(ng, 1) * 4));
  bag.bufs.push_back(rc);
  SX_TRY(alloc(ctx, (char**)&rd, (size_t)std::max<int64_t>(ng, 1) * 4));
  bag.bufs.push_back(rd);
  SX_TRY(alloc(ctx, (char**)&rp, (size_t)std::max<int64_t>(ng, 1) * 8));
  bag.bufs.push_back(rp);
  int* nf = ctx->d_flags + 8;
  SX_CUDA(cudaMemsetAsync(nf, 0, sizeof(int), ctx->stream));
  if (ng > 0) {
    const unsigned grid = persistent_grid(ctx, 8, (ng + kBlock - 1) / kBlock);
    if (k4)
      k_q18_join<int32_t><<<grid, kBlock, 0, SX_STREAM(ctx)>>>(
          (const int32_t*)keys.data, ng, (const int32_t*)t->o_orderkey.data, t->o_orderkey.len,
          (const int32_t*)t->o_custkey.data, (const int32_t*)t->o_orderdate.data, (const long long*)t->o_totalprice.data,
          (const int32_t*)t->c_custkey.data, t->c_custkey.len, (int32_t*)rk, (int32_t*)rc, (int32_t*)rd, (long long*)rp, nf);
    else
      k_q18_join<long long><<<grid, kBlock, 0, SX_STREAM(ctx)>>>(
          (const long long*)keys.data, ng, (const long long*)t->o_orderkey.data, t->o_orderkey.len,
          (const int32_t*)t->o_custkey.data, (const int32_t*)t->o_orderdate.data, (const long long*)t->o_totalprice.data,
          (const int32_t*)t->c_custkey.data, t->c_custkey.len, (long long*)rk, (int32_t*)rc, (int32_t*)rd, (long long*)rp, nf);
    SX_CHECK_LAUNCH();
  }
  int h = 0;
  SX_CUDA(cudaMemcpyAsync(&h, nf, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  SX_CUDA(cudaStreamSynchronize(ctx->stream));
  R[1] = sx_col{t->o_orderkey.type, t->o_orderkey.scale, ng, rk, nullptr, nullptr};
  R[2] = sx_col{t->o_custkey.type, t->o_custkey.scale, ng, rc, nullptr, nullptr};
  R[3] = sx_col{t->o_orderdate.type, t->o_orderdate.scale, ng, rd, nullptr, nullptr};
  R[4] = sx_col{t->o_totalprice.type, t->o_totalprice.scale, ng, rp, nullptr, nullptr};
  *ok = h == 0;
  return SX_OK;
}

static const char* kNation[25] = {"ALGERIA", "ARGENTINA", "BRAZIL", "CANADA", "EGYPT", "ETHIOPIA", "FRANCE",
                                  "GERMANY", "INDIA", "INDONESIA", "IRAN", "IRAQ", "JAPAN", "JORDAN", "KENYA",
                                  "MOROCCO", "MOZAMBIQUE", "PERU", "CHINA", "ROMANIA", "SAUDI ARABIA", "VIETNAM",
                                  "RUSSIA", "UNITED KINGDOM", "UNITED STATES"};

}  // namespace

SX_EXPORT void sx_tpch_default_params(sx_tpch_params* p) {
  std::memset(p, 0, sizeof(*p));
  p->q1_shipdate_max = 10471;
  p->q3_segment = 1;
  p->q3_date = 9204;
  p->q6_date_lo = 8766;
  p->q6_date_hi = 9131;
  p->q6_disc_lo = 5;
  p->q6_disc_hi = 7;
  p->q6_qty_lt = 2400;
  std::strcpy(p->q9_color, "green");
  p->q18_qty_gt = 30000;
  p->q3_limit = 10;
  p->q18_limit = 100;
}

// ------------------------------------------------------------------------------------- Q1
SX_EXPORT sx_status sx_tpch_q1(sx_ctx* ctx, const sx_tpch_tables* t, const sx_tpch_params* p, sx_q1_row* out,
                               int64_t cap, int64_t* nrows) {
  if (!ctx || !t || !p || !nrows) return SX_EINVAL;
  *nrows = 0;
  ProfScope ps(ctx, "Q1");
  Bag bag(ctx);
  sx_col cols[7] = {t->l_shipdate, t->l_returnflag, t->l_linestatus, t->l_quantity, t->l_extendedprice, t->l_discount,
                    t->l_tax};
  sx_key keys[2] = {{1, SX_KEY_IDENTITY}, {2, SX_KEY_IDENTITY}};
  sx_pred where = P(0, SX_LE, p->q1_shipdate_max);
  sx_agg aggs[8] = {
      A(SX_SUM, E1(1, {F(3)})),                                  // sum_qty            scale 2
      A(SX_SUM, E1(1, {F(4)})),                                  // sum_base_price     scale 2
      A(SX_SUM, E1(1, {F(4), F(5, -1, 100)})),                   // sum_disc_price     scale 4
      A(SX_SUM, E1(1, {F(4), F(5, -1, 100), F(6, 1, 100)})),     // sum_charge         scale 6
      A(SX_AVG, E1(1, {F(3)}), 2),                               // avg_qty
      A(SX_AVG, E1(1, {F(4)}), 2),                               // avg_price
      A(SX_AVG, E1(1, {F(5)}), 2),                               // avg_disc
      Count()};                                                  // count_order
  sx_col ok[2], oa[8];
  int64_t ng = 0;
  if (w4(t->l_shipdate) && w1(t->l_returnflag) && w1(t->l_linestatus) && w8(t->l_quantity) &&
      w8(t->l_extendedprice) && w8(t->l_discount) && w8(t->l_tax)) {
    ProfScope pg(ctx, "groupby");
    GbPlan plan;
    SX_TRY(to_dcols_check(ctx, cols, 7));
    SX_TRY(gb_plan(ctx, cols, 7, keys, 2, aggs, 8, nullptr, &plan));
    SX_TRY(check_states(ctx, plan, {ST_SUM, ST_SUM, ST_SUM, ST_SUM, ST_COUNT, ST_SUM}));
    Q1Prog prog{(const int32_t*)t->l_shipdate.data, (const uint8_t*)t->l_returnflag.data,
                (const uint8_t*)t->l_linestatus.data, (const long long*)t->l_quantity.data,
                (const long long*)t->l_extendedprice.data, (const long long*)t->l_discount.data,
                (const long long*)t->l_tax.data, p->q1_shipdate_max, ctx->d_flags};
    SX_TRY(gb_run(ctx, prog, plan, nullptr, t->l_shipdate.len, 4, ok, oa, &ng));
    pg.set_bytes(38.0 * t->l_shipdate.len + (2 + 4 * 16 + 3 * 8 + 8) * (double)ng);  // 7 columns once + G rows
  } else {
    SX_TRY(sx_groupby_agg(ctx, cols, 7, keys, 2, nullptr, &where, 1, aggs, 8, nullptr, 4, ok, oa, &ng));
  }
  bag.keep(ok, 2);
  bag.keep(oa, 8);
  // order by l_returnflag, l_linestatus
  sx_col sk[2] = {ok[0], ok[1]};
  sx_sortkey sks[2] = {{0, 0}, {1, 0}};
  sx_sel perm;
  SX_TRY(sx_sort_topk(ctx, sk, 2, sks, 2, nullptr, -1, &perm));
  bag.keep(perm);
  sx_col all[10] = {ok[0], ok[1], oa[0], oa[1], oa[2], oa[3], oa[4], oa[5], oa[6], oa[7]};
  std::vector<std::vector<uint8_t>> h;
  SX_TRY(fetch_rows(ctx, bag, all, 10, perm, h));
  if (perm.len > cap) return set_err(ctx, SX_EINVAL, "Q1: %lld rows > cap", (long long)perm.len);
  for (int64_t i = 0; i < perm.len; ++i) {
    sx_q1_row& r = out[i];
    std::memset(&r, 0, sizeof r);
    r.returnflag = h[0][i];
    r.linestatus = h[1][i];
    r.sum_qty = i128_at(h[2], i);
    r.sum_base_price = i128_at(h[3], i);
    r.sum_disc_price = i128_at(h[4], i);
    r.sum_charge = i128_at(h[5], i);
    r.avg_qty = at<double>(h[6], i);
    r.avg_price = at<double>(h[7], i);
    r.avg_disc = at<double>(h[8], i);
    r.count_order = at<int64_t>(h[9], i);
  }
  *nrows = perm.len;
  return SX_OK;
}

// ------------------------------------------------------------------------------------- Q6
SX_EXPORT sx_status sx_tpch_q6(sx_ctx* ctx, const sx_tpch_tables* t, const sx_tpch_params* p, sx_q6_row* out,
                               int64_t* nrows) {
  if (!ctx || !t || !p || !nrows || !out) return SX_EINVAL;
  *nrows = 0;
  ProfScope ps(ctx, "Q6");
  Bag bag(ctx);
  sx_col cols[4] = {t->l_shipdate, t->l_discount, t->l_quantity, t->l_extendedprice};
  sx_pred where[4] = {P(0, SX_GE, p->q6_date_lo), P(0, SX_LT, p->q6_date_hi),
                      P(1, SX_BETWEEN, p->q6_disc_lo, p->q6_disc_hi), P(2, SX_LT, p->q6_qty_lt)};
  sx_agg aggs[2] = {A(SX_SUM, E1(1, {F(3), F(1)})), Count()};  // sum(l_extendedprice*l_discount) scale 4
  sx_col oa[2];
  int64_t ng = 0;
  if (w4(t->l_shipdate) && w8(t->l_discount) && w8(t->l_quantity) && w8(t->l_extendedprice)) {
    ProfScope pg(ctx, "groupby");
    GbPlan plan;
    SX_TRY(to_dcols_check(ctx, cols, 4));
    SX_TRY(gb_plan(ctx, cols, 4, nullptr, 0, aggs, 2, nullptr, &plan));
    SX_TRY(check_states(ctx, plan, {ST_SUM, ST_COUNT}));
    Q6Prog prog{(const int32_t*)t->l_shipdate.data, (const long long*)t->l_discount.data,
                (const long long*)t->l_quantity.data, (const long long*)t->l_extendedprice.data, p->q6_date_lo,
                p->q6_date_hi, p->q6_disc_lo, p->q6_disc_hi, p->q6_qty_lt, ctx->d_flags,
                getenv("SX_Q6_LAZY3") && getenv("SX_Q6_LAZY3")[0] == '1' ? 1 : 0};
    SX_TRY(gb_run(ctx, prog, plan, nullptr, t->l_shipdate.len, 1, nullptr, oa, &ng));
    pg.set_bytes(28.0 * t->l_shipdate.len + 24.0);  // 4 columns once + the result
  } else {
    SX_TRY(sx_groupby_agg(ctx, cols, 4, nullptr, 0, nullptr, where, 4, aggs, 2, nullptr, 1, nullptr, oa, &ng));
  }
  bag.keep(oa, 2);
  std::vector<uint8_t> hs, hc;
  SX_TRY(d2h(ctx, oa[0], hs));
  SX_TRY(d2h(ctx, oa[1], hc));
  SX_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memset(out, 0, sizeof *out);
  out->revenue = i128_at(hs, 0);
  out->is_null = at<int64_t>(hc, 0) == 0;
  *nrows = 1;
  return SX_OK;
}

// ------------------------------------------------------------------------------------- Q3
SX_EXPORT sx_status sx_tpch_q3(sx_ctx* ctx, const sx_tpch_tables* t, const sx_tpch_params* p, sx_q3_row* out,
                               int64_t cap, int64_t* nrows) {
  if (!ctx || !t || !p || !nrows) return SX_EINVAL;
  *nrows = 0;
  ProfScope ps(ctx, "Q3");
  Bag bag(ctx);
  // 1. C = {c_custkey | c_mktsegment = SEGMENT}
  sx_col ccols[2] = {t->c_custkey, t->c_mktsegment};
  sx_pred cseg = P(1, SX_EQ, p->q3_segment);
  sx_sel sel_c;
  SX_TRY(sx_filter(ctx, ccols, 2, &cseg, 1, nullptr, nullptr, 0, &sel_c, nullptr));
  bag.keep(sel_c);
  int32_t k0 = 0;
  sx_ht* ht_c;
  SX_TRY(sx_hash_build(ctx, ccols, 2, &k0, 1, &sel_c, nullptr, 0, 1, &ht_c));
  bag.keep(ht_c);
  // 2-4 fused (default; SX_Q3_PLAN=ops forces the operator-at-a-time steps below): one pass over
  // orders sets the exact bitmap of the qualifying orderkeys (k_q3_orders), one pass over lineitem
  // probes it and sums revenue per orderkey (k_q3_fused), and the groups' o_orderdate /
  // o_shippriority come from a search of o_orderkey (orders in key order; any key not found sends
  // the plan to the operator steps).  (3.27 vs 3.61 ms for Q3 at SF100 with a membership build.)
  const bool ops_plan = getenv("SX_Q3_PLAN") && std::strcmp(getenv("SX_Q3_PLAN"), "ops") == 0;
  const int64_t no = t->o_orderkey.len;
  uint32_t* obm = nullptr;
  long long omin = 0;
  unsigned long long obits = 0;
  int64_t nqual = 0;
  bool fused = false;
  if (!ops_plan && ht_c->bm && w4(t->o_orderkey) && w4(t->o_custkey) && w4(t->o_orderdate) &&
      w4(t->o_shippriority) && t->o_custkey.len == no && t->o_orderdate.len == no && no > 0 && w4(t->l_orderkey) &&
      w4(t->l_shipdate) && w8(t->l_extendedprice) && w8(t->l_discount) && t->l_shipdate.len == t->l_orderkey.len &&
      t->l_extendedprice.len == t->l_orderkey.len && t->l_discount.len == t->l_orderkey.len &&
      t->l_orderkey.len > 0) {
    ProfScope pb(ctx, "probe_semi");  // the semi-join and the orderkey bitmap in one pass
    int32_t* hp = (int32_t*)(ctx->h_pinned + 20);
    SX_CUDA(cudaMemcpyAsync(hp, t->o_orderkey.data, 4, cudaMemcpyDeviceToHost, ctx->stream));
    SX_CUDA(cudaMemcpyAsync(hp + 1, (const int32_t*)t->o_orderkey.data + no - 1, 4, cudaMemcpyDeviceToHost, ctx->stream));
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
    omin = hp[0];
    if (hp[1] >= hp[0] && (unsigned long long)((long long)hp[1] - hp[0]) + 1 <= (1ull << 30)) {
      obits = (unsigned long long)((long long)hp[1] - hp[0]) + 1;
      const size_t words = (size_t)((obits + 31) / 32);
      SX_TRY(alloc(ctx, &obm, words));
      bag.bufs.push_back(obm);
      SX_CUDA(cudaMemsetAsync(obm, 0, words * sizeof(uint32_t), ctx->stream));
      unsigned long long* cntp = (unsigned long long*)ctx->d_counters;
      SX_CUDA(cudaMemsetAsync(cntp, 0, 8, ctx->stream));
      SX_CUDA(cudaMemsetAsync(ctx->d_flags, 0, sizeof(int), ctx->stream));
      k_q3_orders<<<persistent_grid(ctx, 8, ((no + 7) / 8 + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
          (const int32_t*)t->o_orderkey.data, (const int32_t*)t->o_custkey.data, (const int32_t*)t->o_orderdate.data,
          no, (int32_t)std::max<int64_t>(INT32_MIN, std::min<int64_t>(INT32_MAX, p->q3_date)), ht_c->bm, ht_c->bm_min,
          ht_c->bm_bits, obm, omin, obits, cntp, ctx->d_flags);
      SX_CHECK_LAUNCH();
      SX_TRY(read_i64(ctx, cntp, &nqual));
      int fl = 0;
      SX_CUDA(cudaMemcpy(&fl, ctx->d_flags, sizeof(int), cudaMemcpyDeviceToHost));
      fused = fl == 0;
      pb.set_bytes(12.0 * no + (double)words * 4);
    }
  }
  if (fused) {
    const int64_t n = t->l_orderkey.len;
    const int64_t gcap = std::max<int64_t>(1, nqual);  // groups are qualifying orders
    int32_t* gk;
    longlong2* grev;
    SX_TRY(alloc(ctx, &gk, (size_t)gcap));
    bag.bufs.push_back(gk);
    SX_TRY(alloc(ctx, &grev, (size_t)gcap));
    bag.bufs.push_back(grev);
    Q3Fused a{};
    a.okey = (const int32_t*)t->l_orderkey.data;
    a.ship = (const int32_t*)t->l_shipdate.data;
    a.ext = (const long long*)t->l_extendedprice.data;
    a.disc = (const long long*)t->l_discount.data;
    a.date = (int32_t)std::max<int64_t>(INT32_MIN, std::min<int64_t>(INT32_MAX, p->q3_date));
    a.bm = obm;
    a.bm_min = omin;
    a.bm_bits = obits;
    a.out_key = gk;
    a.out_rev = grev;
    a.cap = gcap;
    a.cursor = (unsigned long long*)ctx->d_counters;
    a.flags = ctx->d_flags;
    int64_t cnt = 0;
    int fl[2] = {0, 0};
    {
      ProfScope pg(ctx, "probe_groupby");
      SX_CUDA(cudaMemsetAsync(a.cursor, 0, 8, ctx->stream));
      SX_CUDA(cudaMemsetAsync(a.flags, 0, 2 * sizeof(int), ctx->stream));
      // one warp per contiguous range of whole 256-row chunks, every warp of a persistent grid
      const unsigned grid = persistent_grid(ctx, 4, ((n + 255) / 256 + (kBlock / 32) - 1) / (kBlock / 32));
      const int64_t warps = (int64_t)grid * (kBlock / 32);
      const int64_t per = ((n + warps - 1) / warps + 255) / 256 * 256;
      k_q3_fused<<<grid, kBlock, 0, SX_STREAM(ctx)>>>(a, n, per);
      SX_CHECK_LAUNCH();
      SX_TRY(read_i64(ctx, a.cursor, &cnt));
      SX_CUDA(cudaMemcpy(fl, a.flags, sizeof fl, cudaMemcpyDeviceToHost));
      // algorithmic bytes: l_orderkey + l_shipdate once, ext + disc of the joined rows, the groups
      pg.set_bytes(8.0 * n + 20.0 * cnt);
    }
    const bool grouped = !fl[0] && !fl[1] && cnt <= gcap;
    bool carried = false;
    sx_col pay[2];
    if (grouped) {
      ProfScope pc(ctx, "probe_inner");
      int32_t *cd, *cp;
      SX_TRY(alloc(ctx, &cd, (size_t)std::max<int64_t>(cnt, 1)));
      bag.bufs.push_back(cd);
      SX_TRY(alloc(ctx, &cp, (size_t)std::max<int64_t>(cnt, 1)));
      bag.bufs.push_back(cp);
      SX_CUDA(cudaMemsetAsync(a.flags, 0, sizeof(int), ctx->stream));
      if (cnt > 0) {
        k_q3_carry<<<persistent_grid(ctx, 8, (cnt + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
            gk, cnt, (const int32_t*)t->o_orderkey.data, t->o_orderkey.len, (const int32_t*)t->o_orderdate.data,
            (const int32_t*)t->o_shippriority.data, cd, cp, a.flags);
        SX_CHECK_LAUNCH();
      }
      int nf = 0;
      SX_CUDA(cudaMemcpy(&nf, a.flags, sizeof(int), cudaMemcpyDeviceToHost));
      carried = nf == 0;
      pay[0] = sx_col{t->o_orderdate.type, 0, cnt, cd, nullptr, nullptr};
      pay[1] = sx_col{t->o_shippriority.type, 0, cnt, cp, nullptr, nullptr};
      pc.set_bytes(4.0 * cnt * 3 + 8.0 * cnt);
    }
    if (carried) {
      sx_col gkc{SX_I32, 0, cnt, gk, nullptr, nullptr};
      sx_col grc{SX_I128, 4, cnt, grev, nullptr, nullptr};
      sx_col scols[3] = {grc, pay[0], gkc};
      sx_sortkey sks[3] = {{0, 1}, {1, 0}, {2, 0}};
      sx_sel perm;
      SX_TRY(sx_sort_topk(ctx, scols, 3, sks, 3, nullptr, p->q3_limit, &perm));
      bag.keep(perm);
      sx_col all[4] = {gkc, grc, pay[0], pay[1]};
      std::vector<std::vector<uint8_t>> h;
      SX_TRY(fetch_rows(ctx, bag, all, 4, perm, h));
      if (perm.len > cap) return set_err(ctx, SX_EINVAL, "Q3: %lld rows > cap", (long long)perm.len);
      for (int64_t i = 0; i < perm.len; ++i) {
        out[i].l_orderkey = key_at(h[0], SX_I32, i);
        out[i].revenue = i128_at(h[1], i);
        out[i].o_orderdate = (int32_t)key_at(h[2], pay[0].type, i);
        out[i].o_shippriority = (int32_t)key_at(h[3], pay[1].type, i);
      }
      *nrows = perm.len;
      return SX_OK;
    }
    // unsorted lineitem, an overflow, or orders not in key order: the operator plan decides
  }
  // 2. orders with o_orderdate < DATE and o_custkey in C (semi join), then build orderkey -> row
  sx_col ocols[2] = {t->o_custkey, t->o_orderdate};
  sx_pred odate = P(1, SX_LT, p->q3_date);
  sx_sel sel_o;
  SX_TRY(sx_hash_probe(ctx, ht_c, ocols, 2, &k0, 1, nullptr, &odate, 1, SX_SEMI, nullptr, 0, nullptr, 0, nullptr, 0,
                       &sel_o, nullptr, nullptr));
  bag.keep(sel_o);
  sx_col okey[1] = {t->o_orderkey};
  sx_ht* ht_o;
  SX_TRY(sx_hash_build(ctx, okey, 1, &k0, 1, &sel_o, nullptr, 0, 1, &ht_o));
  bag.keep(ht_o);
  // 3. lineitem with l_shipdate > DATE joined to those orders (unique build: ordered output)
  sx_col lcols[4] = {t->l_orderkey, t->l_shipdate, t->l_extendedprice, t->l_discount};
  sx_pred lship = P(1, SX_GT, p->q3_date);
  sx_col bcols[2] = {t->o_orderdate, t->o_shippriority};
  int32_t bp[2] = {0, 1}, pp[3] = {0, 2, 3};
  sx_sel jp, jb;
  sx_col pay[5];  // o_orderdate, o_shippriority, l_orderkey, ext, disc
  SX_TRY(sx_hash_probe(ctx, ht_o, lcols, 4, &k0, 1, nullptr, &lship, 1, SX_INNER, bcols, 2, bp, 2, pp, 3, &jp, &jb, pay));
  bag.keep(jp);
  bag.keep(jb);
  bag.keep(pay, 5);
  // 4. group by l_orderkey: revenue = sum(ext*(100-disc)) [scale 4]; o_orderdate, o_shippriority are
  //    functionally dependent on the key and carried with min() (reading R7)
  sx_col gcols[5] = {pay[2], pay[3], pay[4], pay[0], pay[1]};
  sx_key gk = {0, SX_KEY_IDENTITY};
  sx_agg gaggs[3] = {A(SX_SUM, E1(1, {F(1), F(2, -1, 100)})), A(SX_MIN, E1(1, {F(3)})), A(SX_MIN, E1(1, {F(4)}))};
  sx_col gok[1], goa[3];
  int64_t ng = 0;
  SX_TRY(sx_groupby_agg(ctx, gcols, 5, &gk, 1, nullptr, nullptr, 0, gaggs, 3, nullptr, jp.len / 2 + 1, gok, goa, &ng));
  bag.keep(gok, 1);
  bag.keep(goa, 3);
  // 5. order by revenue desc, o_orderdate asc, l_orderkey asc (reading R6); limit
  sx_col scols[3] = {goa[0], goa[1], gok[0]};
  sx_sortkey sks[3] = {{0, 1}, {1, 0}, {2, 0}};
  sx_sel perm;
  SX_TRY(sx_sort_topk(ctx, scols, 3, sks, 3, nullptr, p->q3_limit, &perm));
  bag.keep(perm);
  sx_col all[4] = {gok[0], goa[0], goa[1], goa[2]};
  std::vector<std::vector<uint8_t>> h;
  SX_TRY(fetch_rows(ctx, bag, all, 4, perm, h));
  if (perm.len > cap) return set_err(ctx, SX_EINVAL, "Q3: %lld rows > cap", (long long)perm.len);
  for (int64_t i = 0; i < perm.len; ++i) {
    out[i].l_orderkey = key_at(h[0], gok[0].type, i);
    out[i].revenue = i128_at(h[1], i);
    out[i].o_orderdate = (int32_t)at<int64_t>(h[2], i);
    out[i].o_shippriority = (int32_t)at<int64_t>(h[3], i);
  }
  *nrows = perm.len;
  return SX_OK;
}

// ------------------------------------------------------------------------------------- Q9
SX_EXPORT sx_status sx_tpch_q9(sx_ctx* ctx, const sx_tpch_tables* t, const sx_tpch_params* p, sx_q9_row* out,
                               int64_t cap, int64_t* nrows) {
  if (!ctx || !t || !p || !nrows) return SX_EINVAL;
  *nrows = 0;
  ProfScope ps(ctx, "Q9");
  Bag bag(ctx);
  int32_t k0 = 0;
  // 1. P = {p_partkey | p_name like '%COLOR%'}
  sx_col pn[1] = {t->p_name};
  sx_pred like = sx_pred{0, SX_CONTAINS, 0, 0, p->q9_color, (int32_t)strnlen(p->q9_color, sizeof p->q9_color), 0};
  sx_sel sel_p;
  SX_TRY(sx_filter(ctx, pn, 1, &like, 1, nullptr, nullptr, 0, &sel_p, nullptr));
  bag.keep(sel_p);
  sx_col pk[1] = {t->p_partkey};
  sx_ht* ht_p;
  SX_TRY(sx_hash_build(ctx, pk, 1, &k0, 1, &sel_p, nullptr, 0, 1, &ht_p));
  bag.keep(ht_p);
  sx_col gok[2], goa[1];
  int64_t ng = 0;
  // Fused plan (default): lineitem semi-join green parts (selection only); PK tables for
  // partsupp' (partkey, suppkey), supplier and the orders that have a green line (semi-join
  // reduction through a membership-only build); then one group-by pass over the selected lineitem
  // rows probing all three tables (Q9FusedProg).  SX_Q9_PLAN=ops: the operator-at-a-time plan below
  // (every join output materialised).
  const bool ops_plan = getenv("SX_Q9_PLAN") && std::strcmp(getenv("SX_Q9_PLAN"), "ops") == 0;
  const bool okb4 = w4(t->o_orderkey) && w4(t->l_orderkey), okb8 = w8(t->o_orderkey) && w8(t->l_orderkey);
  // the fused plan needs exact key-range bitmaps (key ranges <= 2^30); SX_EUNSUPPORTED from it
  // (e.g. SF1000's 64-bit orderkey range) falls back to the operator-at-a-time plan
  auto fused = [&]() -> sx_status {
    // default (SX_Q9_SCAN=wscan): one pass over lineitem (K10w) streams l_partkey, tests the
    // green-part bitmap, compacts the green rows per warp and runs the lookup chain on them with
    // every lane busy; no semi-join pass, no selection vector (8.1 vs 11.6 ms for Q9 at SF100).
    // SX_Q9_SCAN=gather: semi-join first, then the probe-chain group-by gathers the selected rows
    // (K10); =mat: the semi-join materialises the six columns densely first (one pure gather
    // kernel) and the group-by streams them; =dense: every lineitem column streamed with the
    // lookups per thread (K10d, latency-bound: 46 ms).  DESIGN.md §6.
    const char* scan_env = getenv("SX_Q9_SCAN");
    const bool wscan = !scan_env || std::strcmp(scan_env, "wscan") == 0;
    const bool dense_scan = wscan || (scan_env && std::strcmp(scan_env, "dense") == 0);
    const bool gather = !dense_scan;
    const bool mat = gather && scan_env && std::strcmp(scan_env, "mat") == 0;
    // lineitem rows with a green part (exact bitmap semi-join)
    sx_sel sel_l{0, nullptr};
    sx_col LM[6];  // materialised: partkey, suppkey, orderkey, qty, ext, disc of the green rows
    if (gather) {
      if (mat) {
        sx_col lc[6] = {t->l_partkey, t->l_suppkey, t->l_orderkey, t->l_quantity, t->l_extendedprice, t->l_discount};
        int32_t lpp[6] = {0, 1, 2, 3, 4, 5};
        SX_TRY(sx_hash_probe(ctx, ht_p, lc, 6, &k0, 1, nullptr, nullptr, 0, SX_SEMI, nullptr, 0, nullptr, 0, lpp, 6,
                             &sel_l, nullptr, LM));
        bag.keep(LM, 6);
      } else {
        SX_TRY(sx_hash_probe(ctx, ht_p, &t->l_partkey, 1, &k0, 1, nullptr, nullptr, 0, SX_SEMI, nullptr, 0, nullptr,
                             0, nullptr, 0, &sel_l, nullptr, nullptr));
      }
      bag.keep(sel_l);
    }
    sx_col pscols[2] = {t->ps_partkey, t->ps_suppkey};
    // PK lookup tables with the looked-up value inline (PayloadTable: one random access each)
    struct PtBag {
      sx_ctx* c;
      PayloadTable t[3];
      ~PtBag() {
        for (auto& x : t) free_payload_table(c, &x);
      }
    } pt{ctx, {}};
    sx_ht* ht_lo;
    {
      sx_sel sel_ps;
      SX_TRY(sx_hash_probe(ctx, ht_p, pscols, 2, &k0, 1, nullptr, nullptr, 0, SX_SEMI, nullptr, 0, nullptr, 0, nullptr,
                           0, &sel_ps, nullptr, nullptr));
      bag.keep(sel_ps);
      ProfScope pb(ctx, "hash_build");
      SX_TRY(build_payload_table(ctx, pscols, 2, t->ps_supplycost, &sel_ps, &pt.t[0]));
      pb.set_bytes((8.0 + 4.0 + 16.0) * sel_ps.len);
    }
    // supplier: membership bitmap over the suppkey range + a direct nation array
    sx_ht* ht_s;
    SX_TRY(sx_hash_build(ctx, &t->s_suppkey, 1, &k0, 1, nullptr, nullptr, 0, SX_BUILD_UNIQUE | SX_BUILD_MEMBERSHIP, &ht_s));
    bag.keep(ht_s);
    int32_t* s_nat = nullptr;
    if (!ht_s->bm && t->s_suppkey.len > 0) return set_err(ctx, SX_EUNSUPPORTED, "Q9: suppkey range too wide");
    SX_TRY(alloc(ctx, &s_nat, (size_t)(ht_s->bm_bits > 0 ? ht_s->bm_bits : 1)));
    bag.bufs.push_back(s_nat);
    if (t->s_suppkey.len > 0) {
      const int64_t ns = t->s_suppkey.len;
      k_direct_fill<int32_t, int32_t><<<persistent_grid(ctx, 8, (ns + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
          (const int32_t*)t->s_suppkey.data, (const int32_t*)t->s_nationkey.data, ns, nullptr, ht_s->bm_min,
          ht_s->bm_bits, s_nat, nullptr);
      SX_CHECK_LAUNCH();
    }
    // orders: the exact bitmap of the orderkeys that can be looked up (gather mode: the green
    // lines' keys, a semi-join reduction; dense mode: every orderkey), then o_orderdate scattered
    // into a direct array over that key range (one pass over orders, no hash table: each later
    // lookup is one bitmap word and one 4-byte read)
    const int64_t no = t->o_orderkey.len;
    long long o_min = 0;
    unsigned long long o_n = 0;
    const uint32_t* o_bm = nullptr;
    if (gather) {
      if (mat)
        SX_TRY(sx_hash_build(ctx, &LM[2], 1, &k0, 1, nullptr, nullptr, 0, SX_BUILD_MEMBERSHIP, &ht_lo));
      else
        SX_TRY(sx_hash_build(ctx, &t->l_orderkey, 1, &k0, 1, &sel_l, nullptr, 0, SX_BUILD_MEMBERSHIP, &ht_lo));
      bag.keep(ht_lo);
      if (!ht_lo->bm && sel_l.len > 0) return set_err(ctx, SX_EUNSUPPORTED, "Q9: orderkey range too wide");
      o_min = ht_lo->bm_min;
      o_n = ht_lo->bm ? ht_lo->bm_bits : 0;
      o_bm = ht_lo->bm;
    }
    uint8_t* o_date = nullptr;
    long long* d_bad = nullptr;
    SX_TRY(alloc(ctx, &d_bad, 2));
    bag.bufs.push_back(d_bad);
    SX_CUDA(cudaMemsetAsync(d_bad, 0, 2 * sizeof(long long), ctx->stream));
    bool filled = false;
    if (!gather && no > 0) {
      // orders in key order (the common case): the range from the end keys, one fill pass
      ProfScope pb(ctx, "hash_build");
      long long ends[2];
      const size_t kw = type_width(t->o_orderkey.type);
      int64_t* hp = ctx->h_pinned + 16;
      SX_CUDA(cudaMemcpyAsync(hp, t->o_orderkey.data, kw, cudaMemcpyDeviceToHost, ctx->stream));
      SX_CUDA(cudaMemcpyAsync(hp + 1, (const uint8_t*)t->o_orderkey.data + (no - 1) * kw, kw, cudaMemcpyDeviceToHost,
                              ctx->stream));
      SX_CUDA(cudaStreamSynchronize(ctx->stream));
      ends[0] = kw == 4 ? (long long)*(const int32_t*)hp : (long long)hp[0];
      ends[1] = kw == 4 ? (long long)*(const int32_t*)(hp + 1) : (long long)hp[1];
      const bool sorted_shape = ends[1] >= ends[0] && (unsigned long long)(ends[1] - ends[0]) + 1 <= (1ull << 30) &&
                                (unsigned long long)(ends[1] - ends[0]) + 1 >= (unsigned long long)no;
      if (sorted_shape) {
        o_min = ends[0];
        o_n = (unsigned long long)(ends[1] - ends[0]) + 1;
        SX_TRY(alloc(ctx, &o_date, (size_t)o_n));
        bag.bufs.push_back(o_date);
        const int64_t threads = (no + 255) / 256 * 32;  // one warp per 256 orders
        if (okb4)
          k_date_fill_sorted<int32_t><<<persistent_grid(ctx, 8, (threads + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
              (const int32_t*)t->o_orderkey.data, (const int32_t*)t->o_orderdate.data, no, o_min, o_n, o_date, d_bad);
        else
          k_date_fill_sorted<long long><<<persistent_grid(ctx, 8, (threads + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
              (const long long*)t->o_orderkey.data, (const int32_t*)t->o_orderdate.data, no, o_min, o_n, o_date, d_bad);
        SX_CHECK_LAUNCH();
        int64_t bb[2] = {0, 0};
        SX_TRY(read_i64(ctx, d_bad, bb, 2));
        filled = bb[1] == 0;  // else: not in key order, the scatter below
        if (!filled) SX_CUDA(cudaMemsetAsync(d_bad, 0, 2 * sizeof(long long), ctx->stream));
        pb.set_bytes((type_width(t->o_orderkey.type) + 4.0) * no + 1.0 * o_n);
      }
    }
    if (!gather && no > 0 && !filled) {
      // every order: the key range only (no bitmap); the date array starts as "no order"
      ProfScope pb(ctx, "hash_build");
      long long* d_mm = nullptr;
      SX_TRY(alloc(ctx, &d_mm, 2));
      bag.bufs.push_back(d_mm);
      long long init[2] = {LLONG_MAX, LLONG_MIN};
      SX_CUDA(cudaMemcpyAsync(d_mm, init, sizeof init, cudaMemcpyHostToDevice, ctx->stream));
      if (okb4)
        k_key_range<int32_t><<<persistent_grid(ctx, 8, (no + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
            (const int32_t*)t->o_orderkey.data, no, d_mm);
      else
        k_key_range<long long><<<persistent_grid(ctx, 8, (no + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
            (const long long*)t->o_orderkey.data, no, d_mm);
      SX_CHECK_LAUNCH();
      int64_t mm[2] = {0, 0};
      SX_TRY(read_i64(ctx, d_mm, mm, 2));
      if (mm[1] < mm[0] || (unsigned long long)(mm[1] - mm[0]) + 1 > (1ull << 30))
        return set_err(ctx, SX_EUNSUPPORTED, "Q9: orderkey range too wide");
      o_min = mm[0];
      o_n = (unsigned long long)(mm[1] - mm[0]) + 1;
      pb.set_bytes((double)type_width(t->o_orderkey.type) * no);
    }
    // year(o_orderdate) as one byte (kYear0 .. kYear0 + 127; a quarter of the bytes of int32
    // dates); a year outside that range makes the fused plan step aside (SX_EUNSUPPORTED)
    if (!filled) {
      SX_TRY(alloc(ctx, &o_date, (size_t)(o_n > 0 ? o_n : 1)));
      bag.bufs.push_back(o_date);
      ProfScope pb(ctx, "hash_build");
      if (!gather && o_n > 0) SX_CUDA(cudaMemsetAsync(o_date, kNoYear, o_n, ctx->stream));
      // gather: only the green lines' orderkeys (test the bitmap); otherwise every order
      if (no > 0 && o_n > 0) {
        if (okb4)
          k_direct_fill<int32_t, uint8_t><<<persistent_grid(ctx, 8, (no + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
              (const int32_t*)t->o_orderkey.data, (const int32_t*)t->o_orderdate.data, no, o_bm, o_min, o_n, o_date,
              d_bad);
        else
          k_direct_fill<long long, uint8_t><<<persistent_grid(ctx, 8, (no + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
              (const long long*)t->o_orderkey.data, (const int32_t*)t->o_orderdate.data, no, o_bm, o_min, o_n,
              o_date, d_bad);
        SX_CHECK_LAUNCH();
      }
      pb.set_bytes((type_width(t->o_orderkey.type) + 4.0) * no);
    }
    int64_t bad = 0;
    SX_TRY(read_i64(ctx, d_bad, &bad));
    if (bad) return set_err(ctx, SX_EUNSUPPORTED, "Q9: year(o_orderdate) outside the year-byte range");
    if (pt.t[0].kb != 8) return set_err(ctx, SX_EINVAL, "Q9: unexpected table layouts");
    ProfScope pg(ctx, "probe_groupby");
    sx_col tcols[6] = {t->s_nationkey, t->ps_supplycost, t->l_quantity, t->l_extendedprice, t->l_discount,
                       t->o_orderdate};  // types only: the plan's state layout
    sx_key gk[2] = {{0, SX_KEY_IDENTITY}, {5, SX_KEY_YEAR}};
    sx_agg ga;
    std::memset(&ga, 0, sizeof ga);
    ga.op = SX_SUM;
    ga.value.nterms = 2;
    ga.value.t[0].coef = 1;
    ga.value.t[0].nf = 2;
    ga.value.t[0].f[0] = F(3);
    ga.value.t[0].f[1] = F(4, -1, 100);
    ga.value.t[1].coef = -1;
    ga.value.t[1].nf = 2;
    ga.value.t[1].f[0] = F(1);
    ga.value.t[1].f[1] = F(2);
    GbPlan plan;
    SX_TRY(gb_plan(ctx, tcols, 6, gk, 2, &ga, 1, nullptr, &plan));
    SX_TRY(check_states(ctx, plan, {ST_SUM}));
    const int64_t n = gather ? sel_l.len : t->l_partkey.len;
    const int32_t* gsel = (gather && !mat) ? sel_l.idx : nullptr;
    const sx_col* src = mat ? LM : nullptr;
    auto fill = [&](auto& pr) {
      pr.partkey = (const int32_t*)(mat ? src[0].data : t->l_partkey.data);
      pr.suppkey = (const int32_t*)(mat ? src[1].data : t->l_suppkey.data);
      pr.qty = (const long long*)(mat ? src[3].data : t->l_quantity.data);
      pr.ext = (const long long*)(mat ? src[4].data : t->l_extendedprice.data);
      pr.disc = (const long long*)(mat ? src[5].data : t->l_discount.data);
      pr.pbm = gather ? nullptr : ht_p->bm;
      pr.pbm_min = ht_p->bm_min;
      pr.pbm_bits = ht_p->bm_bits;
      pr.ps = pt.t[0].slots;
      pr.ps_mask = pt.t[0].mask;
      pr.ps_bits = pt.t[0].pbits;
      pr.sup_bm = ht_s->bm;
      pr.sup_min = ht_s->bm_min;
      pr.sup_n = ht_s->bm_bits;
      pr.sup_val = s_nat;
      pr.ord_bm = o_bm;
      pr.ord_min = o_min;
      pr.ord_n = o_n;
      pr.ord_val = o_date;
      pr.ovf_flag = ctx->d_flags;
      pr.wscan = wscan ? 1 : 0;
    };
    if (okb4) {
      Q9FusedProg<int32_t, 4> pr;
      fill(pr);
      pr.orderkey = (const int32_t*)(mat ? src[2].data : t->l_orderkey.data);
      SX_TRY(gb_run(ctx, pr, plan, gsel, n, 256, gok, goa, &ng));
    } else {
      Q9FusedProg<long long, 8> pr;
      fill(pr);
      pr.orderkey = (const long long*)(mat ? src[2].data : t->l_orderkey.data);
      SX_TRY(gb_run(ctx, pr, plan, gsel, n, 256, gok, goa, &ng));
    }
    // the scanned lineitem rows' referenced columns once (+ selection when gathering, + G output rows)
    pg.set_bytes((4.0 + 4.0 + (gather && !mat ? 4.0 : 0.0) + type_width(t->l_orderkey.type) + 24.0) * n + 24.0 * ng);
    return SX_OK;
  };
  bool fused_done = false;
  if (!ops_plan && ht_p->bm && (okb4 || okb8) && w4(t->l_partkey) && w4(t->l_suppkey) && w8(t->l_quantity) && w8(t->l_extendedprice) && w8(t->l_discount) && w4(t->ps_partkey) && w4(t->ps_suppkey) && w8(t->ps_supplycost) && w4(t->s_suppkey) && w4(t->s_nationkey) && w4(t->o_orderdate)) {
    const sx_status fs = fused();
    if (fs == SX_OK) fused_done = true;
    else if (fs != SX_EUNSUPPORTED) return fs;
    else ctx->err.clear();
  }
  if (!fused_done) {
  // 2. lineitem semi-join P, materialising the columns the plan needs
  sx_col lcols[6] = {t->l_partkey, t->l_suppkey, t->l_orderkey, t->l_quantity, t->l_extendedprice, t->l_discount};
  int32_t lpp[6] = {0, 1, 2, 3, 4, 5};
  sx_sel sel_l;
  sx_col L2[6];
  SX_TRY(sx_hash_probe(ctx, ht_p, lcols, 6, &k0, 1, nullptr, nullptr, 0, SX_SEMI, nullptr, 0, nullptr, 0, lpp, 6, &sel_l,
                       nullptr, L2));
  bag.keep(sel_l);
  bag.keep(L2, 6);
  // 3. partsupp semi-join P, build (ps_partkey, ps_suppkey) -> row
  sx_col pscols[3] = {t->ps_partkey, t->ps_suppkey, t->ps_supplycost};
  sx_sel sel_ps;
  SX_TRY(sx_hash_probe(ctx, ht_p, pscols, 3, &k0, 1, nullptr, nullptr, 0, SX_SEMI, nullptr, 0, nullptr, 0, nullptr, 0,
                       &sel_ps, nullptr, nullptr));
  bag.keep(sel_ps);
  int32_t k01[2] = {0, 1};
  sx_ht* ht_ps;
  SX_TRY(sx_hash_build(ctx, pscols, 3, k01, 2, &sel_ps, nullptr, 0, 1, &ht_ps));
  bag.keep(ht_ps);
  // 4. lineitem'' join partsupp on (partkey, suppkey) -> supplycost
  int32_t bp4[1] = {2}, pp4[5] = {1, 2, 3, 4, 5};
  sx_sel j4p, j4b;
  sx_col L3[6];  // supplycost, suppkey, orderkey, qty, ext, disc
  SX_TRY(sx_hash_probe(ctx, ht_ps, L2, 6, k01, 2, nullptr, nullptr, 0, SX_INNER, pscols, 3, bp4, 1, pp4, 5, &j4p, &j4b, L3));
  bag.keep(j4p);
  bag.keep(j4b);
  bag.keep(L3, 6);
  // 5. join supplier on suppkey -> s_nationkey
  sx_col scols[2] = {t->s_suppkey, t->s_nationkey};
  sx_ht* ht_s;
  SX_TRY(sx_hash_build(ctx, scols, 2, &k0, 1, nullptr, nullptr, 0, 1, &ht_s));
  bag.keep(ht_s);
  int32_t ks = 1, bp5[1] = {1}, pp5[5] = {0, 2, 3, 4, 5};
  sx_sel j5p, j5b;
  sx_col L4[6];  // nationkey, supplycost, orderkey, qty, ext, disc
  SX_TRY(sx_hash_probe(ctx, ht_s, L3, 6, &ks, 1, nullptr, nullptr, 0, SX_INNER, scols, 2, bp5, 1, pp5, 5, &j5p, &j5b, L4));
  bag.keep(j5p);
  bag.keep(j5b);
  bag.keep(L4, 6);
  // 6. join orders on orderkey -> o_orderdate (build the smaller side: lineitem'''s orderkeys)
  int32_t kl = 2;
  sx_ht* ht_l;
  SX_TRY(sx_hash_build(ctx, L4, 6, &kl, 1, nullptr, nullptr, 0, 0, &ht_l));
  bag.keep(ht_l);
  sx_col ocols[2] = {t->o_orderkey, t->o_orderdate};
  int32_t bp6[5] = {0, 1, 3, 4, 5}, pp6[1] = {1};
  sx_sel j6p, j6b;
  sx_col L5[6];  // nationkey, supplycost, qty, ext, disc, orderdate
  SX_TRY(sx_hash_probe(ctx, ht_l, ocols, 2, &k0, 1, nullptr, nullptr, 0, SX_INNER, L4, 6, bp6, 5, pp6, 1, &j6p, &j6b, L5));
  bag.keep(j6p);
  bag.keep(j6b);
  bag.keep(L5, 6);
  // 7. group by (nation, year(o_orderdate)): sum(ext*(100-disc) - supplycost*qty) [scale 4]
  sx_key gk[2] = {{0, SX_KEY_IDENTITY}, {5, SX_KEY_YEAR}};
  sx_agg ga;
  std::memset(&ga, 0, sizeof ga);
  ga.op = SX_SUM;
  ga.value.nterms = 2;
  ga.value.t[0].coef = 1;
  ga.value.t[0].nf = 2;
  ga.value.t[0].f[0] = F(3);
  ga.value.t[0].f[1] = F(4, -1, 100);
  ga.value.t[1].coef = -1;
  ga.value.t[1].nf = 2;
  ga.value.t[1].f[0] = F(1);
  ga.value.t[1].f[1] = F(2);
  if (w4(L5[0]) && w8(L5[1]) && w8(L5[2]) && w8(L5[3]) && w8(L5[4]) && w4(L5[5])) {
    ProfScope pg(ctx, "groupby");
    GbPlan plan;
    SX_TRY(to_dcols_check(ctx, L5, 6));
    SX_TRY(gb_plan(ctx, L5, 6, gk, 2, &ga, 1, nullptr, &plan));
    SX_TRY(check_states(ctx, plan, {ST_SUM}));
    Q9Prog prog{(const int32_t*)L5[0].data, (const long long*)L5[1].data, (const long long*)L5[2].data,
                (const long long*)L5[3].data, (const long long*)L5[4].data, (const int32_t*)L5[5].data, ctx->d_flags};
    SX_TRY(gb_run(ctx, prog, plan, nullptr, L5[0].len, 256, gok, goa, &ng));
    pg.set_bytes(40.0 * L5[0].len + 24.0 * ng);  // 6 columns once + G rows
  } else {
    SX_TRY(sx_groupby_agg(ctx, L5, 6, gk, 2, nullptr, nullptr, 0, &ga, 1, nullptr, 256, gok, goa, &ng));
  }
  }  // operator-at-a-time plan
  bag.keep(gok, 2);
  bag.keep(goa, 1);
  // 8. order by n_name asc (string order of the nation dimension), o_year desc
  std::vector<int> order(25);
  for (int i = 0; i < 25; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [](int a, int b) { return std::strcmp(kNation[a], kNation[b]) < 0; });
  int32_t rank_h[25];
  for (int r = 0; r < 25; ++r) rank_h[order[r]] = r;
  int32_t *rank_d, *rk;
  SX_TRY(alloc(ctx, &rank_d, 25));
  bag.bufs.push_back(rank_d);
  SX_CUDA(cudaMemcpyAsync(rank_d, rank_h, sizeof rank_h, cudaMemcpyHostToDevice, ctx->stream));
  SX_TRY(alloc(ctx, &rk, (size_t)(ng > 0 ? ng : 1)));
  bag.bufs.push_back(rk);
  if (ng > 0) k_lookup_rank<<<(unsigned)((ng + 255) / 256), 256, 0, SX_STREAM(ctx)>>>((const int32_t*)gok[0].data, ng, rank_d, 25, rk);
  SX_CHECK_LAUNCH();
  sx_col scol[2] = {sx_col{SX_I32, 0, ng, rk, nullptr, nullptr}, gok[1]};
  sx_sortkey sks[2] = {{0, 0}, {1, 1}};
  sx_sel perm;
  SX_TRY(sx_sort_topk(ctx, scol, 2, sks, 2, nullptr, -1, &perm));
  bag.keep(perm);
  sx_col all[3] = {gok[0], gok[1], goa[0]};
  std::vector<std::vector<uint8_t>> h;
  SX_TRY(fetch_rows(ctx, bag, all, 3, perm, h));
  if (perm.len > cap) return set_err(ctx, SX_EINVAL, "Q9: %lld rows > cap", (long long)perm.len);
  for (int64_t i = 0; i < perm.len; ++i) {
    out[i].nationkey = at<int32_t>(h[0], i);
    out[i].o_year = at<int32_t>(h[1], i);
    out[i].sum_profit = i128_at(h[2], i);
  }
  *nrows = perm.len;
  return SX_OK;
}

// ------------------------------------------------------------------------------------- Q18
SX_EXPORT sx_status sx_tpch_q18(sx_ctx* ctx, const sx_tpch_tables* t, const sx_tpch_params* p, sx_q18_row* out,
                                int64_t cap, int64_t* nrows) {
  if (!ctx || !t || !p || !nrows) return SX_EINVAL;
  *nrows = 0;
  ProfScope ps(ctx, "Q18");
  Bag bag(ctx);
  int32_t k0 = 0;
  // 1. subquery: l_orderkey groups with sum(l_quantity) > QUANTITY
  sx_col lcols[2] = {t->l_orderkey, t->l_quantity};
  sx_key gk = {0, SX_KEY_IDENTITY};
  sx_agg ga = A(SX_SUM, E1(1, {F(1)}));
  sx_having hv = {0, SX_GT, p->q18_qty_gt, 0};
  sx_col gok[1], goa[1];
  int64_t ng = 0;
  if (w8(t->l_quantity) && (w4(t->l_orderkey) || w8(t->l_orderkey))) {
    ProfScope pg(ctx, "groupby");
    GbPlan plan;
    SX_TRY(to_dcols_check(ctx, lcols, 2));
    SX_TRY(gb_plan(ctx, lcols, 2, &gk, 1, &ga, 1, &hv, &plan));
    SX_TRY(check_states(ctx, plan, {ST_SUM}));
    if (w4(t->l_orderkey)) {
      Q18Prog<int32_t> prog{(const int32_t*)t->l_orderkey.data, (const long long*)t->l_quantity.data, ctx->d_flags};
      SX_TRY(gb_run(ctx, prog, plan, nullptr, t->l_orderkey.len, t->o_orderkey.len, gok, goa, &ng));
    } else {
      Q18Prog<long long> prog{(const long long*)t->l_orderkey.data, (const long long*)t->l_quantity.data, ctx->d_flags};
      SX_TRY(gb_run(ctx, prog, plan, nullptr, t->l_orderkey.len, t->o_orderkey.len, gok, goa, &ng));
    }
    // key + qty once, and the per-order state (one row per order: key + sum) written and read once
    const double kw = type_width(t->l_orderkey.type);
    pg.set_bytes((kw + 8) * t->l_orderkey.len + 2.0 * (kw + 8) * t->o_orderkey.len);
  } else {
    SX_TRY(sx_groupby_agg(ctx, lcols, 2, &gk, 1, nullptr, nullptr, 0, &ga, 1, &hv, t->o_orderkey.len, gok, goa, &ng));
  }
  bag.keep(gok, 1);
  bag.keep(goa, 1);
  // 2+3 by sorted-PK lookups (default; SX_Q18_JOIN=hash forces the hash joins below): the ~6.4e3
  //    qualifying orderkeys are looked up in o_orderkey and their custkeys in c_custkey (both
  //    tables in key order) instead of scanning 1.5e8 orders and 1.5e7 customers
  const bool hash_joins = getenv("SX_Q18_JOIN") && std::strcmp(getenv("SX_Q18_JOIN"), "hash") == 0;
  if (!hash_joins) {
    ProfScope pl(ctx, "probe_inner");
    sx_col R[5];
    bool found = false;
    // one fused kernel (SX_Q18_JOIN=lookup: the separate lookups + gathers)
    const bool sep = getenv("SX_Q18_JOIN") && std::strcmp(getenv("SX_Q18_JOIN"), "lookup") == 0;
    if (!sep) {
      R[0] = goa[0];
      SX_TRY(q18_join(ctx, bag, t, gok[0], R, &found));
    }
    int32_t* orow = nullptr;
    bool ok = false;
    if (!found) SX_TRY(sorted_lookup(ctx, bag, t->o_orderkey, gok[0], &orow, &ok));
    if (!found && ok) {
      const sx_sel os{ng, orow};
      sx_col oc[4] = {t->o_orderkey, t->o_custkey, t->o_orderdate, t->o_totalprice};
      R[0] = goa[0];
      for (int c = 0; c < 4; ++c) {
        SX_TRY(sx_gather(ctx, &oc[c], &os, &R[1 + c]));
        bag.keep(R[1 + c]);
      }
      int32_t* crow;
      SX_TRY(sorted_lookup(ctx, bag, t->c_custkey, R[2], &crow, &found));  // every order's customer exists
    }
    pl.set_bytes(ng * (2.0 * type_width(t->o_orderkey.type) + 4.0 + 4 + 4 + 8 + 4 + 4));
    if (found) {
      sx_col scols[3] = {R[4], R[3], R[1]};
      sx_sortkey sks[3] = {{0, 1}, {1, 0}, {2, 0}};
      sx_sel perm;
      SX_TRY(sx_sort_topk(ctx, scols, 3, sks, 3, nullptr, p->q18_limit, &perm));
      bag.keep(perm);
      std::vector<std::vector<uint8_t>> h;
      SX_TRY(fetch_rows(ctx, bag, R, 5, perm, h));
      if (perm.len > cap) return set_err(ctx, SX_EINVAL, "Q18: %lld rows > cap", (long long)perm.len);
      for (int64_t i = 0; i < perm.len; ++i) {
        out[i].o_orderkey = key_at(h[1], R[1].type, i);
        out[i].c_custkey = at<int32_t>(h[2], i);
        out[i].o_orderdate = at<int32_t>(h[3], i);
        out[i].o_totalprice = at<int64_t>(h[4], i);
        out[i].sum_qty = i128_at(h[0], i);
      }
      *nrows = perm.len;
      return SX_OK;
    }
  }
  // 2. orders with o_orderkey in that set; carry sum(l_quantity) from the group-by (equal to the
  //    literal re-aggregation over the joined lineitems; reading for Q18)
  sx_col big[2] = {gok[0], goa[0]};
  sx_ht* ht_b;
  SX_TRY(sx_hash_build(ctx, big, 2, &k0, 1, nullptr, nullptr, 0, 1, &ht_b));
  bag.keep(ht_b);
  sx_col ocols[4] = {t->o_orderkey, t->o_custkey, t->o_orderdate, t->o_totalprice};
  int32_t bp[1] = {1}, pp[4] = {0, 1, 2, 3};
  sx_sel jp, jb;
  sx_col C[5];  // sum_qty, orderkey, custkey, orderdate, totalprice
  SX_TRY(sx_hash_probe(ctx, ht_b, ocols, 4, &k0, 1, nullptr, nullptr, 0, SX_INNER, big, 2, bp, 1, pp, 4, &jp, &jb, C));
  bag.keep(jp);
  bag.keep(jb);
  bag.keep(C, 5);
  // 3. join customer on custkey (build the small candidate side)
  int32_t kc = 2;
  sx_ht* ht_c;
  SX_TRY(sx_hash_build(ctx, C, 5, &kc, 1, nullptr, nullptr, 0, 0, &ht_c));
  bag.keep(ht_c);
  sx_col cc[1] = {t->c_custkey};
  int32_t bp3[5] = {0, 1, 2, 3, 4};
  sx_sel j3p, j3b;
  sx_col R[5];
  SX_TRY(sx_hash_probe(ctx, ht_c, cc, 1, &k0, 1, nullptr, nullptr, 0, SX_INNER, C, 5, bp3, 5, nullptr, 0, &j3p, &j3b, R));
  bag.keep(j3p);
  bag.keep(j3b);
  bag.keep(R, 5);
  // 4. order by o_totalprice desc, o_orderdate asc, o_orderkey asc (reading R6); limit
  sx_col scols[3] = {R[4], R[3], R[1]};
  sx_sortkey sks[3] = {{0, 1}, {1, 0}, {2, 0}};
  sx_sel perm;
  SX_TRY(sx_sort_topk(ctx, scols, 3, sks, 3, nullptr, p->q18_limit, &perm));
  bag.keep(perm);
  std::vector<std::vector<uint8_t>> h;
  SX_TRY(fetch_rows(ctx, bag, R, 5, perm, h));
  if (perm.len > cap) return set_err(ctx, SX_EINVAL, "Q18: %lld rows > cap", (long long)perm.len);
  for (int64_t i = 0; i < perm.len; ++i) {
    out[i].o_orderkey = key_at(h[1], R[1].type, i);
    out[i].c_custkey = at<int32_t>(h[2], i);
    out[i].o_orderdate = at<int32_t>(h[3], i);
    out[i].o_totalprice = at<int64_t>(h[4], i);
    out[i].sum_qty = i128_at(h[0], i);
  }
  *nrows = perm.len;
  return SX_OK;
}

// ------------------------------------------------------------------------------- host upload
namespace {
constexpr int kTpchCols = (int)(sizeof(sx_tpch_tables) / sizeof(sx_col));
}

SX_EXPORT sx_status sx_tpch_upload(sx_ctx* ctx, const sx_tpch_tables* host, sx_tpch_tables* dev) {
  if (!ctx || !host || !dev) return SX_EINVAL;
  std::memset(dev, 0, sizeof *dev);
  const sx_col* hc = (const sx_col*)host;
  sx_col* dc = (sx_col*)dev;
  for (int i = 0; i < kTpchCols; ++i) {
    const sx_col& h = hc[i];
    sx_col& d = dc[i];
    d = h;
    d.data = nullptr;
    d.offsets = nullptr;
    if (h.len <= 0 && h.type != SX_STR) continue;
    size_t bytes;
    if (h.type == SX_STR) {
      if (!h.offsets) continue;
      bytes = (size_t)h.offsets[h.len];  // host offsets
      int64_t* doff;
      sx_status st = alloc(ctx, &doff, (size_t)h.len + 1);
      if (st != SX_OK) { sx_tpch_tables_free(ctx, dev); return st; }
      d.offsets = doff;
      SX_CUDA(cudaMemcpyAsync(doff, h.offsets, sizeof(int64_t) * (h.len + 1), cudaMemcpyHostToDevice, ctx->stream));
    } else {
      bytes = (size_t)h.len * type_width(h.type);
    }
    char* buf;
    sx_status st = alloc(ctx, &buf, bytes + 16);
    if (st != SX_OK) { sx_tpch_tables_free(ctx, dev); return st; }
    d.data = buf;
    if (bytes) SX_CUDA(cudaMemcpyAsync(buf, h.data, bytes, cudaMemcpyHostToDevice, ctx->stream));
  }
  return SX_OK;
}

SX_EXPORT void sx_tpch_tables_free(sx_ctx* ctx, sx_tpch_tables* dev) {
  if (!ctx || !dev) return;
  sx_col* dc = (sx_col*)dev;
  for (int i = 0; i < kTpchCols; ++i) {
    if (dc[i].data) dfree(ctx, (void*)dc[i].data);
    if (dc[i].type == SX_STR && dc[i].offsets) dfree(ctx, (void*)dc[i].offsets);
    dc[i].data = nullptr;
    dc[i].offsets = nullptr;
  }
}
