// gb_host.cuh — group-by planning (agg -> state mapping, slot layout), the host driver
// (table sizing, strategy, retry on a full table) and result extraction/emission.
#pragma once
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "compact.cuh"
#include "groupby.cuh"
#include "radix.cuh"
#include "ring.cuh"

namespace sx {

struct GbPlan {
  Layout L;
  sx_expr state_expr[kMaxStates];
  int nkeys;
  int key_types[2];
  int key_fn[2];
  int out_key_type[2];
  int naggs;
  int agg_op[SX_MAX_AGGS];
  int agg_state[SX_MAX_AGGS];   // SUM/MIN/MAX/AVG: state holding the value
  int agg_scale[SX_MAX_AGGS];
  int count_state;              // -1 if none
  int has_having;
  sx_having hv;
};

inline bool expr_equal(const sx_expr& a, const sx_expr& b) {
  if (a.nterms != b.nterms) return false;
  for (int t = 0; t < a.nterms; ++t) {
    if (a.t[t].coef != b.t[t].coef || a.t[t].nf != b.t[t].nf) return false;
    for (int f = 0; f < a.t[t].nf; ++f)
      if (a.t[t].f[f].col != b.t[t].f[f].col || a.t[t].f[f].mul != b.t[t].f[f].mul || a.t[t].f[f].add != b.t[t].f[f].add)
        return false;
  }
  return true;
}

inline sx_status gb_plan(sx_ctx* ctx, const sx_col* cols, int ncols, const sx_key* keys, int nkeys, const sx_agg* aggs,
                         int naggs, const sx_having* having, GbPlan* P) {
  std::memset(P, 0, sizeof(*P));
  if (nkeys < 0 || nkeys > 2) return set_err(ctx, SX_EINVAL, "nkeys %d (0..2)", nkeys);
  if (naggs < 0 || naggs > SX_MAX_AGGS) return set_err(ctx, SX_EINVAL, "naggs %d (0..%d)", naggs, SX_MAX_AGGS);
  P->nkeys = nkeys;
  int kbits_total = 0;
  for (int k = 0; k < nkeys; ++k) {
    int c = keys[k].col;
    if (c < 0 || c >= ncols) return set_err(ctx, SX_EINVAL, "key column %d out of range", c);
    int t = cols[c].type;
    if (t != SX_U8 && t != SX_I32 && t != SX_DATE32 && t != SX_I64) return set_err(ctx, SX_ETYPE, "key type %d", t);
    if (keys[k].fn == SX_KEY_YEAR && t != SX_DATE32) return set_err(ctx, SX_ETYPE, "SX_KEY_YEAR needs a DATE32 key");
    if (keys[k].fn != SX_KEY_IDENTITY && keys[k].fn != SX_KEY_YEAR) return set_err(ctx, SX_EINVAL, "key fn %d", keys[k].fn);
    P->key_types[k] = t;
    P->key_fn[k] = keys[k].fn;
    P->out_key_type[k] = keys[k].fn == SX_KEY_YEAR ? SX_I32 : t;
    int b = keys[k].fn == SX_KEY_YEAR ? 32 : key_bits(t);
    if (nkeys == 2 && b > 32) return set_err(ctx, SX_ETYPE, "two-column group keys must each be <= 32 bits");
    kbits_total += b;
  }
  Layout& L = P->L;
  // two keys are packed as (k0 << 32) | k1, so they always need the 8-byte key field
  L.key_bytes = nkeys == 0 ? 0 : (nkeys == 1 && kbits_total <= 32 ? 4 : 8);
  // states
  int nst = 0;
  P->count_state = -1;
  auto add_state = [&](int kind, const sx_expr* e) -> int {
    for (int s = 0; s < nst; ++s)
      if (L.kind[s] == kind && (kind == ST_COUNT || expr_equal(P->state_expr[s], *e))) return s;
    L.kind[nst] = kind;
    if (e) P->state_expr[nst] = *e;
    else std::memset(&P->state_expr[nst], 0, sizeof(sx_expr));
    return nst++;
  };
  P->naggs = naggs;
  for (int a = 0; a < naggs; ++a) {
    int op = aggs[a].op;
    if (op != SX_COUNT) SX_TRY(check_expr(ctx, cols, ncols, aggs[a].value));
    if (nst >= kMaxStates - 1 && op == SX_AVG) return set_err(ctx, SX_EINVAL, "too many aggregate states");
    P->agg_op[a] = op;
    P->agg_scale[a] = aggs[a].scale;
    switch (op) {
      case SX_SUM: P->agg_state[a] = add_state(ST_SUM, &aggs[a].value); break;
      case SX_COUNT: P->agg_state[a] = P->count_state = add_state(ST_COUNT, nullptr); break;
      case SX_MIN: P->agg_state[a] = add_state(ST_MIN, &aggs[a].value); break;
      case SX_MAX: P->agg_state[a] = add_state(ST_MAX, &aggs[a].value); break;
      case SX_AVG:
        P->agg_state[a] = add_state(ST_SUM, &aggs[a].value);
        P->count_state = add_state(ST_COUNT, nullptr);
        if (aggs[a].scale < 0 || aggs[a].scale > 18) return set_err(ctx, SX_EINVAL, "avg scale %d", aggs[a].scale);
        break;
      default: return set_err(ctx, SX_EINVAL, "aggregate op %d", op);
    }
    if (nst > kMaxStates) return set_err(ctx, SX_EINVAL, "too many aggregate states");
  }
  if (nkeys == 0 && P->count_state < 0) {
    if (nst >= kMaxStates) return set_err(ctx, SX_EINVAL, "too many aggregate states");
    P->count_state = add_state(ST_COUNT, nullptr);
  }
  L.nst = nst;
  // byte layout: key, then 8-byte fields, then 4-byte sum-hi fields (first one packed next to a 4-byte key)
  int off = L.key_bytes;
  int n4 = 0;
  for (int s = 0; s < nst; ++s) n4 += L.kind[s] == ST_SUM;
  int first4 = -1;
  if (L.key_bytes == 4 && n4 > 0) {
    for (int s = 0; s < nst && first4 < 0; ++s)
      if (L.kind[s] == ST_SUM) first4 = s;
    L.off4[first4] = 4;
    off = 8;
  }
  off = (off + 7) & ~7;
  for (int s = 0; s < nst; ++s) { L.off8[s] = off; off += 8; }
  for (int s = 0; s < nst; ++s)
    if (L.kind[s] == ST_SUM && s != first4) { L.off4[s] = off; off += 4; }
  L.slot_bytes = (off + 7) & ~7;
  if (L.slot_bytes == 0) L.slot_bytes = 8;
  P->has_having = having != nullptr;
  if (having) {
    if (having->agg < 0 || having->agg >= naggs) return set_err(ctx, SX_EINVAL, "having agg index out of range");
    if (P->agg_op[having->agg] == SX_AVG) return set_err(ctx, SX_EUNSUPPORTED, "HAVING on AVG");
    if (having->op < SX_LT || having->op > SX_BETWEEN) return set_err(ctx, SX_EINVAL, "having op");
    P->hv = *having;
  }
  return SX_OK;
}

// ------------------------------------------------------------------------ extraction
struct SlotFn {
  const uint8_t* slots;
  uint64_t cap;     // slots per (sub-)table; sub-table s occupies [s*(cap+1), (s+1)*(cap+1)), side slot last
  int slot_bytes, key_bytes;
  const int* side_used;  // one flag per sub-table
  int nsub;
  int has_having, hv_kind, hv_op, hv_off8, hv_off4;
  int64_t hv_lo, hv_hi;
  // HAVING on a state given by value: SUM as {lo, hi} 96-bit, else the 8-byte slot word.
  __device__ __forceinline__ bool hv_ok_state(unsigned long long lo, int32_t hi) const {
    if (!has_having) return true;
    if (hv_kind == ST_SUM) {
      __int128 v = ((__int128)hi << 64) | (__int128)lo;
      __int128 l = hv_lo, h = hv_hi;
      switch (hv_op) {
        case SX_LT: return v < l;
        case SX_LE: return v <= l;
        case SX_GT: return v > l;
        case SX_GE: return v >= l;
        case SX_EQ: return v == l;
        case SX_NE: return v != l;
        default: return l <= v && v <= h;
      }
    }
    int64_t v = hv_kind == ST_COUNT ? (int64_t)lo
              : hv_kind == ST_MAX ? (int64_t)(lo ^ 0x8000000000000000ull)
                                  : (int64_t)(~lo ^ 0x8000000000000000ull);
    return cmp(hv_op, v, hv_lo, hv_hi);
  }
  __device__ __forceinline__ bool hv_ok(const uint8_t* p) const {
    if (!has_having) return true;
    if (hv_kind == ST_SUM) {
      __int128 v = ((__int128)(*(const int*)(p + hv_off4)) << 64) | (__int128)(*(const unsigned long long*)(p + hv_off8));
      __int128 lo = hv_lo, hi = hv_hi;
      switch (hv_op) {
        case SX_LT: return v < lo;
        case SX_LE: return v <= lo;
        case SX_GT: return v > lo;
        case SX_GE: return v >= lo;
        case SX_EQ: return v == lo;
        case SX_NE: return v != lo;
        default: return lo <= v && v <= hi;
      }
    }
    unsigned long long u = *(const unsigned long long*)(p + hv_off8);
    int64_t v = hv_kind == ST_COUNT ? (int64_t)u
              : hv_kind == ST_MAX ? (int64_t)(u ^ 0x8000000000000000ull)
                                  : (int64_t)(~u ^ 0x8000000000000000ull);
    return cmp(hv_op, v, hv_lo, hv_hi);
  }
  template <int ITEMS>
  __device__ __forceinline__ void eval(const int32_t (&row)[ITEMS], const bool (&valid)[ITEMS], bool (&alive)[ITEMS],
                                       int32_t (&aux)[ITEMS]) const {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      bool occ = false;
      if (valid[i]) {
        const uint8_t* p = slots + (uint64_t)row[i] * slot_bytes;
        if (key_bytes == 0) occ = true;
        else if (nsub == 1 ? (uint64_t)row[i] == cap : (uint64_t)row[i] % (cap + 1) == cap)
          occ = side_used[nsub == 1 ? 0 : (uint64_t)row[i] / (cap + 1)] != 0;
        else if (key_bytes == 4) occ = *(const unsigned*)p != 0u;
        else occ = *(const unsigned long long*)p != 0ull;
        occ = occ && hv_ok(p);
      }
      alive[i] = occ;
    }
  }
};

// ------------------------------------------------------------------ K10r: owned runs + HAVING
// Sorted-input group-by with the HAVING predicate pushed into the aggregation (Q18's subquery:
// 1.5e8 orderkey runs of 1-7 lineitems, ~6.4e3 survive).  Each thread takes kRunItems consecutive
// rows and OWNS the groups whose first row lies among them; it sums each owned group in registers
// (96-bit), reading past its rows while the key continues (at most kRunAhead rows, else the host
// falls back), applies HAVING and appends only the survivors (atomic cursor).  No per-group state
// is written for the groups that fail HAVING and no group numbering pass is needed; a key that
// decreases anywhere flags the input as unsorted (host falls back to hashing).
constexpr int kRunAhead = 64;
constexpr int kRunOwnRows = 8;   // rows per thread in k_runs_own_dense (16 measured slower: 4.35 vs 3.44 ms)

template <class P, class = void>
struct runs_dense : std::false_type {};
template <class P>
struct runs_dense<P, std::void_t<decltype(P::kDenseRuns)>> : std::integral_constant<bool, P::kMaxNst == 1> {};

template <class P>
__device__ __forceinline__ void runs_acc(int kd, int64_t v, unsigned long long& lo, int32_t& hi) {
  if (kd == ST_SUM || kd == ST_COUNT) {
    const unsigned long long nl = lo + (unsigned long long)v;
    const bool cy = nl < lo, neg = v < 0;
    if (kd == ST_SUM && cy != neg) hi += cy ? 1 : -1;
    lo = nl;
  } else {
    const unsigned long long u = kd == ST_MIN ? ~order_u(v) : order_u(v);
    lo = u > lo ? u : lo;
  }
}

template <class P>
__global__ void __launch_bounds__(kBlock) k_runs_own(const __grid_constant__ P prog, int64_t n,
                                                     const __grid_constant__ Layout L, const __grid_constant__ SlotFn hv,
                                                     uint8_t* __restrict__ out, int64_t cap_out,
                                                     unsigned long long* cursor, int* flags) {
  constexpr int NST = P::kMaxNst;
  constexpr int R = kRunItems;
  static_assert(NST <= 2, "k_runs_own keeps every state of a group in registers");
  bool ovf = false;
  for (int64_t r0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * R; r0 < n;
       r0 += (int64_t)gridDim.x * blockDim.x * R) {
    int32_t row[R];
    bool valid[R], alive[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      valid[i] = r0 + i < n;
      alive[i] = valid[i];
      row[i] = valid[i] ? (int32_t)(r0 + i) : 0;
    }
    uint64_t key[R], pk[1];
    int64_t v[NST][R];
    if constexpr (runs_dense<P>::value) {  // one-state programs with 128-bit row loads
      prog.template runs_dense<R>(r0, n, key, v[0]);
    } else {
      typename P::template Cache<R> cache;
      prog.template where_keys<R>(row, alive, key, cache);
#pragma unroll
      for (int a = 0; a < NST; ++a) {
        if (a >= L.nst) break;
        if (prog.kind(a, L) == ST_COUNT) {
#pragma unroll
          for (int i = 0; i < R; ++i) v[a][i] = 1;
        } else {
          prog.template state<R>(a, row, alive, cache, v[a], ovf);
        }
      }
    }
    int32_t prow[1] = {(int32_t)(r0 - 1)};
    bool pv[1] = {r0 > 0};
    prog.template keys_only<1>(prow, pv, pk);
    bool bad = false;
    unsigned long long lo[NST];
    int32_t hi[NST];
    bool owned = false;
    uint64_t gkey = 0;
    uint64_t prev = pk[0];
    bool has_prev = pv[0];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      if (!valid[i]) break;
      const bool head = !has_prev || key[i] != prev;
      bad |= has_prev && (int64_t)key[i] < (int64_t)prev;
      if (head) {
        owned = true;
        gkey = key[i];
#pragma unroll
        for (int a = 0; a < NST; ++a) { lo[a] = 0; hi[a] = 0; }
      }
      if (owned) {
#pragma unroll
        for (int a = 0; a < NST; ++a)
          if (a < L.nst) runs_acc<P>(prog.kind(a, L), v[a][i], lo[a], hi[a]);
      }
      prev = key[i];
      has_prev = true;
      // does the owned group end at row i?
      bool ends;
      if (i + 1 < R && valid[i + 1]) {
        ends = key[i + 1] != key[i];
      } else if (r0 + i + 1 >= n) {
        ends = true;
      } else if (owned) {  // read ahead into the following rows while the key continues
        ends = true;
        int64_t r = r0 + i + 1;
        int steps = 0;
        for (; r < n && steps < kRunAhead; ++r, ++steps) {
          int32_t rr[1] = {(int32_t)r};
          bool al[1] = {true};
          uint64_t kk[1];
          typename P::template Cache<1> c1;
          prog.template where_keys<1>(rr, al, kk, c1);
          if (kk[0] != gkey) {
            bad |= (int64_t)kk[0] < (int64_t)gkey;
            break;
          }
#pragma unroll
          for (int a = 0; a < NST; ++a) {
            if (a >= L.nst) break;
            int64_t vv[1] = {1};
            if (prog.kind(a, L) != ST_COUNT) prog.template state<1>(a, rr, al, c1, vv, ovf);
            runs_acc<P>(prog.kind(a, L), vv[0], lo[a], hi[a]);
          }
        }
        if (steps == kRunAhead && r < n) atomicExch(flags + 1, 1);  // a long run: host falls back
      } else {
        ends = false;
      }
      if (ends && owned) {
        alignas(16) uint8_t buf[64];
        if (L.key_bytes == 4) *(unsigned*)buf = (unsigned)gkey;
        else *(unsigned long long*)buf = gkey;
#pragma unroll
        for (int a = 0; a < NST; ++a) {
          if (a >= L.nst) break;
          *(unsigned long long*)(buf + L.off8[a]) = lo[a];
          if (L.kind[a] == ST_SUM) *(int*)(buf + L.off4[a]) = hi[a];
        }
        if (hv.hv_ok(buf)) {
          const unsigned long long pos = atomicAdd(cursor, 1ull);
          if ((int64_t)pos < cap_out) {
            uint8_t* d = out + pos * L.slot_bytes;
            for (int b = 0; b < L.slot_bytes; b += 4) *(unsigned*)(d + b) = *(const unsigned*)(buf + b);
          }
        }
        owned = false;
      }
    }
    if (bad) atomicExch(flags, 1);
  }
  if (ovf) atomicExch(prog.ovf_flag, 1);
}

// Dense variant of K10r for one-state programs with runs_dense (Q18): a thread loads its 8 rows
// with 128-bit loads; the rows at its start that continue the previous thread's last group (its
// "lead") are summed locally and handed to the previous lane with one shuffle, so a run that
// crosses a thread boundary is finished without reloading rows (lane 31, and runs longer than the
// next thread's 8 rows, read ahead row by row).  4 CTAs per SM (64 registers, no spills):
// 2.91 vs 3.42 ms for Q18 at SF100 with 3 — the loop is issue/latency bound, more warps help.
template <class P>
__global__ void __launch_bounds__(kBlock, 4) k_runs_own_dense(const __grid_constant__ P prog, int64_t n,
                                                           const __grid_constant__ Layout L,
                                                           const __grid_constant__ SlotFn hv, uint8_t* __restrict__ out,
                                                           int64_t cap_out, unsigned long long* cursor, int* flags) {
  constexpr int R = kRunOwnRows;
  bool bad = false, ovf = false;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * R;
  // HAVING and the slot layout in registers (not re-read from the parameter bank in every branch)
  const int hv_op = hv.hv_op, kb = L.key_bytes, o8 = L.off8[0], o4 = L.off4[0], sb = L.slot_bytes;
  const long long hv_lo = hv.hv_lo, hv_hi = hv.hv_hi;
  const bool has_hv = hv.has_having != 0;
  auto passes = [&](unsigned long long lo, int32_t hi) -> bool {
    if (!has_hv) return true;
    if (hi == ((long long)lo < 0 ? -1 : 0)) return cmp(hv_op, (long long)lo, hv_lo, hv_hi);  // fits int64
    return hv.hv_ok_state(lo, hi);
  };
  auto emit = [&](uint64_t gk, unsigned long long lo, int32_t hi) {
    const unsigned long long pos = atomicAdd(cursor, 1ull);
    if ((int64_t)pos < cap_out) {
      uint8_t* d = out + pos * sb;
      if (kb == 4) *(unsigned*)d = (unsigned)gk;
      else *(unsigned long long*)d = gk;
      *(unsigned long long*)(d + o8) = lo;
      *(int*)(d + o4) = hi;
    }
  };
  // all lanes of a warp run the same number of iterations (shuffles below)
  for (int64_t wbase = (blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31)) * R; wbase < n; wbase += stride) {
    const int64_t r0 = wbase + (int64_t)lane * R;
    uint64_t key[R];
    int64_t v[R];
    prog.template runs_dense<R>(r0, n, key, v);
    const int m = (int)max((int64_t)0, min((int64_t)R, n - r0));
    uint64_t prev = 0;
    const bool has_prev = r0 > 0 && r0 <= n;
    if (has_prev) {
      int32_t pr[1] = {(int32_t)(r0 - 1)};
      bool pv[1] = {true};
      uint64_t pk[1];
      prog.template keys_only<1>(pr, pv, pk);
      prev = pk[0];
    }
    // |v| < 2^40 for all rows (TPC-H quantities are < 2^13): the window's partial sums are exact
    // in int64 and the 96-bit carry tracking is only needed once per emitted group
    unsigned long long big = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) big |= (unsigned long long)(v[i] < 0 ? -v[i] : v[i]);
    // (the vote must run on every lane: `(big >> 40) == 0 && __all_sync(...)` short-circuited it on
    // the lanes holding a wide value and hung the warp)
    const bool small = __all_sync(kFull, (big >> 40) == 0);
    // lead: leading rows continuing the previous thread's last group
    unsigned long long lead_lo = 0;
    int32_t lead_hi = 0;
    int lead = 0;
    bool in_lead = has_prev;
    if (small) {
      long long acc = 0;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        if (i < m && in_lead && key[i] == prev) {
          acc += v[i];
          ++lead;
        } else {
          in_lead = false;
        }
      }
      lead_lo = (unsigned long long)acc;
      lead_hi = acc < 0 ? -1 : 0;
    } else {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        if (i < m && in_lead && key[i] == prev) {
          runs_acc<P>(ST_SUM, v[i], lead_lo, lead_hi);
          ++lead;
        } else {
          in_lead = false;
        }
      }
    }
    // the next thread's lead continues my last group
    const unsigned long long nx_lo = __shfl_down_sync(kFull, lead_lo, 1);
    const int32_t nx_hi = __shfl_down_sync(kFull, lead_hi, 1);
    const int nx_len = __shfl_down_sync(kFull, lead, 1);
    // my groups: heads at rows i >= lead (a head: first row, or key change)
    unsigned long long lo = 0;
    int32_t hi = 0;
    bool open = false;
    uint64_t gk = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      if (i >= m || i < lead) continue;
      const uint64_t pk = i > 0 ? key[i - 1] : prev;
      const bool head = !(i > 0 || has_prev) || key[i] != pk;
      bad |= (i > 0 || has_prev) && (int64_t)key[i] < (int64_t)pk;
      if (head) {
        if (open && small) {  // the int64 partial as 96 bits
          hi = (long long)lo < 0 ? -1 : 0;
        }
        if (open && passes(lo, hi)) emit(gk, lo, hi);  // the previous owned group ended at row i - 1
        open = true;
        gk = key[i];
        lo = 0;
        hi = 0;
      }
      if (small) lo = (unsigned long long)((long long)lo + v[i]);
      else runs_acc<P>(ST_SUM, v[i], lo, hi);
    }
    if (open) {  // my last owned group: finish it with the following rows
      if (small) hi = (long long)lo < 0 ? -1 : 0;
      const int64_t nxt = r0 + R;  // first row of the next thread
      if (nxt < n) {
        bool more;
        int64_t r;
        if (lane < 31) {
          // the next lane's lead (same warp) continues this group
          const unsigned long long nl = lo + nx_lo;
          const int carry = nl < lo ? 1 : 0;
          hi += nx_hi + carry;
          lo = nl;
          more = nx_len == R;
          r = nxt + R;
        } else {
          more = true;
          r = nxt;
        }
        int steps = 0;
        for (; more && r < n && steps < kRunAhead; ++r, ++steps) {  // rare: scalar continuation
          int32_t rr[1] = {(int32_t)r};
          bool al[1] = {true};
          uint64_t kk[1];
          typename P::template Cache<1> c1;
          prog.template where_keys<1>(rr, al, kk, c1);
          if (kk[0] != gk) break;
          int64_t vv[1];
          prog.template state<1>(0, rr, al, c1, vv, ovf);
          runs_acc<P>(ST_SUM, vv[0], lo, hi);
        }
        if (more && steps == kRunAhead && r < n) atomicExch(flags + 1, 1);
      }
      if (passes(lo, hi)) emit(gk, lo, hi);
    }
  }
  if (bad) atomicExch(flags, 1);
  if (ovf) atomicExch(prog.ovf_flag, 1);
}

// K10l: lean owned runs for 32-bit keys and one int64 SUM whose values are < 2^40 in magnitude
// (programs with kLeanRuns: Q18).  Same ownership rule as K10r (a thread owns the groups whose
// first row lies among its 8 rows; the next lane's leading rows finish its last group), but the
// per-row work is branch-free 32-bit key compares and selects with int64 run sums: K10r's
// generic form executes ~100 instructions per row (round-1 ncu: 1.93e9 warp instructions for
// 6e8 rows, issue-bound at 2.8 ms).  The previous key comes from the neighbouring lane.  Rare
// cases go to flags: flags[0] a decreasing key (unsorted: host hashes), flags[1] a value >= 2^40
// or a run longer than kRunAhead rows past its thread (host reruns K10r).
template <class P, class = void>
struct has_lean_runs : std::false_type {};
template <class P>
struct has_lean_runs<P, std::void_t<decltype(P::kLeanRuns)>> : std::integral_constant<bool, P::kLeanRuns> {};

template <class P>
__global__ void __launch_bounds__(kBlock, 4) k_runs_lean(const __grid_constant__ P prog, int64_t n,
                                                      const __grid_constant__ Layout L,
                                                      const __grid_constant__ SlotFn hv, uint8_t* __restrict__ out,
                                                      int64_t cap_out, unsigned long long* cursor, int* flags) {
  constexpr int R = 8;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * R;
  const int hv_op = hv.hv_op, o8 = L.off8[0], o4 = L.off4[0], sb = L.slot_bytes;
  const long long hv_lo = hv.hv_lo, hv_hi = hv.hv_hi;
  unsigned bad = 0, wide = 0;
  auto emit = [&](int32_t gk, long long s) {
    if (!cmp(hv_op, s, hv_lo, hv_hi)) return;
    const unsigned long long pos = atomicAdd(cursor, 1ull);
    if ((int64_t)pos < cap_out) {
      uint8_t* d = out + pos * sb;
      *(int32_t*)d = gk;
      *(long long*)(d + o8) = s;
      *(int*)(d + o4) = s < 0 ? -1 : 0;
    }
  };
  // The next window's 8 keys + 8 values per lane are copied into this thread's slot of a
  // shared double buffer by cp.async while the current window is aggregated (ncu: the register
  // version was long-scoreboard bound at 4.0 TB/s; loading the next window into registers
  // measured slower, 2.35 vs 1.98 ms — the extra registers cost a CTA per SM).
  __shared__ __align__(16) int32_t s_k[2][kBlock * R];
  __shared__ __align__(16) long long s_v[2][kBlock * R];
  const int32_t* gk = prog.lean_kp();
  const long long* gv = prog.lean_vp();
  auto issue = [&](int64_t rr, int b) {  // whole 8-row chunks only (the tail loads directly)
    if (rr + R <= n) {
      const unsigned sk = (unsigned)__cvta_generic_to_shared(&s_k[b][threadIdx.x * R]);
      const unsigned sv = (unsigned)__cvta_generic_to_shared(&s_v[b][threadIdx.x * R]);
#pragma unroll
      for (int j = 0; j < 2; ++j)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sk + 16 * j), "l"(gk + rr + 4 * j));
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sv + 16 * j), "l"(gv + rr + 2 * j));
    }
    asm volatile("cp.async.commit_group;");
  };
  int buf = 0;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31)) * R;
  if (w0 < n) issue(w0 + (int64_t)lane * R, 0);
  for (int64_t wbase = w0; wbase < n; wbase += stride) {
    const int64_t r0 = wbase + (int64_t)lane * R;
    issue(wbase + stride + (int64_t)lane * R, buf ^ 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    int32_t k[R];
    long long v[R];
    if (r0 + R <= n) {  // (16-byte shared reads of this thread's own slot)
      const int4* pk = (const int4*)&s_k[buf][threadIdx.x * R];
      const longlong2* pv = (const longlong2*)&s_v[buf][threadIdx.x * R];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int4 a = pk[j];
        k[4 * j] = a.x; k[4 * j + 1] = a.y; k[4 * j + 2] = a.z; k[4 * j + 3] = a.w;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const longlong2 q = pv[j];
        v[2 * j] = q.x;
        v[2 * j + 1] = q.y;
      }
    } else {
      prog.lean_load(r0, n, k, v);  // rows >= n: v = 0, k = 0 (masked by m below)
    }
    buf ^= 1;
    const int m = (int)max((int64_t)0, min((int64_t)R, n - r0));
    int32_t pk = __shfl_up_sync(kFull, k[R - 1], 1);
    if (lane == 0 && r0 > 0 && r0 <= n) pk = prog.lean_key(r0 - 1);
    const bool has_prev = r0 > 0;
    long long lead = 0, s = 0;
    int lead_len = 0;
    bool open = false;
    int32_t ck = 0, prev = pk;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const bool in = i < m;
      wide |= in ? (unsigned)((int32_t)(v[i] >> 32) + 256) >> 9 : 0u;  // |v| >= 2^40
      const bool head = in && (k[i] != prev || (i == 0 && !has_prev));
      bad |= (in && (i > 0 || has_prev) && k[i] < prev) ? 1u : 0u;
      if (head && open) emit(ck, s);
      open = open || head;
      lead += (in && !open) ? v[i] : 0;
      lead_len += (in && !open) ? 1 : 0;
      s = head ? v[i] : s + v[i];
      ck = head ? k[i] : ck;
      prev = in ? k[i] : prev;
    }
    // the next lane's leading rows continue my last group
    const long long nx_lead = __shfl_down_sync(kFull, lead, 1);
    const int nx_len = __shfl_down_sync(kFull, lead_len, 1);
    if (open) {
      const int64_t nxt = r0 + R;
      bool more = true;
      int64_t r = nxt;
      if (lane < 31 && nxt < n) {
        s += nx_lead;
        more = nx_len == R;
        r = nxt + R;
      }
      int steps = 0;
      for (; more && r < n && steps < kRunAhead; ++r, ++steps) {  // rare: scalar continuation
        if (prog.lean_key(r) != ck) break;
        const long long x = prog.lean_val(r);
        wide |= (unsigned)((int32_t)(x >> 32) + 256) >> 9;
        s += x;
      }
      if (more && steps == kRunAhead && r < n) wide = 1;
      emit(ck, s);
    }
  }
  if (bad) atomicExch(flags, 1);
  if (wide) atomicExch(flags + 1, 1);
}

// K10wr: K10w's selective scan fed by the tile ring (ring.cuh) instead of per-lane loads and
// gathers (programs with kWRing: Q9).  One producer warp bulk-copies whole tiles of every column
// the pass reads (partkey, suppkey, orderkey, quantity, price, discount: 36 B/row streamed once at
// full bandwidth, no 128-byte line over-fetch from gathering the 5.4% green rows) into a 3-stage
// shared ring; each of the 16 consumer warps tests its 64 rows of a tile against the green-part
// bitmap, copies the green rows' values into a per-warp buffer, and once 32 are buffered every
// lane runs one row's three lookups (the program's lookups<1>) and aggregates into the per-CTA
// shared table, exactly as K10w.  Rows after the last whole tile: global loads, same path.
template <class P, class = void>
struct has_wring : std::false_type {};
template <class P>
struct has_wring<P, std::void_t<decltype(P::kWRing)>> : std::true_type {};

constexpr int kWrBuf = 96;  // per-warp buffered green rows (<= 31 left + 64 new)

template <class P>
__host__ __device__ constexpr size_t wring_buf_bytes() {
  return (size_t)kWrBuf * (4 + 4 + sizeof(typename P::KeyT) + 8 + 8 + 8);
}

template <class P>
__global__ void __launch_bounds__((P::RingCols::kRingConsumers + 1) * 32, 1)
    k_gb_wring(const __grid_constant__ P prog, const __grid_constant__ typename P::RingCols rc, int64_t n,
               const __grid_constant__ Layout L, Table t, uint32_t scap) {
  using RC = typename P::RingCols;
  using KT = typename P::KeyT;
  constexpr int S = RC::kRingStages, T = RC::kRingTile, NC = RC::kRingConsumers, SL = T / NC;
  static_assert(SL % 32 == 0, "a consumer warp's slice is whole 32-row groups");
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ __align__(8) uint64_t empty[S];
  __shared__ int s_side, s_full;
  uint8_t* const wbufs = ring + (size_t)S * ring_stage_bytes<RC>();
  uint8_t* const sm_tab = wbufs + (size_t)NC * wring_buf_bytes<P>();
  const size_t tbytes = (size_t)(scap + 1) * L.slot_bytes;
  for (size_t j = threadIdx.x * 8; j < tbytes; j += blockDim.x * 8) *(unsigned long long*)(sm_tab + j) = 0;
  if (threadIdx.x == 0) { s_side = 0; s_full = 0; }
  ring_init_bars<RC>(full, empty);
  __syncthreads();
  const Table st{sm_tab, scap - 1, &s_side, &s_full};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // this warp's buffer (consumers only)
  uint8_t* wb = wbufs + (size_t)(warp < NC ? warp : 0) * wring_buf_bytes<P>();
  int32_t* b_pk = (int32_t*)wb;
  int32_t* b_sk = b_pk + kWrBuf;
  KT* b_ok = (KT*)(b_sk + kWrBuf);
  long long* b_q = (long long*)(wb + (size_t)kWrBuf * (8 + sizeof(KT)));
  long long* b_e = b_q + kWrBuf;
  long long* b_d = b_e + kWrBuf;
  bool ovf = false;
  int cnt = 0;  // buffered green rows (warp-uniform)
  const unsigned lt = lanemask_lt();
  auto process = [&](int m) {  // entries [0, m), m <= 32: lane i takes entry i
    bool alive[1] = {lane < m};
    const int i = alive[0] ? lane : 0;
    int32_t pk[1] = {b_pk[i]}, sk[1] = {b_sk[i]};
    KT ok[1] = {b_ok[i]};
    int64_t q[1] = {b_q[i]}, e[1] = {b_e[i]}, d[1] = {b_d[i]};
    uint64_t key[1];
    int64_t v[1];
    prog.template lookups<1>(pk, sk, ok, q, e, d, alive, key, v, ovf);
    if (alive[0]) {
      uint8_t* sp = *(volatile int*)&s_full ? nullptr : find_or_insert(st, L, key[0]);
      if (sp) apply_state_smem(sp, L, 0, (unsigned long long)v[0], v[0] < 0 ? -1 : 0);
      else gb_row_to_global(t, L, key[0], 0, v[0]);
    }
    __syncwarp();
    // move the entries past m (<= 63 of them) to the front: read both into registers, then write
    const int rem = cnt - m;
    int32_t mp[2], ms[2];
    KT mo[2];
    long long mq[2], me[2], md[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = m + h * 32 + lane;
      const bool in = h * 32 + lane < rem;
      mp[h] = in ? b_pk[j] : 0; ms[h] = in ? b_sk[j] : 0; mo[h] = in ? b_ok[j] : (KT)0;
      mq[h] = in ? b_q[j] : 0; me[h] = in ? b_e[j] : 0; md[h] = in ? b_d[j] : 0;
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = h * 32 + lane;
      if (j < rem) {
        b_pk[j] = mp[h]; b_sk[j] = ms[h]; b_ok[j] = mo[h]; b_q[j] = mq[h]; b_e[j] = me[h]; b_d[j] = md[h];
      }
    }
    __syncwarp();
    cnt = rem;
  };
  // append one row (all lanes call; `green` per lane), values given
  auto append = [&](bool green, int32_t pk, int32_t sk, KT ok, long long q, long long e, long long d) {
    const unsigned bal = __ballot_sync(kFull, green);
    if (green) {
      const int pos = cnt + __popc(bal & lt);
      b_pk[pos] = pk; b_sk[pos] = sk; b_ok[pos] = ok; b_q[pos] = q; b_e[pos] = e; b_d[pos] = d;
    }
    cnt += __popc(bal);
    __syncwarp();
  };
  const bool consumer = ring_pipeline(rc, n, ring, full, empty, [&](const uint8_t* const* b, int64_t, int cw, int ln) {
#pragma unroll
    for (int j = 0; j < SL / 32; ++j) {
      const int idx = cw * SL + j * 32 + ln;
      const int32_t pk = ((const int32_t*)b[0])[idx];
      const bool green = prog.wring_green(pk);
      append(green, pk, ((const int32_t*)b[1])[idx], ((const KT*)b[2])[idx], ((const long long*)b[3])[idx],
             ((const long long*)b[4])[idx], ((const long long*)b[5])[idx]);
    }
    while (cnt >= 32) process(32);
  });
  if (consumer) {
    const int64_t ntiles = n / T;
    if (blockIdx.x == gridDim.x - 1) {  // rows after the last whole tile
      for (int64_t r0 = ntiles * T + (int64_t)warp * 32; r0 < n; r0 += (int64_t)NC * 32) {
        const int64_t r = r0 + lane;
        const bool in = r < n;
        const int32_t pk = in ? __ldg((const int32_t*)rc.ring_col(0) + r) : 0;
        const bool green = in && prog.wring_green(pk);
        append(green, pk, green ? __ldg((const int32_t*)rc.ring_col(1) + r) : 0,
               green ? __ldg((const KT*)rc.ring_col(2) + r) : (KT)0, green ? __ldg((const long long*)rc.ring_col(3) + r) : 0,
               green ? __ldg((const long long*)rc.ring_col(4) + r) : 0, green ? __ldg((const long long*)rc.ring_col(5) + r) : 0);
        while (cnt >= 32) process(32);
      }
    }
    while (cnt > 0) process(cnt < 32 ? cnt : 32);
  }
  if (ovf) atomicExch(prog.ovf_flag, 1);
  __syncthreads();
  for (uint32_t e = threadIdx.x; e <= scap; e += blockDim.x) {
    const uint8_t* sl = sm_tab + (size_t)e * L.slot_bytes;
    uint64_t key;
    if (e == scap) {
      if (!s_side) continue;
      key = 0;
    } else {
      key = L.key_bytes == 4 ? (uint64_t)*(const unsigned*)sl : *(const unsigned long long*)sl;
      if (!key) continue;
    }
    uint8_t* p = find_or_insert(t, L, key);
    if (p) merge_slot(p, sl, L);
  }
}

struct EmitArgs {
  const uint8_t* slots;
  const int32_t* ids;
  int64_t n;
  uint64_t cap;
  Layout L;
  int nkeys;
  int out_key_type[2];
  void* out_key[2];
  int naggs;
  int agg_op[SX_MAX_AGGS];
  int agg_state[SX_MAX_AGGS];
  int agg_scale[SX_MAX_AGGS];
  int count_state;
  void* out_agg[SX_MAX_AGGS];
};

__device__ __forceinline__ void put_key(void* dst, int type, int64_t i, int64_t v) {
  switch (type) {
    case SX_U8: ((uint8_t*)dst)[i] = (uint8_t)v; break;
    case SX_I32:
    case SX_DATE32: ((int32_t*)dst)[i] = (int32_t)v; break;
    default: ((int64_t*)dst)[i] = v; break;
  }
}

__device__ __forceinline__ double i128_to_double(unsigned long long lo, long long hi) {
  if ((hi == 0 && (long long)lo >= 0) || (hi == -1 && (long long)lo < 0)) return (double)(long long)lo;
  return (double)hi * 18446744073709551616.0 + (double)lo;
}

static __global__ void k_gb_emit(const __grid_constant__ EmitArgs a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t slot = (uint64_t)a.ids[i];
    const uint8_t* p = a.slots + slot * a.L.slot_bytes;
    if (a.nkeys > 0) {
      uint64_t k = 0;
      if (slot % (a.cap + 1) != a.cap) k = a.L.key_bytes == 4 ? (uint64_t)*(const unsigned*)p : *(const unsigned long long*)p;
      if (a.nkeys == 1) {
        int64_t v = a.L.key_bytes == 4 ? (int64_t)(int32_t)(uint32_t)k : (int64_t)k;
        if (a.out_key_type[0] == SX_U8) v = (uint8_t)k;
        put_key(a.out_key[0], a.out_key_type[0], i, v);
      } else {
        int64_t k0 = (int32_t)(uint32_t)(k >> 32), k1 = (int32_t)(uint32_t)k;
        if (a.out_key_type[0] == SX_U8) k0 = (uint8_t)(k >> 32);
        if (a.out_key_type[1] == SX_U8) k1 = (uint8_t)k;
        put_key(a.out_key[0], a.out_key_type[0], i, k0);
        put_key(a.out_key[1], a.out_key_type[1], i, k1);
      }
    }
    unsigned long long count = a.count_state >= 0 ? *(const unsigned long long*)(p + a.L.off8[a.count_state]) : 0;
    for (int j = 0; j < a.naggs; ++j) {
      int s = a.agg_state[j];
      unsigned long long u = *(const unsigned long long*)(p + a.L.off8[s]);
      switch (a.agg_op[j]) {
        case SX_SUM: {
          long long hi = *(const int*)(p + a.L.off4[s]);
          ((longlong2*)a.out_agg[j])[i] = make_longlong2((long long)u, hi);
          break;
        }
        case SX_COUNT: ((long long*)a.out_agg[j])[i] = (long long)count; break;
        case SX_MIN: ((long long*)a.out_agg[j])[i] = (long long)(~u ^ 0x8000000000000000ull); break;
        case SX_MAX: ((long long*)a.out_agg[j])[i] = (long long)(u ^ 0x8000000000000000ull); break;
        default: {  // AVG = (double)sum / (double)count / 10^scale (reading R3)
          long long hi = *(const int*)(p + a.L.off4[s]);
          double sc = 1.0;
          for (int q = 0; q < a.agg_scale[j]; ++q) sc *= 10.0;
          ((double*)a.out_agg[j])[i] = i128_to_double(u, hi) / (double)count / sc;
          break;
        }
      }
    }
  }
}

// K18 (gbsimple.cu): the plain-shape fast path; SX_EUNSUPPORTED when the call is not of that shape
sx_status gb_simple(sx_ctx* ctx, const sx_col* cols, int ncols, const sx_key* keys, int nkeys, const sx_sel* in_sel,
                    int nwhere, const sx_agg* aggs, int naggs, const sx_having* having, int64_t groups_hint,
                    sx_col* out_keys, sx_col* out_aggs, int64_t* out_ngroups);

inline int agg_out_type(int op) {
  switch (op) {
    case SX_SUM: return SX_I128;
    case SX_AVG: return SX_F64;
    default: return SX_I64;
  }
}

constexpr int64_t kSharedMaxGroups = 4096;      // K10 eligibility (hinted groups)
constexpr uint64_t kRangesMaxBytes = 100u << 10; // K10p per-CTA table bytes (at most; smaller when it suffices)
constexpr int kSharedItems = 1;                  // K10 rows per thread per step (code size vs MLP)
// A program may ask for more rows per thread (P::kSharedItems): fused probe chains need the
// memory-level parallelism of several independent rows per thread.
template <class P, class = void>
struct shared_items { static constexpr int value = kSharedItems; };
template <class P>
struct shared_items<P, std::void_t<decltype(P::kSharedItems)>> { static constexpr int value = P::kSharedItems; };
constexpr uint64_t kSharedMaxBytes = 96u << 10;  // K10 per-CTA table bytes

inline uint64_t pow2_at_least(uint64_t x) {
  uint64_t c = 16;
  while (c < x) c <<= 1;
  return c;
}

// Run the aggregation with program `prog` and produce the outputs.  `force_small` selects K9.
// Strategies: K9 (keyless / <= kSmallSlots groups), K11 into one table when it fits in half the
// L2, otherwise partitioned K11 (records into 2^pbits hash partitions, each merged into an
// L2-resident sub-table).  A table that fills up (bad hint) is resized and the step redone.
// K10p host side: partition every column the program references (keys, predicates, expressions)
// by the group key, remap the program onto the partitioned columns, cut each partition into row
// ranges and aggregate the ranges in shared-memory tables (k_gb_ranges).
inline sx_status gb_ranges(sx_ctx* ctx, const InterpProg& prog, const GbPlan& P, const int32_t* sel, int64_t n,
                           int64_t groups_hint, const Layout& L, const Table& t, Scratch& scr) {
  const GbArgs& A = prog.A;
  bool used[SX_MAX_COLS] = {};
  for (int k = 0; k < P.nkeys; ++k) used[A.kc[k]] = true;
  for (int q = 0; q < A.np; ++q) used[A.preds[q].col] = true;
  for (int a = 0; a < L.nst; ++a)
    for (int tt = 0; tt < A.expr[a].nterms; ++tt)
      for (int f = 0; f < A.expr[a].t[tt].nf; ++f) used[A.expr[a].t[tt].f[f].col] = true;
  DCol carry[SX_MAX_COLS];
  int width[SX_MAX_COLS], map[SX_MAX_COLS], nc = 0;
  void* out[SX_MAX_COLS];
  for (int c = 0; c < SX_MAX_COLS; ++c) {
    map[c] = -1;
    if (!used[c]) continue;
    const int w = A.cols[c].type == SX_U8 ? 1 : (A.cols[c].type == SX_I32 || A.cols[c].type == SX_DATE32) ? 4 : 8;
    carry[nc] = A.cols[c];
    width[nc] = w;
    SX_TRY(scr.get((char**)&out[nc], (size_t)n * w));
    map[c] = nc++;
  }
  if (nc > 12) return set_err(ctx, SX_EINVAL, "group-by references too many columns for partitioning");
  // the largest shared table that fits kRangesMaxBytes (two CTAs per SM); partitions sized so
  // their expected group count fills at most half of it (load <= 0.5)
  uint64_t smax = 1;
  while ((2 * smax + 1) * (uint64_t)L.slot_bytes <= kRangesMaxBytes) smax <<= 1;
  if (smax < 256) return SX_EUNSUPPORTED;
  // partitions of ~512 groups (tables of 1024 slots: several CTAs per SM), more per partition
  // only when the fan-out limit (2^10) forces it
  int bits = 1;
  while (bits < 10 && (uint64_t)(groups_hint >> bits) > 512) ++bits;
  const uint64_t gpp = (uint64_t)(groups_hint >> bits) + 1;
  uint64_t scap = pow2_at_least(gpp + gpp / 2);  // load <= 2/3
  if (scap > smax) return SX_EUNSUPPORTED;  // too many groups per partition: other paths
  std::vector<int64_t> off(((size_t)1 << bits) + 1);
  const DCol k0 = A.cols[A.kc[0]], k1 = A.cols[P.nkeys > 1 ? A.kc[1] : A.kc[0]];
  SX_TRY(radix_partition_carry(ctx, k0, k1, P.nkeys, carry, width, nc, sel, n, bits, out, off.data()));
  InterpProg pp = prog;
  for (int c = 0; c < SX_MAX_COLS; ++c)
    if (map[c] >= 0) pp.A.cols[c].p = out[map[c]];
  // row ranges: each partition cut into pieces of ~n / (4 x SMs) rows
  const int64_t piece = std::max<int64_t>(1 << 16, n / (4 * (int64_t)ctx->num_sms));
  std::vector<int64_t> items;
  for (size_t p = 0; p + 1 < off.size(); ++p)
    for (int64_t lo = off[p]; lo < off[p + 1]; lo += piece) {
      items.push_back(lo);
      items.push_back(std::min(off[p + 1], lo + piece));
    }
  const int64_t nitems = (int64_t)items.size() / 2;
  int64_t* d_items;
  SX_TRY(scr.get(&d_items, items.size() + 1));
  SX_CUDA(cudaMemcpyAsync(d_items, items.data(), items.size() * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
  const size_t smem = (size_t)(scap + 1) * L.slot_bytes;
  SX_CUDA(cudaFuncSetAttribute(k_gb_ranges<InterpProg, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gb_ranges<InterpProg, 4>, kBlock, smem));
  if (per_sm < 1) per_sm = 1;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->num_sms * per_sm, nitems));
  if (nitems > 0)
    k_gb_ranges<InterpProg, 4><<<grid, kBlock, smem, SX_STREAM(ctx)>>>(pp, d_items, nitems, L, t, (uint32_t)scap);
  SX_CHECK_LAUNCH();
  // keep the partitioned columns alive until the kernel has run (Scratch frees stream-ordered)
  return SX_OK;
}

template <class Prog>
sx_status gb_run(sx_ctx* ctx, const Prog& prog, const GbPlan& P, const int32_t* sel, int64_t n,
                 int64_t groups_hint, sx_col* out_keys, sx_col* out_aggs, int64_t* out_ngroups,
                 int force_small = -1) {
  // row ids are int32 everywhere below (K10w compacts them, sel entries are int32): P:271
  if (n > INT32_MAX) return set_err(ctx, SX_EINDEX, "group-by over %lld rows > INT32_MAX", (long long)n);
  Scratch scr(ctx);
  const Layout& L = P.L;
  bool keyless = P.nkeys == 0;
  bool small = keyless || (groups_hint >= 1 && groups_hint <= kSmallSlots);
  if (force_small >= 0) small = force_small != 0;
  // load factor <= 0.75 (linear probing); unknown hint: size for min(n, 2^20) groups, retry if full
  uint64_t want = groups_hint > 0 ? (uint64_t)groups_hint : (uint64_t)(n < (1 << 20) ? n : (1 << 20));
  uint64_t cap = keyless ? 1 : pow2_at_least(want + want / 3 + 1);
  uint8_t* table = nullptr;
  int32_t* ids = nullptr;
  int* side = nullptr;
  int64_t ng = 0;
  int flags[4];
  uint64_t cap_p = cap;  // slots per sub-table
  bool no_part = false;
  int nsub = 1;
  bool sorted_done = false;
  // Sorted-input strategy (see k_runs_count): worth trying when the hash table would not be
  // L2-resident; falls back to hashing if the key column turns out not to be non-decreasing.
  if constexpr (Prog::kSortedOK) {
    // SX_GB_SORTED: 0 = never, 2 = whenever eligible regardless of table size (tests)
    const char* env = getenv("SX_GB_SORTED");
    const int mode = env ? atoi(env) : 1;
    bool own_done = false;
    if constexpr (Prog::kMaxNst <= 2) {
      // K10r: HAVING pushed into an owned-run aggregation (no per-group state written)
      if (mode != 0 && !small && !keyless && P.nkeys == 1 && !sel && n > 0 && prog.no_filter() && P.has_having &&
          L.slot_bytes <= 64 && (mode == 2 || cap * (uint64_t)L.slot_bytes > ctx->l2_bytes / 2)) {
        SlotFn hv;
        std::memset(&hv, 0, sizeof hv);
        hv.has_having = 1;
        const int sh = P.agg_state[P.hv.agg];
        hv.hv_kind = L.kind[sh];
        hv.hv_off8 = L.off8[sh];
        hv.hv_off4 = L.off4[sh];
        hv.hv_op = P.hv.op;
        hv.hv_lo = P.hv.lo;
        hv.hv_hi = P.hv.hi;
        int64_t cap_out = std::max<int64_t>(1 << 16, n / 256);
        unsigned long long* cursor = (unsigned long long*)ctx->d_counters;
        bool lean_failed = false;
        for (int attempt = 0; attempt < 2 && !own_done; ++attempt) {
          uint8_t* out;
          SX_TRY(scr.get(&out, (size_t)cap_out * L.slot_bytes));
          SX_CUDA(cudaMemsetAsync(ctx->d_flags, 0, 4 * sizeof(int), ctx->stream));
          SX_CUDA(cudaMemsetAsync(cursor, 0, 8, ctx->stream));
          const int64_t threads = (n + kRunItems - 1) / kRunItems;
          bool lean = false;
          if constexpr (has_lean_runs<Prog>::value) {
            // K10l first (SX_RUNS_LEAN=0: K10r); a wide value or a long run retries with K10r
            const bool lean_off = getenv("SX_RUNS_LEAN") && getenv("SX_RUNS_LEAN")[0] == '0';
            lean = !lean_off && !lean_failed && L.nst == 1 && L.kind[0] == ST_SUM && L.key_bytes == 4 &&
                   L.slot_bytes <= 32;
            if (lean)
              k_runs_lean<Prog><<<persistent_grid(ctx, 8, ((n + 7) / 8 + kBlock - 1) / kBlock), kBlock, 0,
                                  SX_STREAM(ctx)>>>(prog, n, L, hv, out, cap_out, cursor, ctx->d_flags + 2);
          }
          if (lean) {
          } else if constexpr (runs_dense<Prog>::value) {
            if (L.nst == 1 && L.kind[0] == ST_SUM && L.slot_bytes <= 32)
              k_runs_own_dense<Prog><<<persistent_grid(ctx, 8, ((n + kRunOwnRows - 1) / kRunOwnRows + kBlock - 1) / kBlock),
                                       kBlock, 0, SX_STREAM(ctx)>>>(prog, n, L, hv, out, cap_out, cursor, ctx->d_flags + 2);
            else
              k_runs_own<Prog><<<persistent_grid(ctx, 8, (threads + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
                  prog, n, L, hv, out, cap_out, cursor, ctx->d_flags + 2);
          } else {
            k_runs_own<Prog><<<persistent_grid(ctx, 8, (threads + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
                prog, n, L, hv, out, cap_out, cursor, ctx->d_flags + 2);
          }
          SX_CHECK_LAUNCH();
          int64_t cnt = 0;
          SX_TRY(read_i64(ctx, cursor, &cnt));
          SX_CUDA(cudaMemcpy(flags, ctx->d_flags, 4 * sizeof(int), cudaMemcpyDeviceToHost));
          if (lean && !flags[2] && flags[3]) {  // |v| >= 2^40 or a long run: K10r decides
            lean_failed = true;
            --attempt;
            continue;
          }
          if (flags[2] || flags[3]) break;  // unsorted or a run longer than kRunAhead: other strategies
          if (flags[0]) return set_err(ctx, SX_EOVERFLOW, "a value expression left int64");
          if (cnt > cap_out) {
            cap_out = cnt;
            continue;
          }
          // the survivors form a dense table of cnt groups for the extraction below
          SlotFn sf = hv;
          sf.slots = out;
          sf.cap = (uint64_t)cnt;
          sf.slot_bytes = L.slot_bytes;
          sf.key_bytes = 0;
          sf.nsub = 1;
          sf.side_used = ctx->d_flags + 2;
          GatherSpec none;
          none.n = 0;
          SX_TRY(run_compact(ctx, sf, cnt, nullptr, &ids, nullptr, none, &ng));
          scr.ptrs.push_back(ids);
          table = out;
          cap_p = (uint64_t)cnt;
          sorted_done = own_done = true;
        }
      }
    }
    if (!own_done && mode != 0 && !small && !keyless && P.nkeys == 1 && !sel && n > 0 && prog.no_filter() &&
        (mode == 2 || cap * (uint64_t)L.slot_bytes > ctx->l2_bytes / 2)) {
      const int64_t ntiles = (n + kRunTile - 1) / kRunTile;
      int32_t* heads;
      int64_t *first, *bsum, *carry_gid;
      uint8_t* carry;
      SX_TRY(scr.get(&heads, (size_t)ntiles));
      SX_TRY(scr.get(&first, (size_t)ntiles + 1));
      const int64_t nb = (ntiles + 1023) / 1024;
      SX_TRY(scr.get(&bsum, (size_t)nb + 1));
      SX_CUDA(cudaMemsetAsync(ctx->d_flags, 0, 4 * sizeof(int), ctx->stream));
      k_runs_count<Prog><<<persistent_grid(ctx, 8, ntiles), kBlock, 0, SX_STREAM(ctx)>>>(prog, n, heads, ntiles,
                                                                                      ctx->d_flags + 3);
      k_scan_counts_local<<<(unsigned)nb, 1024, 0, SX_STREAM(ctx)>>>(heads, ntiles, first, bsum);
      k_scan_counts_sums<<<1, 32, 0, SX_STREAM(ctx)>>>(bsum, nb, first + ntiles);
      k_scan_counts_add<<<(unsigned)nb, 1024, 0, SX_STREAM(ctx)>>>(first, ntiles, bsum);
      SX_CHECK_LAUNCH();
      int64_t G = 0;
      SX_TRY(read_i64(ctx, first + ntiles, &G));
      SX_CUDA(cudaMemcpy(flags, ctx->d_flags, 4 * sizeof(int), cudaMemcpyDeviceToHost));
      if (!flags[3]) {
        SX_TRY(scr.get(&table, (size_t)G * L.slot_bytes));  // every slot is written (no zero-fill)
        SX_TRY(scr.get(&carry, (size_t)ntiles * L.slot_bytes));
        SX_TRY(scr.get(&carry_gid, (size_t)ntiles));
        const size_t smem = runs_smem_bytes(L.nst);
        SX_CUDA(cudaFuncSetAttribute(k_runs_agg<Prog>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        SX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_runs_agg<Prog>, kBlock, smem));
        if (per_sm < 1) return set_err(ctx, SX_ENOMEM, "sorted aggregation: %zu B shared memory per CTA", smem);
        unsigned grid = (unsigned)std::min<int64_t>((int64_t)ctx->num_sms * per_sm, ntiles);
        k_runs_agg<Prog><<<grid, kBlock, smem, SX_STREAM(ctx)>>>(prog, n, first, L, table, carry, carry_gid, ntiles);
        k_runs_fix<<<persistent_grid(ctx, 8, (ntiles + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
            L, table, carry, carry_gid, ntiles);
        SX_CHECK_LAUNCH();
        SlotFn sf;
        std::memset(&sf, 0, sizeof sf);
        sf.slots = table;
        sf.cap = (uint64_t)G;
        sf.slot_bytes = L.slot_bytes;
        sf.key_bytes = 0;  // dense: every slot < G is a group
        sf.nsub = 1;
        sf.side_used = ctx->d_flags + 2;
        sf.has_having = P.has_having;
        if (P.has_having) {
          int s = P.agg_state[P.hv.agg];
          sf.hv_kind = L.kind[s];
          sf.hv_off8 = L.off8[s];
          sf.hv_off4 = L.off4[s];
          sf.hv_op = P.hv.op;
          sf.hv_lo = P.hv.lo;
          sf.hv_hi = P.hv.hi;
        }
        GatherSpec none;
        none.n = 0;
        SX_TRY(run_compact(ctx, sf, G, nullptr, &ids, nullptr, none, &ng));
        scr.ptrs.push_back(ids);
        SX_CUDA(cudaMemcpy(flags, ctx->d_flags, 4 * sizeof(int), cudaMemcpyDeviceToHost));
        if (flags[0]) return set_err(ctx, SX_EOVERFLOW, "a value expression left int64");
        cap_p = (uint64_t)G;  // emit: no slot index equals G, so no side-slot key rewrite
        sorted_done = true;
      }
    }
  }
  bool ring_retry = false;  // K9r's per-CTA list of exact-path rows overflowed: redo with K9d
  for (int attempt = 0; !sorted_done; ++attempt) {
    bool ring_used = false;
    // partition when the table would not stay L2-resident
    int pbits = 0;
    // (opt-in until phase A beats the single HBM table: SX_GB_PARTITION=1)
    static const bool part_enabled = getenv("SX_GB_PARTITION") && getenv("SX_GB_PARTITION")[0] == '1';
    if (part_enabled && !small && !keyless && !no_part && cap * (uint64_t)L.slot_bytes > ctx->l2_bytes / 2) {
      while (pbits < 8 && (cap >> pbits) * (uint64_t)L.slot_bytes > ctx->l2_bytes / 4) ++pbits;
    }
    nsub = 1 << pbits;
    cap_p = keyless ? 1 : cap >> pbits;
    // K10 when a hinted group count fits a per-CTA shared-memory table at load <= 0.5
    uint32_t shared_cap = 0;
    if (!small && !keyless && attempt == 0 && groups_hint > 0 && groups_hint <= kSharedMaxGroups) {
      uint64_t sc = pow2_at_least(2 * (uint64_t)groups_hint);
      if ((sc + 1) * (uint64_t)L.slot_bytes <= kSharedMaxBytes) shared_cap = (uint32_t)sc;
    }
    uint64_t nslots = keyless ? 1 : (uint64_t)nsub * (cap_p + 1);
    SX_TRY(scr.get(&table, nslots * L.slot_bytes));
    SX_CUDA(cudaMemsetAsync(table, 0, nslots * L.slot_bytes, ctx->stream));
    SX_CUDA(cudaMemsetAsync(ctx->d_flags, 0, 4 * sizeof(int), ctx->stream));
    SX_TRY(scr.get(&side, (size_t)nsub));
    SX_CUDA(cudaMemsetAsync(side, 0, nsub * sizeof(int), ctx->stream));
    Table t{table, keyless ? 0 : cap_p - 1, side, ctx->d_flags + 1};
    bool part_overflow = false;
    bool dense_done = false;
    if constexpr (has_dense<Prog>::value) {
      // K9d: dense input + vector-loading program (see k_gb_dense); the grid must keep every
      // thread at <= 2^21 rows so that its int64 partial sums of |v| < 2^41 values cannot overflow
      if (n > 0 && small && !sel && L.nst == Prog::kDenseNst) {
        bool staged = false;
        if constexpr (has_ring<Prog>::value) {
          // K9r (ring.cuh): producer warp + bulk-copy tile ring, one CTA per SM; every column base
          // is 16-B aligned (to_dcols) and a tile's column chunks are multiples of 16 B.  SX_RING=0: K9d.
          const bool ring_off = getenv("SX_RING") && getenv("SX_RING")[0] == '0';
          if (!ring_off && !ring_retry && n >= (int64_t)Prog::kRingTile * ctx->num_sms) {
            const size_t smem = ring_smem_bytes<Prog>();
            SX_CUDA(cudaFuncSetAttribute(k_gb_ring<Prog>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_gb_ring<Prog><<<(unsigned)ctx->num_sms, (Prog::kRingConsumers + 1) * 32, smem, SX_STREAM(ctx)>>>(prog, n, L, t);
            SX_CHECK_LAUNCH();
            staged = dense_done = ring_used = true;
          }
        }
        if constexpr (has_bulk<Prog>::value) if (!staged) {
          // K9s: bulk-staged (cp.async.bulk) tiles, one CTA per SM, when every column base is 16-B aligned
          // opt-in (SX_BULK=1): measured slower than K9d on Q1 at SF100 (6.1 vs 4.3 ms) — one 8-warp CTA
          // per SM cannot hide the shared-memory latency of the per-row aggregation (profiles/)
          const bool bulk_off = !(getenv("SX_BULK") && getenv("SX_BULK")[0] == '1');
          bool aligned = true;
          for (int c = 0; c < Prog::kBulkCols; ++c) aligned = aligned && ((uintptr_t)prog.bulk_col(c) % 16) == 0;
          const int64_t rows_per_thread = (n + (int64_t)ctx->num_sms * kDenseThreads - 1) / ((int64_t)ctx->num_sms * kDenseThreads);
          if (!bulk_off && aligned && n >= (int64_t)kBulkTile * ctx->num_sms && rows_per_thread <= kDenseMaxRowsPerThread) {
            size_t smem = dense_smem_bytes<Prog::kDenseNst>() + 128 + (size_t)kBulkStages * bulk_stage_bytes<Prog>();
            SX_CUDA(cudaFuncSetAttribute(k_gb_dense<Prog, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_gb_dense<Prog, true><<<(unsigned)ctx->num_sms, kDenseThreads, smem, SX_STREAM(ctx)>>>(prog, n, L, t);
            SX_CHECK_LAUNCH();
            staged = dense_done = true;
          }
        }
        if (!staged) {
          size_t smem = dense_smem_bytes<Prog::kDenseNst>();
          SX_CUDA(cudaFuncSetAttribute(k_gb_dense<Prog, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          int per_sm = 0;
          SX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gb_dense<Prog, false>, kDenseThreads, smem));
          if (per_sm < 1) per_sm = 1;
          int64_t groups = (n + Prog::kDenseRows - 1) / Prog::kDenseRows;
          int64_t ctas = std::min<int64_t>((int64_t)ctx->num_sms * per_sm, (groups + kDenseThreads - 1) / kDenseThreads);
          if ((groups + ctas * kDenseThreads - 1) / (ctas * kDenseThreads) * Prog::kDenseRows <= kDenseMaxRowsPerThread) {
            k_gb_dense<Prog, false><<<(unsigned)ctas, kDenseThreads, smem, SX_STREAM(ctx)>>>(prog, n, L, t);
            SX_CHECK_LAUNCH();
            dense_done = true;
          }
        }
      }
    }
    bool ranges_done = false;
    if constexpr (std::is_same<Prog, InterpProg>::value) {
      // K10p: radix-partition the referenced columns on the group key, then per-range shared tables
      static const bool ranges_off = getenv("SX_GB_RANGES") && getenv("SX_GB_RANGES")[0] == '0';
      bool ident = true;
      for (int k = 0; k < P.nkeys; ++k) ident = ident && P.key_fn[k] == SX_KEY_IDENTITY;
      if (!ranges_off && n >= (1 << 22) && !small && !keyless && nsub == 1 && attempt == 0 && ident &&
          shared_cap == 0 && groups_hint > 256) {  // (K10 covers what fits one shared table)
        const sx_status rs = gb_ranges(ctx, prog, P, sel, n, groups_hint, L, t, scr);
        if (rs == SX_OK) ranges_done = true;
        else if (rs != SX_EUNSUPPORTED) return rs;
      }
    }
    if constexpr (has_wring<Prog>::value) {
      // K10wr: the selective scan fed by the tile ring; one CTA per SM.  Opt-in (SX_Q9_RING=1):
      // measured 8.6 vs 4.3 ms for K10w at SF100 — its 16 consumer warps per SM cannot hide the
      // latency of the green rows' lookups (ncu: 69% long-scoreboard stalls, 3.2 TB/s)
      using RC = typename Prog::RingCols;
      const bool ring_off = !(getenv("SX_Q9_RING") && getenv("SX_Q9_RING")[0] == '1');
      const typename Prog::RingCols rc = prog.ring_cols();
      bool aligned = true;
      for (int c = 0; c < RC::kRingCols; ++c) aligned = aligned && ((uintptr_t)rc.ring_col(c) % 16) == 0;
      if (!ring_off && aligned && !dense_done && n >= (int64_t)RC::kRingTile * ctx->num_sms && !sel && shared_cap &&
          nsub == 1 && L.nst == 1 && prog.wscan_ok()) {
        const size_t smem = (size_t)RC::kRingStages * ring_stage_bytes<RC>() + (size_t)RC::kRingConsumers * wring_buf_bytes<Prog>() +
                            (size_t)(shared_cap + 1) * L.slot_bytes;
        SX_CUDA(cudaFuncSetAttribute(k_gb_wring<Prog>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_gb_wring<Prog><<<(unsigned)ctx->num_sms, (RC::kRingConsumers + 1) * 32, smem, SX_STREAM(ctx)>>>(
            prog, rc, n, L, t, shared_cap);
        SX_CHECK_LAUNCH();
        dense_done = true;
      }
    }
    if constexpr (has_wscan<Prog>::value) {
      // K10w: warp-compacted scan (selective streaming filter + lookup chain), hinted mid G
      if (!dense_done && n > 0 && !sel && shared_cap && nsub == 1 && L.nst == 1 && prog.wscan_ok()) {
        size_t smem = (size_t)(kBlock / 32) * 2 * (32 * 8 * Prog::kWChunks) * sizeof(int32_t) +
                      (size_t)(shared_cap + 1) * L.slot_bytes;
        SX_CUDA(cudaFuncSetAttribute(k_gb_wscan<Prog>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        SX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gb_wscan<Prog>, kBlock, smem));
        if (per_sm < 1) per_sm = 1;
        const int64_t windows = (n + 32 * 8 * Prog::kWChunks - 1) / (32 * 8 * Prog::kWChunks);
        const unsigned grid = (unsigned)std::min<int64_t>((int64_t)ctx->num_sms * per_sm, (windows + kBlock / 32 - 1) / (kBlock / 32));
        k_gb_wscan<Prog><<<grid, kBlock, smem, SX_STREAM(ctx)>>>(prog, n, L, t, shared_cap);
        SX_CHECK_LAUNCH();
        dense_done = true;
      }
    }
    if constexpr (has_dense_shared<Prog>::value) {
      // K10d: dense vector-loading program into a per-CTA shared table (hinted mid G)
      if (!dense_done && n > 0 && !sel && shared_cap && nsub == 1 && prog.dense_ok()) {
        size_t smem = (size_t)(shared_cap + 1) * L.slot_bytes;
        SX_CUDA(cudaFuncSetAttribute(k_gb_dense_shared<Prog>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        SX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gb_dense_shared<Prog>, kBlock, smem));
        if (per_sm < 1) per_sm = 1;
        const int64_t groups = (n + Prog::kDenseRows - 1) / Prog::kDenseRows;
        const unsigned grid = (unsigned)std::min<int64_t>((int64_t)ctx->num_sms * per_sm, (groups + kBlock - 1) / kBlock);
        k_gb_dense_shared<Prog><<<grid, kBlock, smem, SX_STREAM(ctx)>>>(prog, n, L, t, shared_cap);
        SX_CHECK_LAUNCH();
        dense_done = true;
      }
    }
    if (dense_done || ranges_done) {
    } else if (n > 0 && small) {
      size_t smem = small_smem_bytes(L.nst);
      SX_CUDA(cudaFuncSetAttribute(k_gb_small<Prog, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = 0;
      SX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gb_small<Prog, 4>, kSmallThreads, smem));
      if (per_sm < 1) per_sm = 1;
      int64_t tiles = (n + (int64_t)kSmallThreads * 4 - 1) / ((int64_t)kSmallThreads * 4);
      unsigned grid = (unsigned)std::min<int64_t>((int64_t)ctx->num_sms * per_sm, tiles);
      k_gb_small<Prog, 4><<<grid, kSmallThreads, smem, SX_STREAM(ctx)>>>(prog, sel, n, L, t);
      SX_CHECK_LAUNCH();
    } else if (n > 0 && nsub == 1 && shared_cap) {
      constexpr int SI = shared_items<Prog>::value;
      size_t smem = (size_t)(shared_cap + 1) * L.slot_bytes;
      SX_CUDA(cudaFuncSetAttribute(k_gb_shared<Prog, SI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = 0;
      SX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gb_shared<Prog, SI>, kBlock, smem));
      if (per_sm < 1) per_sm = 1;
      int64_t tiles = (n + (int64_t)kBlock * 4 - 1) / ((int64_t)kBlock * 4);
      unsigned grid = (unsigned)std::min<int64_t>((int64_t)ctx->num_sms * per_sm, tiles);
      k_gb_shared<Prog, SI><<<grid, kBlock, smem, SX_STREAM(ctx)>>>(prog, sel, n, L, t, shared_cap);
      SX_CHECK_LAUNCH();
    } else if (n > 0 && nsub == 1) {
      int64_t tiles = (n + 32 * 4 - 1) / (32 * 4) / (kBlock / 32) + 1;
      k_gb_global<Prog, 4><<<persistent_grid(ctx, 8, tiles), kBlock, 0, SX_STREAM(ctx)>>>(prog, sel, n, L, t);
      SX_CHECK_LAUNCH();
    } else if (n > 0) {
      // phase A: evaluate + pre-reduce runs + scatter partial records into hash partitions
      PartOut po;
      std::memset(&po, 0, sizeof po);
      po.pbits = pbits;
      po.regcap = n / nsub + n / nsub / 4 + 4096;
      int64_t total = po.regcap * nsub;
      SX_TRY(scr.get(&po.key, (size_t)total));
      for (int a = 0; a < L.nst; ++a) {
        SX_TRY(scr.get(&po.lo[a], (size_t)total));
        if (L.kind[a] == ST_SUM) SX_TRY(scr.get(&po.hi[a], (size_t)total));
      }
      SX_TRY(scr.get(&po.cursor, (size_t)nsub));
      SX_CUDA(cudaMemsetAsync(po.cursor, 0, nsub * sizeof(unsigned), ctx->stream));
      po.overflow = ctx->d_flags + 3;
      // write-combining staging: ~160 KB of shared memory per CTA, one CTA per SM
      size_t rec = 8 + 8 * (size_t)L.nst + 4 * (size_t)L.nst;
      int wc_cap = (int)std::min<size_t>(128, (160u << 10) / ((size_t)nsub * rec));
      if (wc_cap < 8) wc_cap = 8;
      size_t smem = (size_t)nsub * wc_cap * rec;
      // expected records per partition per tile ~ tile_rows / nsub; flush at ~half the region
      int wc_tiles = std::max(1, (int)(wc_cap / 2 * nsub / 1024));
      SX_CUDA(cudaFuncSetAttribute(k_gb_part<Prog, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int64_t tiles = (n + (int64_t)kBlock * 4 - 1) / ((int64_t)kBlock * 4);
      unsigned grid = (unsigned)std::min<int64_t>(ctx->num_sms, tiles);
      k_gb_part<Prog, 4><<<grid, kBlock, smem, SX_STREAM(ctx)>>>(prog, sel, n, L, po, wc_cap, wc_tiles);
      SX_CHECK_LAUNCH();
      std::vector<unsigned> cnt((size_t)nsub);
      SX_CUDA(cudaMemcpyAsync(cnt.data(), po.cursor, nsub * sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
      SX_CUDA(cudaMemcpyAsync(flags, ctx->d_flags, 4 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      SX_CUDA(cudaStreamSynchronize(ctx->stream));
      if (flags[3]) {
        part_overflow = true;  // a skewed partition: redo unpartitioned
      } else {
        // phase B: one launch per partition, each into its own L2-resident sub-table
        for (int q = 0; q < nsub; ++q) {
          if (!cnt[q]) continue;
          MergeArgs m;
          std::memset(&m, 0, sizeof m);
          int64_t off = (int64_t)q * po.regcap;
          m.key = po.key + off;
          for (int a = 0; a < L.nst; ++a) {
            m.lo[a] = po.lo[a] + off;
            m.hi[a] = po.hi[a] ? po.hi[a] + off : nullptr;
            m.lo_stride[a] = 1;
            m.hi_stride[a] = 1;
          }
          m.n = cnt[q];
          Table tq{table + (uint64_t)q * (cap_p + 1) * L.slot_bytes, cap_p - 1, side + q, ctx->d_flags + 1};
          k_gb_merge_records<<<persistent_grid(ctx, 8, (m.n + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(m, L, tq);
          SX_CHECK_LAUNCH();
        }
      }
      for (int a = 0; a < L.nst; ++a) {
        dfree(ctx, po.lo[a]); scr.release(po.lo[a]);
        if (po.hi[a]) { dfree(ctx, po.hi[a]); scr.release(po.hi[a]); }
      }
      dfree(ctx, po.key); scr.release(po.key);
    }
    if (part_overflow) {
      if (attempt >= 2) return set_err(ctx, SX_ENOMEM, "partitioned aggregation overflow");
      dfree(ctx, table); scr.release(table);
      // fall back to a single HBM table
      small = false;
      no_part = true;
      continue;
    }
    SlotFn sf;
    sf.slots = table;
    sf.cap = keyless ? 1 : cap_p;
    sf.slot_bytes = L.slot_bytes;
    sf.key_bytes = L.key_bytes;
    sf.side_used = side;
    sf.nsub = nsub;
    sf.has_having = P.has_having;
    if (P.has_having) {
      int s = P.agg_state[P.hv.agg];
      sf.hv_kind = L.kind[s];
      sf.hv_off8 = L.off8[s];
      sf.hv_off4 = L.off4[s];
      sf.hv_op = P.hv.op;
      sf.hv_lo = P.hv.lo;
      sf.hv_hi = P.hv.hi;
    }
    GatherSpec none;
    none.n = 0;
    SX_TRY(run_compact(ctx, sf, (int64_t)nslots, nullptr, &ids, nullptr, none, &ng));
    scr.ptrs.push_back(ids);
    SX_CUDA(cudaMemcpy(flags, ctx->d_flags, 4 * sizeof(int), cudaMemcpyDeviceToHost));
    if (flags[0]) return set_err(ctx, SX_EOVERFLOW, "a value expression left int64");
    if (ring_used && flags[3]) {
      if (attempt >= 2) return set_err(ctx, SX_ENOMEM, "ring aggregation retry failed");
      dfree(ctx, table); scr.release(table);
      dfree(ctx, ids); scr.release(ids);
      ring_retry = true;
      continue;
    }
    if (!flags[1]) break;
    // table full: the hint was too small; retry at an upper bound (G <= n)
    if (attempt >= 2) return set_err(ctx, SX_ENOMEM, "aggregation table full after resizing");
    dfree(ctx, table); scr.release(table);
    dfree(ctx, ids); scr.release(ids);
    cap = pow2_at_least((uint64_t)(2 * n > 32 ? 2 * n : 32));
    small = false;
  }
  // outputs
  EmitArgs ea;
  std::memset(&ea, 0, sizeof(ea));
  ea.slots = table;
  ea.ids = ids;
  ea.n = ng;
  ea.cap = keyless ? 1 : cap_p;
  ea.L = L;
  ea.nkeys = P.nkeys;
  ea.naggs = P.naggs;
  ea.count_state = P.count_state;
  for (int k = 0; k < P.nkeys; ++k) {
    ea.out_key_type[k] = P.out_key_type[k];
    SX_TRY(scr.get((char**)&ea.out_key[k], (size_t)ng * type_width(P.out_key_type[k])));
  }
  for (int j = 0; j < P.naggs; ++j) {
    ea.agg_op[j] = P.agg_op[j];
    ea.agg_state[j] = P.agg_state[j];
    ea.agg_scale[j] = P.agg_scale[j];
    SX_TRY(scr.get((char**)&ea.out_agg[j], (size_t)ng * type_width(agg_out_type(P.agg_op[j]))));
  }
  if (ng > 0) {
    k_gb_emit<<<persistent_grid(ctx, 8, (ng + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(ea);
    SX_CHECK_LAUNCH();
  }
  for (int k = 0; k < P.nkeys; ++k) {
    out_keys[k] = sx_col{P.out_key_type[k], 0, ng, ea.out_key[k], nullptr, nullptr};
    scr.release(ea.out_key[k]);
  }
  for (int j = 0; j < P.naggs; ++j) {
    out_aggs[j] = sx_col{agg_out_type(P.agg_op[j]), 0, ng, ea.out_agg[j], nullptr, nullptr};
    scr.release(ea.out_agg[j]);
  }
  *out_ngroups = ng;
  return SX_OK;
}

}  // namespace sx
