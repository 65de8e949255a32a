// groupby.cuh — hash group-by skeletons (K9 register-privatised small-G, K11
// global open addressing) shared by the generic sx_groupby_agg and the
// fixed-plan executor's compile-time-specialised row functors.
//
// Aggregation table: AoS slots of `slot_bytes`; key field first (4 or 8 bytes,
// 0 = EMPTY; a real key 0 goes to the side slot at index cap, flagged in
// d_flags[2]).  States:
//   SUM/AVG: {u64 lo at off8; i32 hi at off4}  (96-bit two's complement; cannot
//            overflow: <= 2^31 rows x |v| < 2^63 < 2^94)
//   COUNT:   u64 at off8
//   MIN/MAX: u64 at off8, order-preserving u = v ^ 2^63; MAX stores u, MIN stores ~u,
//            both updated with atomicMax so an all-zero slot is the identity.
// The whole table is zero-initialised with one memset.
#pragma once
#include "common.cuh"

namespace sx {

constexpr int kMaxStates = SX_MAX_AGGS;
enum StateKind : int32_t { ST_SUM = 0, ST_COUNT = 1, ST_MIN = 2, ST_MAX = 3 };

struct Layout {
  int32_t key_bytes;          // 0 (keyless), 4 or 8
  int32_t slot_bytes;
  int32_t nst;                // states
  int32_t kind[kMaxStates];
  int32_t off8[kMaxStates];   // byte offset of the 8-byte field
  int32_t off4[kMaxStates];   // byte offset of the 4-byte hi field (SUM only)
};

struct Table {
  uint8_t* slots;
  uint64_t mask;     // cap - 1 (cap power of two); side slot at index cap
  int* side_used;    // d_flags + 2
  int* full;         // d_flags + 1
};

__device__ __forceinline__ uint8_t* slot_ptr(const Table& t, int slot_bytes, uint64_t i) {
  return t.slots + i * (uint64_t)slot_bytes;
}

// Find or claim the slot of `key`; returns nullptr (and raises *full) if the table is full.
__device__ __forceinline__ uint8_t* find_or_insert(const Table& t, const Layout& L, uint64_t key) {
  if (L.key_bytes == 0) return t.slots;
  if (key == 0) {
    if (!*(volatile int*)t.side_used) atomicExch(t.side_used, 1);
    return slot_ptr(t, L.slot_bytes, t.mask + 1);
  }
  uint64_t h = hash64(key) & t.mask;
  for (uint64_t probe = 0; probe <= t.mask; ++probe) {
    uint8_t* s = slot_ptr(t, L.slot_bytes, h);
    if (L.key_bytes == 4) {
      unsigned* k = (unsigned*)s;
      unsigned cur = *(volatile unsigned*)k;
      if (cur == (unsigned)key) return s;
      if (cur == 0) {
        unsigned old = atomicCAS(k, 0u, (unsigned)key);
        if (old == 0u || old == (unsigned)key) return s;
      }
    } else {
      unsigned long long* k = (unsigned long long*)s;
      unsigned long long cur = *(volatile unsigned long long*)k;
      if (cur == key) return s;
      if (cur == 0) {
        unsigned long long old = atomicCAS(k, 0ull, (unsigned long long)key);
        if (old == 0ull || old == key) return s;
      }
    }
    h = (h + 1) & t.mask;
  }
  atomicExch(t.full, 1);
  return nullptr;
}

__device__ __forceinline__ unsigned long long order_u(int64_t v) { return (unsigned long long)v ^ 0x8000000000000000ull; }

// Apply one row's (or a pre-reduced segment's) state values to a slot.
// sum states carry a 96-bit value {lo, hi}; count in cnt; min/max in lo (as int64).
__device__ __forceinline__ void apply_states(uint8_t* s, const Layout& L, const unsigned long long* lo,
                                             const int32_t* hi, unsigned long long cnt) {
  for (int a = 0; a < L.nst; ++a) {
    switch (L.kind[a]) {
      case ST_SUM:
        atomic_add_sum96((unsigned long long*)(s + L.off8[a]), (int*)(s + L.off4[a]), (int64_t)lo[a], hi[a]);
        break;
      case ST_COUNT: atomicAdd((unsigned long long*)(s + L.off8[a]), cnt); break;
      case ST_MIN: atomicMax((unsigned long long*)(s + L.off8[a]), ~order_u((int64_t)lo[a])); break;
      default: atomicMax((unsigned long long*)(s + L.off8[a]), order_u((int64_t)lo[a])); break;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// K11: global open-addressing aggregation.  Rows are taken warp-contiguously; runs of equal keys
// in consecutive lanes (clustered inputs, e.g. lineitem by orderkey) are pre-reduced with a
// segmented warp scan so only each run's tail lane touches the table.
// RowFn: __device__ bool row(int64_t r, uint64_t& key, int64_t (&v)[kMaxStates]) const
//        (returns false if the row is filtered out); int nst(); kind(a).
template <class RowFn>
__global__ void __launch_bounds__(kBlock) k_gb_global(const __grid_constant__ RowFn fn, const int32_t* __restrict__ sel,
                                                      int64_t n, const __grid_constant__ Layout L, Table t) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < n; base += stride) {
    int64_t idx = base + lane;
    bool alive = idx < n;
    uint64_t key = 0;
    int64_t v[kMaxStates];
    if (alive) {
      int64_t r = sel ? (int64_t)__ldg(sel + idx) : idx;
      alive = fn.row(r, key, v);
    }
    // segmented inclusive scan over lanes: a segment = maximal run of alive lanes with equal key
    uint64_t pkey = __shfl_up_sync(kFull, key, 1);
    bool palive = __shfl_up_sync(kFull, alive, 1);
    bool head = !alive || lane == 0 || !palive || pkey != key;
    unsigned heads = __ballot_sync(kFull, head);
    uint64_t nkey = __shfl_down_sync(kFull, key, 1);
    bool nalive = __shfl_down_sync(kFull, alive, 1);
    bool tail = alive && (lane == 31 || !nalive || nkey != key);
    // segment start lane for this lane
    unsigned below = heads & (0xffffffffu >> (31 - lane));  // heads at lanes <= lane
    int seg_start = 31 - __clz(below);
    unsigned long long lo[kMaxStates];
    int32_t hi[kMaxStates];
    unsigned long long cnt = alive ? 1 : 0;
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long c2 = __shfl_up_sync(kFull, cnt, o);
      if (lane - o >= seg_start) cnt += c2;
    }
    for (int a = 0; a < L.nst; ++a) {
      int k = L.kind[a];
      if (k == ST_COUNT) continue;
      if (k == ST_SUM) {
        unsigned long long l = alive ? (unsigned long long)v[a] : 0;
        int32_t h = alive ? (v[a] < 0 ? -1 : 0) : 0;
        for (int o = 1; o < 32; o <<= 1) {
          unsigned long long l2 = __shfl_up_sync(kFull, l, o);
          int32_t h2 = __shfl_up_sync(kFull, h, o);
          if (lane - o >= seg_start) {
            unsigned long long s = l + l2;
            h += h2 + (s < l ? 1 : 0);
            l = s;
          }
        }
        lo[a] = l;
        hi[a] = h;
      } else {
        int64_t m = alive ? v[a] : (k == ST_MIN ? INT64_MAX : INT64_MIN);
        for (int o = 1; o < 32; o <<= 1) {
          int64_t m2 = __shfl_up_sync(kFull, m, o);
          if (lane - o >= seg_start) m = (k == ST_MIN) ? (m2 < m ? m2 : m) : (m2 > m ? m2 : m);
        }
        lo[a] = (unsigned long long)m;
        hi[a] = 0;
      }
    }
    if (tail) {
      uint8_t* s = find_or_insert(t, L, key);
      if (s) apply_states(s, L, lo, hi, cnt);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// K9: register-privatised aggregation for very few groups (Q1: 4; keyless reduce: 1).
// Each thread keeps NSLOT (key -> states) slots in registers.  Sums are exact without any
// overflow check: v = vh * 2^32 + vl is accumulated as sum(vl) in u64 and sum(vh) in i64
// (neither can overflow for < 2^31 rows).  A row whose key finds no free slot goes straight to
// the global table.  Slots are flushed to the global table once per thread at the end.
template <class RowFn, int NSLOT, int NST>
__global__ void __launch_bounds__(kBlock) k_gb_small(const __grid_constant__ RowFn fn, const int32_t* __restrict__ sel,
                                                     int64_t n, const __grid_constant__ Layout L, Table t) {
  uint64_t skey[NSLOT];
  bool used[NSLOT];
  unsigned long long cnt[NSLOT];
  unsigned long long al[NSLOT][NST];  // SUM: sum of low 32-bit halves; MIN/MAX: ordered u (max)
  long long ah[NSLOT][NST];           // SUM: sum of high halves
#pragma unroll
  for (int k = 0; k < NSLOT; ++k) {
    used[k] = false;
    skey[k] = 0;
    cnt[k] = 0;
#pragma unroll
    for (int a = 0; a < NST; ++a) { al[k][a] = 0; ah[k][a] = 0; }
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += stride) {
    int64_t r = sel ? (int64_t)__ldg(sel + idx) : idx;
    uint64_t key = 0;
    int64_t v[kMaxStates];
    if (!fn.row(r, key, v)) continue;
    int s = -1;
#pragma unroll
    for (int k = 0; k < NSLOT; ++k)
      if (used[k] && skey[k] == key) s = k;
    if (s < 0) {
#pragma unroll
      for (int k = NSLOT - 1; k >= 0; --k)
        if (!used[k]) s = k;
      if (s >= 0) {
#pragma unroll
        for (int k = 0; k < NSLOT; ++k)
          if (k == s) { used[k] = true; skey[k] = key; }
      }
    }
    if (s < 0) {  // slots exhausted: this row goes to the global table directly
      uint8_t* p = find_or_insert(t, L, key);
      if (p) {
        unsigned long long lo[kMaxStates];
        int32_t hi[kMaxStates];
        for (int a = 0; a < L.nst; ++a) { lo[a] = (unsigned long long)v[a]; hi[a] = v[a] < 0 ? -1 : 0; }
        apply_states(p, L, lo, hi, 1);
      }
      continue;
    }
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) {
      if (k != s) continue;
      cnt[k] += 1;
#pragma unroll
      for (int a = 0; a < NST; ++a) {
        if (a >= L.nst) break;
        const int kd = L.kind[a];
        if (kd == ST_SUM) {
          al[k][a] += (unsigned long long)(uint32_t)v[a];
          ah[k][a] += (long long)(v[a] >> 32);
        } else if (kd == ST_MIN) {
          unsigned long long u = ~order_u(v[a]);
          al[k][a] = u > al[k][a] ? u : al[k][a];
        } else if (kd == ST_MAX) {
          unsigned long long u = order_u(v[a]);
          al[k][a] = u > al[k][a] ? u : al[k][a];
        }
      }
    }
  }
  // flush
#pragma unroll
  for (int k = 0; k < NSLOT; ++k) {
    if (!used[k]) continue;
    uint8_t* p = find_or_insert(t, L, skey[k]);
    if (!p) continue;
#pragma unroll
    for (int a = 0; a < NST; ++a) {
      if (a >= L.nst) break;
      const int kd = L.kind[a];
      if (kd == ST_SUM) {
        // total = ah * 2^32 + al  (al < 2^63, |ah| < 2^62) as a 96-bit {lo, hi}
        __int128 tot = ((__int128)ah[k][a] << 32) + (__int128)al[k][a];
        atomic_add_sum96((unsigned long long*)(p + L.off8[a]), (int*)(p + L.off4[a]), (int64_t)(unsigned long long)tot,
                         (int32_t)(tot >> 64));
      } else if (kd == ST_COUNT) {
        atomicAdd((unsigned long long*)(p + L.off8[a]), cnt[k]);
      } else {
        atomicMax((unsigned long long*)(p + L.off8[a]), al[k][a]);
      }
    }
  }
}

}  // namespace sx
