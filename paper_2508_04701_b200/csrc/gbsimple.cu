// gbsimple.cu — K18 / K19t: the plain-shape fast paths of sx_groupby_agg (H7).
//
// Dispatch (gb_simple): the fixed signature (one value column: COUNT + SUM/MIN/MAX/AVG) with
// <= 16384 hinted groups takes K19t (lane-private count/sum cells, below); everything else of the
// plain shape takes K18.
//
// group-by is substantial where few groups cause memory contention (Q1) and where
// many groups need a large table (Q10/Q18); SURVEY §8(d) C5b sweeps G = 2^2 .. 2^26.  For the plain
// shape — one integer key column (identity), no WHERE / selection / HAVING, every aggregate a
// COUNT or SUM / MIN / MAX / AVG of one integer column — the aggregation runs in shared memory
// for every G the partitioner can split down to a shared table:
//
//   K18s (a 2 x hint-slot table fits ~200 KB, G <~ 2500): each CTA aggregates a contiguous chunk
//        of rows into R replicas of a shared-memory hash table (lane l uses replica l % R, so
//        small G does not serialise on a few shared addresses), then merges its replicas into a
//        global table (one atomic per group and state per CTA) from which the groups are emitted;
//   K18p (hinted G <= 2^26): the key and value columns are radix-partitioned on hash bits 48..
//        (K7, the join's partitioner) into 1024 partitions — above 2^21 groups each is split 32
//        ways more by bits 43..47 (K18p2, segment-local) — and one CTA per partition aggregates
//        it in a shared table and writes its groups straight to the output (partitions hold
//        disjoint keys, so no merge).
//
// Exactness (readings R2/R3): shared partial sums are exact while every value is < 2^40 in
// magnitude and a CTA sums <= 2^22 rows (checked: a row outside takes an exact global 96-bit
// atomic instead); global sums are 96-bit; AVG = (double)sum / (double)count / 10^scale exactly
// as the generic path.  Anything else returns SX_EUNSUPPORTED and sx_groupby_agg takes the generic
// path.  Output group order is unspecified (R13).
#include <algorithm>
#include <cstring>
#include <type_traits>
#include <vector>

#include "gb_host.cuh"
#include "radix.cuh"

using namespace sx;

namespace {

constexpr int kGsThreads = 512;
constexpr int kGsMaxStates = 6;
constexpr int kGsMaxVals = 4;
constexpr long long kEmptyKey = LLONG_MIN;  // shared / global EMPTY marker; the real key goes to the side slot
constexpr int kGsPartSlots = 4096;          // K18p shared table (<= ~2048 groups per partition)

struct GsSpec {
  const void* key;
  int key_bytes;  // 4 or 8
  int key_type;
  int nv;
  const void* val[kGsMaxVals];
  int vbytes[kGsMaxVals];
  int nst;
  int kind[kGsMaxStates];  // ST_SUM / ST_COUNT / ST_MIN / ST_MAX
  int vc[kGsMaxStates];    // value column of the state (-1: COUNT)
  // outputs
  int naggs;
  int agg_op[SX_MAX_AGGS];
  int agg_state[SX_MAX_AGGS];
  int agg_scale[SX_MAX_AGGS];
  int count_state;
  void* out_key;
  void* out_agg[SX_MAX_AGGS];
  int64_t out_cap;
  unsigned long long* out_cursor;
  int* flags;  // [0] a shared table filled up
};

// global merge table (K18s): keys[C + 1] (side slot C for kEmptyKey), per state C + 1 u64 (+ hi)
struct GsGlobal {
  unsigned long long* keys;
  int* used;  // per slot: 1 once claimed (the side slot's marker)
  unsigned long long* st[kGsMaxStates];
  int* hi[kGsMaxStates];
  uint64_t mask;
};

__device__ __forceinline__ long long ld_key(const GsSpec& s, int64_t r) {
  return s.key_bytes == 4 ? (long long)__ldcs((const int32_t*)s.key + r) : __ldcs((const long long*)s.key + r);
}
__device__ __forceinline__ long long ld_v(const GsSpec& s, int c, int64_t r) {
  return s.vbytes[c] == 4 ? (long long)__ldcs((const int32_t*)s.val[c] + r) : __ldcs((const long long*)s.val[c] + r);
}
__device__ __forceinline__ long long pick(const long long (&v)[kGsMaxVals], int c) {
  return c == 0 ? v[0] : c == 1 ? v[1] : c == 2 ? v[2] : v[3];  // (no dynamic register indexing)
}
__device__ __forceinline__ bool small_v(long long v) { return ((unsigned)((int32_t)(v >> 32) + 256) >> 9) == 0; }

// shared table: keys[S + 1] then nst arrays of S + 1 u64 (slot S = side slot for kEmptyKey)
struct STab {
  long long* keys;
  unsigned long long* st;  // [nst][S + 1]
  uint32_t S;
  __device__ __forceinline__ unsigned long long* state(int a, uint32_t slot) const { return st + (size_t)a * (S + 1) + slot; }
};

__device__ __forceinline__ void stab_init(const STab& t, const GsSpec& s, int tid, int nt) {
  for (uint32_t i = tid; i <= t.S; i += nt) {
    t.keys[i] = kEmptyKey;
    for (int a = 0; a < s.nst; ++a)
      *t.state(a, i) = s.kind[a] == ST_MIN ? (unsigned long long)LLONG_MAX
                       : s.kind[a] == ST_MAX ? (unsigned long long)LLONG_MIN : 0ull;
  }
}

// slot of `k` in t (inserting it); S + 1 when the table is full
__device__ __forceinline__ uint32_t stab_slot(const STab& t, long long k) {
  if (k == kEmptyKey) return t.S;
  uint32_t h = (uint32_t)hash64((uint64_t)k) & (t.S - 1);
  for (uint32_t probes = 0; probes < t.S; ++probes) {
    const long long cur = t.keys[h];
    if (cur == k) return h;
    if (cur == kEmptyKey) {
      const long long old = (long long)atomicCAS((unsigned long long*)&t.keys[h], (unsigned long long)kEmptyKey,
                                                 (unsigned long long)k);
      if (old == kEmptyKey || old == k) return h;
    }
    h = (h + 1) & (t.S - 1);
  }
  return t.S + 1;
}

// Shared-memory state updates with 32-bit atomics: on sm_100a a 64-bit shared atomicAdd / Min /
// Max compiles to a CAS spin loop (SASS ATOMS.CAST.SPIN.64).  SUM keeps {u32 lo, i32 hi} in the
// state word (v = hi * 2^32 + lo for |v| < 2^40; the carry of lo goes into hi; |sum| < 2^62 for
// <= 2^22 rows), COUNT a u32 in the low word, MIN/MAX the 64-bit value updated by CAS only when
// the row improves on the value read (rare after the first rows of a group).
__device__ __forceinline__ void stab_update(const STab& t, const GsSpec& s, uint32_t slot, const long long (&v)[kGsMaxVals]) {
#pragma unroll
  for (int a = 0; a < kGsMaxStates; ++a) {
    if (a >= s.nst) break;
    unsigned long long* p = t.state(a, slot);
    switch (s.kind[a]) {
      case ST_SUM: {
        const long long x = pick(v, s.vc[a]);
        const unsigned lo = (unsigned)x;
        const int hi = (int)(x >> 32);
        const unsigned old = atomicAdd((unsigned*)p, lo);
        const int h = hi + (old + lo < old ? 1 : 0);
        if (h) atomicAdd((int*)p + 1, h);
        break;
      }
      case ST_COUNT: atomicAdd((unsigned*)p, 1u); break;
      case ST_MIN: {
        const long long x = pick(v, s.vc[a]);
        long long cur = *(volatile long long*)p;
        while (x < cur) {
          const long long old = (long long)atomicCAS(p, (unsigned long long)cur, (unsigned long long)x);
          if (old == cur) break;
          cur = old;
        }
        break;
      }
      default: {
        const long long x = pick(v, s.vc[a]);
        long long cur = *(volatile long long*)p;
        while (x > cur) {
          const long long old = (long long)atomicCAS(p, (unsigned long long)cur, (unsigned long long)x);
          if (old == cur) break;
          cur = old;
        }
        break;
      }
    }
  }
}

// Compile-time state signature for the common one-value-column shape: states in the canonical
// order COUNT, [SUM], [MIN], [MAX] of value column 0 (straight-line per-row code); SigRt runs the
// runtime state list.
struct SigRt {
  static constexpr bool kFixed = false;
};
template <bool SUM, bool MIN, bool MAX>
struct SigFix {
  static constexpr bool kFixed = true, kHasSum = SUM, kHasMin = MIN, kHasMax = MAX;
  static constexpr int kSum = 1, kMin = 1 + SUM, kMax = 1 + SUM + MIN;
};

__device__ __forceinline__ void sh_sum(unsigned long long* p, long long x) {
  const unsigned lo = (unsigned)x;
  const int hi = (int)(x >> 32);
  const unsigned old = atomicAdd((unsigned*)p, lo);
  const int h = hi + (old + lo < old ? 1 : 0);
  if (h) atomicAdd((int*)p + 1, h);
}
__device__ __forceinline__ void sh_min(unsigned long long* p, long long x) {
  long long cur = *(volatile long long*)p;
  while (x < cur) {
    const long long old = (long long)atomicCAS(p, (unsigned long long)cur, (unsigned long long)x);
    if (old == cur) break;
    cur = old;
  }
}
__device__ __forceinline__ void sh_max(unsigned long long* p, long long x) {
  long long cur = *(volatile long long*)p;
  while (x > cur) {
    const long long old = (long long)atomicCAS(p, (unsigned long long)cur, (unsigned long long)x);
    if (old == cur) break;
    cur = old;
  }
}

template <class SIG>
__device__ __forceinline__ void stab_update_t(const STab& t, const GsSpec& s, uint32_t slot,
                                              const long long (&v)[kGsMaxVals]) {
  if constexpr (SIG::kFixed) {
    atomicAdd((unsigned*)t.state(0, slot), 1u);
    if constexpr (SIG::kHasSum) sh_sum(t.state(SIG::kSum, slot), v[0]);
    if constexpr (SIG::kHasMin) sh_min(t.state(SIG::kMin, slot), v[0]);
    if constexpr (SIG::kHasMax) sh_max(t.state(SIG::kMax, slot), v[0]);
  } else {
    stab_update(t, s, slot, v);
  }
}

// a shared state word as its value (SUM: hi * 2^32 + lo; COUNT: the low word; MIN/MAX as stored)
__device__ __forceinline__ unsigned long long stab_value(int kind, unsigned long long w) {
  if (kind == ST_SUM) return (unsigned long long)(((long long)(int)(w >> 32) << 32) + (long long)(unsigned)w);
  if (kind == ST_COUNT) return (unsigned long long)(unsigned)w;
  return w;
}

// ---- global merge table --------------------------------------------------------------------
__device__ __forceinline__ uint64_t g_slot(const GsGlobal& g, long long k, int* flags) {
  if (k == kEmptyKey) {
    g.used[g.mask + 1] = 1;
    return g.mask + 1;
  }
  uint64_t h = hash64((uint64_t)k) & g.mask;
  for (uint64_t probes = 0; probes <= g.mask; ++probes) {
    const unsigned long long old = atomicCAS(&g.keys[h], (unsigned long long)kEmptyKey, (unsigned long long)k);
    if (old == (unsigned long long)kEmptyKey || old == (unsigned long long)k) return h;
    h = (h + 1) & g.mask;
  }
  atomicExch(flags, 1);  // more groups than the hint allowed for: the host takes the generic path
  return g.mask + 1;
}

__device__ __forceinline__ void g_add(const GsGlobal& g, const GsSpec& s, uint64_t slot, int a, unsigned long long x,
                                      bool x_is_sum) {
  switch (s.kind[a]) {
    case ST_SUM:
      if (x_is_sum) atomic_add_i64_to_sum96(g.st[a] + slot, g.hi[a] + slot, (long long)x);
      break;
    case ST_COUNT: atomicAdd(g.st[a] + slot, x); break;
    case ST_MIN: atomicMin((long long*)g.st[a] + slot, (long long)x); break;
    default: atomicMax((long long*)g.st[a] + slot, (long long)x); break;
  }
}

// exact single-row update of the global table (a value >= 2^40: not summed in shared memory)
__device__ __forceinline__ void g_row(const GsGlobal& g, const GsSpec& s, long long k, const long long (&v)[kGsMaxVals]) {
  const uint64_t slot = g_slot(g, k, s.flags);
  for (int a = 0; a < s.nst; ++a)
    g_add(g, s, slot, a, s.kind[a] == ST_COUNT ? 1ull : (unsigned long long)pick(v, s.vc[a]), true);
}

// ---- K18s ----------------------------------------------------------------------------------
template <class SIG>
__global__ void __launch_bounds__(kGsThreads) k_gbs_local(const __grid_constant__ GsSpec s, int64_t n, int64_t chunk,
                                                          uint32_t S, int R, const __grid_constant__ GsGlobal g) {
  extern __shared__ __align__(16) unsigned char smem[];
  const size_t tab_bytes = (size_t)(S + 1) * 8 * (1 + s.nst);
  const int lane = threadIdx.x & 31;
  STab t;
  t.S = S;
  t.keys = (long long*)(smem + (size_t)(lane % R) * tab_bytes);
  t.st = (unsigned long long*)(t.keys + (S + 1));
  for (int r = 0; r < R; ++r) {
    STab x;
    x.S = S;
    x.keys = (long long*)(smem + (size_t)r * tab_bytes);
    x.st = (unsigned long long*)(x.keys + (S + 1));
    stab_init(x, s, threadIdx.x, blockDim.x);
  }
  __syncthreads();
  const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  bool full = false;
  constexpr int U = 4;
  for (int64_t b = lo; b < hi; b += (int64_t)U * blockDim.x) {
    long long k[U], v[U][kGsMaxVals];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = b + (int64_t)u * blockDim.x + threadIdx.x;
      const bool in = r < hi;
      k[u] = in ? ld_key(s, r) : 0;
#pragma unroll
      for (int c = 0; c < kGsMaxVals; ++c) v[u][c] = (in && c < (SIG::kFixed ? 1 : s.nv)) ? ld_v(s, c, r) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = b + (int64_t)u * blockDim.x + threadIdx.x;
      if (r >= hi) continue;
      bool sm = true;
#pragma unroll
      for (int c = 0; c < kGsMaxVals; ++c) sm = sm && (c >= (SIG::kFixed ? 1 : s.nv) || small_v(v[u][c]));
      if (!sm) {
        g_row(g, s, k[u], v[u]);
        continue;
      }
      const uint32_t slot = stab_slot(t, k[u]);
      if (slot > S) {
        full = true;
        continue;
      }
      stab_update_t<SIG>(t, s, slot, v[u]);
    }
  }
  if (full) atomicExch(s.flags, 1);
  __syncthreads();
  // merge every replica into the global table
  for (int r = 0; r < R; ++r) {
    STab x;
    x.S = S;
    x.keys = (long long*)(smem + (size_t)r * tab_bytes);
    x.st = (unsigned long long*)(x.keys + (S + 1));
    for (uint32_t i = threadIdx.x; i <= S; i += blockDim.x) {
      const long long key = x.keys[i];
      // (the side slot holds the key kEmptyKey; its count tells whether it was used)
      const bool used = i < S ? key != kEmptyKey : (unsigned)*x.state(s.count_state, i) != 0;
      if (!used) continue;
      const uint64_t gs = g_slot(g, i < S ? key : kEmptyKey, s.flags);
      for (int a = 0; a < s.nst; ++a) g_add(g, s, gs, a, stab_value(s.kind[a], *x.state(a, i)), true);
    }
  }
}

__global__ void k_gbs_init(const __grid_constant__ GsSpec s, const __grid_constant__ GsGlobal g) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= g.mask + 1; i += (uint64_t)gridDim.x * blockDim.x) {
    g.keys[i] = (unsigned long long)kEmptyKey;
    g.used[i] = 0;
    for (int a = 0; a < s.nst; ++a) {
      g.st[a][i] = s.kind[a] == ST_MIN ? (unsigned long long)LLONG_MAX
                   : s.kind[a] == ST_MAX ? (unsigned long long)LLONG_MIN : 0ull;
      if (g.hi[a]) g.hi[a][i] = 0;
    }
  }
}

__device__ __forceinline__ void put_out_key(const GsSpec& s, int64_t i, long long k) {
  if (s.key_bytes == 4) ((int32_t*)s.out_key)[i] = (int32_t)k;
  else ((long long*)s.out_key)[i] = k;
}

// one output row from states (lo, hi per state)
__device__ __forceinline__ void put_out_aggs(const GsSpec& s, int64_t i, const unsigned long long (&lo)[kGsMaxStates],
                                             const long long (&hi)[kGsMaxStates]) {
  const unsigned long long count = s.count_state >= 0 ? lo[s.count_state] : 0;
  for (int j = 0; j < s.naggs; ++j) {
    const int a = s.agg_state[j];
    switch (s.agg_op[j]) {
      case SX_SUM: ((longlong2*)s.out_agg[j])[i] = make_longlong2((long long)lo[a], hi[a]); break;
      case SX_COUNT: ((long long*)s.out_agg[j])[i] = (long long)count; break;
      case SX_MIN:
      case SX_MAX: ((long long*)s.out_agg[j])[i] = (long long)lo[a]; break;
      default: {  // AVG = (double)sum / (double)count / 10^scale (reading R3)
        double sc = 1.0;
        for (int q = 0; q < s.agg_scale[j]; ++q) sc *= 10.0;
        ((double*)s.out_agg[j])[i] = i128_to_double(lo[a], hi[a]) / (double)count / sc;
        break;
      }
    }
  }
}

__global__ void k_gbs_emit(const __grid_constant__ GsSpec s, const __grid_constant__ GsGlobal g) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= g.mask + 1; i += (uint64_t)gridDim.x * blockDim.x) {
    const bool used = i <= g.mask ? g.keys[i] != (unsigned long long)kEmptyKey : g.used[i] != 0;
    if (!used) continue;
    const unsigned long long pos = atomicAdd(s.out_cursor, 1ull);
    if ((int64_t)pos >= s.out_cap) continue;
    unsigned long long lo[kGsMaxStates];
    long long hi[kGsMaxStates];
    for (int a = 0; a < kGsMaxStates; ++a) {
      lo[a] = a < s.nst ? g.st[a][i] : 0;
      hi[a] = (a < s.nst && s.kind[a] == ST_SUM) ? (long long)g.hi[a][i] : 0;
    }
    put_out_key(s, (int64_t)pos, i <= g.mask ? (long long)g.keys[i] : kEmptyKey);
    put_out_aggs(s, (int64_t)pos, lo, hi);
  }
}

// ---- K18p ----------------------------------------------------------------------------------
// One CTA per partition (grid-stride over partitions): shared table of kGsPartSlots slots, the
// partition's rows [off[p], off[p+1]) of the partitioned key/value columns, then its groups are
// appended to the output (one atomic per CTA).
template <class SIG>
// R replicas of an S-slot table per CTA (warp w uses replica w % R): with few groups per partition
// (e.g. 64 for G = 2^16 over 1024 partitions) one table put 512 threads on the same few shared
// words (ncu: 38% barrier/serialisation stalls).  The replicas are merged into replica 0 (shared
// atomics) before its groups are written.
__global__ void __launch_bounds__(kGsThreads) k_gbs_part(const __grid_constant__ GsSpec s, const int64_t* __restrict__ off,
                                                         int P, uint32_t S, int R, const __grid_constant__ GsGlobal g,
                                                         unsigned* work) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_cnt;
  __shared__ unsigned long long s_base;
  const size_t tab_bytes = (size_t)(S + 1) * 8 * (1 + s.nst);
  auto rep = [&](int r) {
    STab x;
    x.S = S;
    x.keys = (long long*)(smem + (size_t)r * tab_bytes);
    x.st = (unsigned long long*)(x.keys + (S + 1));
    return x;
  };
  STab t = rep((threadIdx.x >> 5) % R);
  const STab t0 = rep(0);
  // partitions are claimed one at a time from a global counter (a static round-robin left the
  // CTAs that drew one partition more running alone: ncu r2x_gb64k, SM cycles max 1.5x avg)
  __shared__ int s_p;
  for (;;) {
    if (threadIdx.x == 0) s_p = (int)atomicAdd(work, 1u);
    __syncthreads();
    const int p = s_p;
    if (p >= P) break;
    for (int r = 0; r < R; ++r) stab_init(rep(r), s, threadIdx.x, blockDim.x);
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    const int64_t lo = off[p], hi = off[p + 1];
    bool full = false;
    constexpr int U = 4;
    for (int64_t b = lo; b < hi; b += (int64_t)U * blockDim.x) {
      long long k[U], v[U][kGsMaxVals];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t r = b + (int64_t)u * blockDim.x + threadIdx.x;
        const bool in = r < hi;
        k[u] = in ? ld_key(s, r) : 0;
#pragma unroll
        for (int c = 0; c < kGsMaxVals; ++c) v[u][c] = (in && c < (SIG::kFixed ? 1 : s.nv)) ? ld_v(s, c, r) : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t r = b + (int64_t)u * blockDim.x + threadIdx.x;
        if (r >= hi) continue;
        bool sm = true;
#pragma unroll
        for (int c = 0; c < kGsMaxVals; ++c) sm = sm && (c >= (SIG::kFixed ? 1 : s.nv) || small_v(v[u][c]));
        if (!sm) {
          full = true;  // exactness needs the 96-bit path: the host reruns generically
          continue;
        }
        const uint32_t slot = stab_slot(t, k[u]);
        if (slot > t.S) {
          full = true;
          continue;
        }
        stab_update_t<SIG>(t, s, slot, v[u]);
      }
    }
    __syncthreads();
    // replicas 1.. into replica 0
    for (uint32_t e = threadIdx.x; e < (uint32_t)(R - 1) * (S + 1); e += blockDim.x) {
      const STab x = rep(1 + (int)(e / (S + 1)));
      const uint32_t i = e % (S + 1);
      const bool used = i < S ? x.keys[i] != kEmptyKey : (unsigned)*x.state(s.count_state, i) != 0;
      if (!used) continue;
      const uint32_t d = i < S ? stab_slot(t0, x.keys[i]) : S;
      if (d > S) {
        full = true;
        continue;
      }
      for (int a = 0; a < s.nst; ++a) {
        const unsigned long long wv = *x.state(a, i);
        unsigned long long* dp = t0.state(a, d);
        switch (s.kind[a]) {
          case ST_SUM: sh_sum(dp, (long long)stab_value(ST_SUM, wv)); break;
          case ST_COUNT: atomicAdd((unsigned*)dp, (unsigned)wv); break;
          case ST_MIN: sh_min(dp, (long long)wv); break;
          default: sh_max(dp, (long long)wv); break;
        }
      }
    }
    if (full) atomicExch(s.flags, 1);
    __syncthreads();
    // count used slots, claim an output run, write the groups
    t = t0;
    for (uint32_t i = threadIdx.x; i <= t.S; i += blockDim.x) {
      const bool used = i < t.S ? t.keys[i] != kEmptyKey : (unsigned)*t.state(s.count_state, i) != 0;
      if (used) atomicAdd(&s_cnt, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = atomicAdd(s.out_cursor, (unsigned long long)s_cnt);
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i <= t.S; i += blockDim.x) {
      const bool used = i < t.S ? t.keys[i] != kEmptyKey : (unsigned)*t.state(s.count_state, i) != 0;
      if (!used) continue;
      const int64_t pos = (int64_t)s_base + atomicAdd(&s_cnt, 1);
      if (pos >= s.out_cap) continue;
      unsigned long long lo[kGsMaxStates];
      long long hi[kGsMaxStates];
      for (int a = 0; a < kGsMaxStates; ++a) {
        lo[a] = a < s.nst ? stab_value(s.kind[a], *t.state(a, i)) : 0;
        hi[a] = (a < s.nst && s.kind[a] == ST_SUM) ? ((long long)lo[a] < 0 ? -1 : 0) : 0;
      }
      put_out_key(s, pos, i < t.S ? t.keys[i] : kEmptyKey);
      put_out_aggs(s, pos, lo, hi);
    }
    t = rep((threadIdx.x >> 5) % R);
    __syncthreads();
  }
  (void)g;
}

// K18p2's second level: each CTA takes whole level-1 partitions (contiguous rows) and splits each
// into kSub sub-partitions by hash bits 43..47 (disjoint from the level-1 bits 48..57 and the
// shared-table slot bits 0..11): a shared histogram, its scan (the sub-partitions' offsets), then a
// scatter of the key and value columns inside the partition's own range of the output.
constexpr int kSubBits = 5, kSub = 1 << kSubBits;
__global__ void __launch_bounds__(kGsThreads) k_gbs_subpart(const __grid_constant__ GsSpec s,
                                                            const int64_t* __restrict__ off1, int P1, int nv,
                                                            const __grid_constant__ GsSpec d, int64_t* __restrict__ off2) {
  __shared__ int cnt[kSub];
  __shared__ int64_t start[kSub];
  __shared__ int cur[kSub];
  for (int p = blockIdx.x; p < P1; p += gridDim.x) {
    const int64_t lo = off1[p], hi = off1[p + 1];
    if (threadIdx.x < kSub) cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t r = lo + threadIdx.x; r < hi; r += blockDim.x)
      atomicAdd(&cnt[(hash64((uint64_t)ld_key(s, r)) >> 43) & (kSub - 1)], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t run = lo;
      for (int b = 0; b < kSub; ++b) {
        start[b] = run;
        off2[(int64_t)p * kSub + b] = run;
        run += cnt[b];
        cur[b] = 0;
      }
      if (p == P1 - 1) off2[(int64_t)P1 * kSub] = run;
    }
    __syncthreads();
    for (int64_t r = lo + threadIdx.x; r < hi; r += blockDim.x) {
      const long long k = ld_key(s, r);
      const int b = (int)((hash64((uint64_t)k) >> 43) & (kSub - 1));
      const int64_t pos = start[b] + atomicAdd(&cur[b], 1);
      if (s.key_bytes == 4) ((int32_t*)d.key)[pos] = (int32_t)k;
      else ((long long*)d.key)[pos] = k;
      for (int c = 0; c < nv; ++c) {
        if (s.vbytes[c] == 4) ((int32_t*)d.val[c])[pos] = __ldcs((const int32_t*)s.val[c] + r);
        else ((long long*)d.val[c])[pos] = __ldcs((const long long*)s.val[c] + r);
      }
    }
    __syncthreads();
  }
}

// ---- K19: warp-private aggregation without returning shared atomics ---------------------
// ncu on K18s at G = 4 (r2r_gb4): 24 ms for 2^30 rows, 755 GB/s — a shared atomic whose old
// value is used costs ~2 cycles per lane (B300_MICROARCH "ATOMS spread-addr"), and K18's SUM
// needs the old word for its carry.  K19t updates COUNT and SUM with plain loads and stores: every
// warp owns a dictionary key -> dense id (<= D ids: 16 or 48) and LANE-PRIVATE cells [id][lane], so no
// two lanes (and no two warps) ever write the same count/sum word; MIN/MAX are lane-private too
// (16 ids) or live per warp and id and change only when a row improves on them (48 ids: a shared
// CAS, rare after a group's first rows) — see GtWarp for the measured choice.
// The common row costs one dictionary read (home slot or the next) and the cell updates; a batch
// whose rows all qualify takes that fast path, any other batch (a key's first rows, a displaced
// key, a wide value, the key kEmptyKey, groups beyond D) the general per-row path, where rows
// without a cell take g_row's exact global atomics.  Above D hinted groups the input is first
// radix-partitioned (K7) to ~4 (16 ids) or ~16 (48 ids) groups per partition, so a warp's chunk of
// one partition fits its cells.  A warp aggregates one chunk of rows (never spanning two partitions), reduces each id's
// cells over its lanes and merges the group into the global table (one atomic per group and
// state, K18s's merge table), which k_gbs_emit turns into the output.  Exactness as K18 (R2/R3):
// a chunk has <= 2^21 rows and only values with |v| < 2^40 are summed in the 64-bit cells.
constexpr int kGwThreads = 256;  // (12 warps per CTA measured slower: 5.9 vs 5.2 ms at G = 4)
constexpr int kGwWarps = kGwThreads / 32;
constexpr int kGwU = 8;       // rows per lane per batch (their loads issued together)
constexpr int kGtSlots = 256;  // K19t: dictionary slots per warp (load <= 1/16: keys stay home)

// multiplicative slot hash (top bits; independent of hash64's partition bits 48..57)
__device__ __forceinline__ uint32_t gw_hash(long long k) {
  const uint64_t x = (uint64_t)k;
  return (uint32_t)x * 0x9E3779B1u + (uint32_t)(x >> 32) * 0x85EBCA77u + ((uint32_t)(x >> 32) >> 15);
}

// Read-only probe of a warp table (S slots, power of two; slot S = the side slot of kEmptyKey,
// present when has_side).  slot >= 0: found; miss: the key is absent (insert it); neither: the
// table is full (S probes).
__device__ __forceinline__ int gw_probe(const long long* keys, uint32_t S, int shift, long long k, bool act, bool has_side,
                                        bool& miss) {
  int slot = -1;
  miss = false;
  bool pend = act && k != kEmptyKey;
  if (act && k == kEmptyKey) {
    if (has_side) slot = (int)S;
    else miss = true;
  }
  uint32_t h = gw_hash(k) >> shift, probes = 0;
  while (__any_sync(kFull, pend)) {
    if (pend) {
      const long long cur = keys[h];
      if (cur == k) {
        slot = (int)h;
        pend = false;
      } else if (cur == kEmptyKey) {
        miss = true;
        pend = false;
      } else {
        h = (h + 1) & (S - 1);
        if (++probes >= S) pend = false;
      }
    }
  }
  return slot;
}

// Insert path (lanes with ins; warp-synchronous): returns the slot, -1 when the table is full.
__device__ __forceinline__ int gw_insert(long long* keys, uint32_t S, int shift, long long k, bool ins) {
  int slot = -1;
  bool pend = ins && k != kEmptyKey;
  if (ins && k == kEmptyKey) slot = (int)S;
  uint32_t h = gw_hash(k) >> shift, probes = 0;
  while (__any_sync(kFull, pend)) {
    const long long cur = pend ? keys[h] : 0;
    __syncwarp();
    const bool wrote = pend && cur == kEmptyKey;
    if (wrote) keys[h] = k;
    __syncwarp();
    if (pend) {
      const long long now = wrote ? keys[h] : cur;
      if (now == k) {
        slot = (int)h;
        pend = false;
      } else {
        h = (h + 1) & (S - 1);
        if (++probes >= S) pend = false;
      }
    }
  }
  __syncwarp();
  return slot;
}

struct GwChunks {
  const int64_t* lo;  // [nchunks] first row
  const int64_t* hi;  // [nchunks] end row
  int nchunks;
};

template <int KB, int VB>
__device__ __forceinline__ void gw_load(const GsSpec& s, int64_t b, int64_t hi, int lane, long long (&k)[kGwU],
                                        long long (&v)[kGwU], bool (&in)[kGwU]) {
#pragma unroll
  for (int u = 0; u < kGwU; ++u) {
    const int64_t r = b + (int64_t)u * 32 + lane;
    in[u] = r < hi;
    if constexpr (KB == 8) k[u] = in[u] ? __ldcs((const long long*)s.key + r) : 0;
    else k[u] = in[u] ? (long long)__ldcs((const int32_t*)s.key + r) : 0;
    if constexpr (VB == 8) v[u] = in[u] ? __ldcs((const long long*)s.val[0] + r) : 0;
    else v[u] = in[u] ? (long long)__ldcs((const int32_t*)s.val[0] + r) : 0;
  }
}

template <class SIG>
__device__ __forceinline__ void gw_merge_group(const GsGlobal& g, const GsSpec& s, long long key, unsigned long long cnt,
                                               long long sum, long long mn, long long mx) {
  const uint64_t gs = g_slot(g, key, s.flags);
  g_add(g, s, gs, 0, cnt, true);
  if constexpr (SIG::kHasSum) g_add(g, s, gs, SIG::kSum, (unsigned long long)sum, true);
  if constexpr (SIG::kHasMin) g_add(g, s, gs, SIG::kMin, (unsigned long long)mn, true);
  if constexpr (SIG::kHasMax) g_add(g, s, gs, SIG::kMax, (unsigned long long)mx, true);
}

// K19t.  Per warp: dictionary keys[kGtSlots + 1] / ids (int8: -1 none, D overflow), id -> key,
// lane-private cells cnt[D][32] u32 and sum[D][32] i64, and MIN/MAX either lane-private too (LP:
// [D][32] i64 each — conflict-free stores, but 16 B per id and lane held the warp to 16 ids) or
// per warp and id (!LP: a row changes them only when it improves on the value read, by a shared
// CAS — rare after a group's first rows — which lets a warp hold 48 ids).  Measured (2^30 rows):
// G = 4..16 direct 5.2 ms <16, LP> vs 6.9 <48>; G = 32 direct 8.3 <48> (K18s 10.6); G = 64..1024
// at ~4 groups per partition <16, LP> 17-21 ms vs 21-22 at ~16 <48>; G = 2048..16384 at ~16 per
// partition <48> 23 / 25 / 35 / 43 ms vs 29 / 36 / 53 / 54 (profiles/r02_mb_gb_variants_v3.txt).
template <int D, bool LP>
struct GtWarp {
  long long keys[kGtSlots + 4];
  long long idkey[D];
  long long sum[D + 1][32];  // (row D: the sink of the fast path's inactive rows)
  unsigned cnt[D + 1][32];
  long long mn[D + 1][LP ? 32 : 1];
  long long mx[D + 1][LP ? 32 : 1];
  signed char id[kGtSlots + 4];
};
constexpr int kGtShift = 32 - 8;  // log2(kGtSlots)

template <class SIG, int D, bool LP>
__device__ __forceinline__ void gt_cell(GtWarp<D, LP>& W, int id, int lane, long long v) {
  W.cnt[id][lane] += 1u;
  if constexpr (SIG::kHasSum) W.sum[id][lane] += v;
  if constexpr (LP) {
    if constexpr (SIG::kHasMin) W.mn[id][lane] = min(W.mn[id][lane], v);
    if constexpr (SIG::kHasMax) W.mx[id][lane] = max(W.mx[id][lane], v);
  } else {
    if constexpr (SIG::kHasMin) {
      long long cur = W.mn[id][0];
      while (v < cur) {
        const long long old = (long long)atomicCAS((unsigned long long*)&W.mn[id][0], (unsigned long long)cur,
                                                   (unsigned long long)v);
        if (old == cur) break;
        cur = old;
      }
    }
    if constexpr (SIG::kHasMax) {
      long long cur = W.mx[id][0];
      while (v > cur) {
        const long long old = (long long)atomicCAS((unsigned long long*)&W.mx[id][0], (unsigned long long)cur,
                                                   (unsigned long long)v);
        if (old == cur) break;
        cur = old;
      }
    }
  }
}

// The general per-row path (a key's first rows, displaced keys, wide values, the key
// kEmptyKey, more than D groups in the chunk: those rows take g_row's global atomics).
template <class SIG, int D, bool LP>
__device__ __noinline__ void gt_slow_batch(GtWarp<D, LP>& W, const GsSpec& s, const GsGlobal& g, int lane, int& nid,
                                           bool& side, const long long (&k)[kGwU], const long long (&v)[kGwU],
                                           const bool (&in)[kGwU]) {
#pragma unroll 1
  for (int u = 0; u < kGwU; ++u) {
    const long long ku = k[u], vu = v[u];
    bool act = in[u];
    bool wide = act && !small_v(vu);
    act = act && !wide;
    bool miss;
    int slot = gw_probe(W.keys, kGtSlots, kGtShift, ku, act, side, miss);
    if (__any_sync(kFull, miss)) {  // first rows of new keys: insert, one id per new slot
      const int ns = gw_insert(W.keys, kGtSlots, kGtShift, ku, miss);
      if (miss) slot = ns;
      const bool need = miss && ns >= 0 && W.id[ns] < 0;
      const unsigned nm = __ballot_sync(kFull, need);
      bool lead = false;
      if (need) lead = (__ffs(__match_any_sync(nm, ns)) - 1) == lane;
      const unsigned lm = __ballot_sync(kFull, lead);
      if (lead) {
        const int nidx = nid + __popc(lm & lanemask_lt());
        W.id[ns] = (signed char)(nidx < D ? nidx : D);
        if (nidx < D) W.idkey[nidx] = ku;
      }
      nid += __popc(lm);
      side = side || __any_sync(kFull, miss && ku == kEmptyKey);
      __syncwarp();
    }
    const int id = slot >= 0 ? W.id[slot] : -1;
    if (act && (id < 0 || id >= D)) wide = true;  // no cell: the exact global path
    if (wide) {
      long long vv[kGsMaxVals] = {vu, 0, 0, 0};
      g_row(g, s, ku, vv);
    } else if (act) {
      gt_cell<SIG, D, LP>(W, id, lane, vu);
    }
    __syncwarp();
  }
}

template <class SIG, int KB, int VB, int D, bool LP>
__global__ void __launch_bounds__(kGwThreads) k_gbt(const __grid_constant__ GsSpec s, const __grid_constant__ GwChunks ch,
                                                    const __grid_constant__ GsGlobal g, unsigned* work) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  GtWarp<D, LP>& W = ((GtWarp<D, LP>*)smem)[threadIdx.x >> 5];
  const int gw = blockIdx.x * kGwWarps + (threadIdx.x >> 5), nw = gridDim.x * kGwWarps;
  (void)gw;
  (void)nw;
  for (;;) {  // chunks claimed one at a time per warp (balances partition tails and slow chunks)
    int c = 0;
    if (lane == 0) c = (int)atomicAdd(work, 1u);
    c = __shfl_sync(kFull, c, 0);
    if (c >= ch.nchunks) break;
    for (int i = lane; i < kGtSlots + 4; i += 32) {
      W.keys[i] = kEmptyKey;  // (slots kGtSlots + 1..3: never-used pads, probed as "home + 1..3")
      W.id[i] = -1;
    }
#pragma unroll
    for (int d = 0; d <= D; ++d) {
      W.cnt[d][lane] = 0;
      W.sum[d][lane] = 0;
      if constexpr (LP) {
        W.mn[d][lane] = LLONG_MAX;
        W.mx[d][lane] = LLONG_MIN;
      }
    }
    if constexpr (!LP)
      for (int d = lane; d <= D; d += 32) {
        W.mn[d][0] = LLONG_MAX;
        W.mx[d][0] = LLONG_MIN;
      }
    int nid = 0;
    bool side = false;  // the key kEmptyKey has an id
    __syncwarp();
    const int64_t lo = ch.lo[c], hi = ch.hi[c];
    long long k[kGwU], v[kGwU];
    bool in[kGwU];
    gw_load<KB, VB>(s, lo, hi, lane, k, v, in);
    for (int64_t b = lo; b < hi; b += 32 * kGwU) {
      long long kn[kGwU], vn[kGwU];
      bool inn[kGwU];
      gw_load<KB, VB>(s, b + 32 * kGwU, hi, lane, kn, vn, inn);
      // fast path: every row's key at its home slot or the next, with an id, and a small value
      // (branch-free: bitwise tests; a row past the chunk updates the sink row D)
      int id[kGwU];
      int ok = 1;
#pragma unroll
      for (int u = 0; u < kGwU; ++u) {
        const uint32_t h = gw_hash(k[u]) >> kGtShift;
        // the home slot and the next (<16>), or the next three (<48>: with up to ~48 keys in 256
        // slots a key sits two or more slots past home in ~6% of the chunks, which then ran the
        // slow path throughout: one SM 2x the average, ncu r2ba_gb8k)
        int iu;
        if constexpr (LP) {
          const long long c0 = W.keys[h], c1 = W.keys[h + 1];
          const int i0 = W.id[h], i1 = W.id[h + 1];
          iu = c0 == k[u] ? i0 : c1 == k[u] ? i1 : -1;
        } else {
          const long long c0 = W.keys[h], c1 = W.keys[h + 1], c2 = W.keys[h + 2], c3 = W.keys[h + 3];
          const int j = c0 == k[u] ? 0 : c1 == k[u] ? 1 : c2 == k[u] ? 2 : c3 == k[u] ? 3 : -1;
          iu = j >= 0 ? (int)W.id[h + j] : -1;
        }
        const int good = ((unsigned)iu < (unsigned)D) & (k[u] != kEmptyKey) & small_v(v[u]);
        ok &= (!in[u]) | good;
        id[u] = in[u] ? iu : D;
      }
      if (__all_sync(kFull, ok)) {
#pragma unroll
        for (int u = 0; u < kGwU; ++u) gt_cell<SIG, D, LP>(W, id[u], lane, v[u]);
      } else {
        gt_slow_batch<SIG, D, LP>(W, s, g, lane, nid, side, k, v, in);
      }
#pragma unroll
      for (int u = 0; u < kGwU; ++u) {
        k[u] = kn[u];
        v[u] = vn[u];
        in[u] = inn[u];
      }
    }
    __syncwarp();
    // the warp's groups: each id's cells reduced over the lanes; lane d merges group d
    const int nd = min(nid, D);
    for (int d = 0; d < nd; ++d) {
      unsigned cn = W.cnt[d][lane];
      long long sm = W.sum[d][lane];
      long long mn = W.mn[d][LP ? lane : 0], mx = W.mx[d][LP ? lane : 0];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        cn += __shfl_xor_sync(kFull, cn, o);
        sm += __shfl_xor_sync(kFull, sm, o);
        if constexpr (LP) {
          mn = min(mn, __shfl_xor_sync(kFull, mn, o));
          mx = max(mx, __shfl_xor_sync(kFull, mx, o));
        }
      }
      if (lane == (d & 31) && cn) gw_merge_group<SIG>(g, s, W.idkey[d], cn, sm, mn, mx);
    }
    __syncwarp();
  }
}

template <class F>
sx_status with_sig(int sig, F&& f) {
  switch (sig) {
    case 0: return f(SigFix<false, false, false>{});
    case 1: return f(SigFix<true, false, false>{});
    case 2: return f(SigFix<false, true, false>{});
    case 3: return f(SigFix<true, true, false>{});
    case 4: return f(SigFix<false, false, true>{});
    case 5: return f(SigFix<true, false, true>{});
    case 6: return f(SigFix<false, true, true>{});
    case 7: return f(SigFix<true, true, true>{});
    default: return f(SigRt{});
  }
}

bool plain_col_expr(const sx_expr& e, int* col) {
  if (e.nterms != 1 || e.t[0].coef != 1 || e.t[0].nf != 1) return false;
  const auto& f = e.t[0].f[0];
  if (f.mul != 1 || f.add != 0) return false;
  *col = f.col;
  return true;
}


// K19 host side (see the kernels): SX_EUNSUPPORTED (nothing allocated) when the shape does not
// fit (not the fixed signature, or more than kGtHintMax hinted groups) or the hinted global merge
// table overflowed.
constexpr int64_t kGtHintMax = 16384;  // 1024 partitions x ~16 groups
sx_status gb_k19(sx_ctx* ctx, GsSpec s, int sig, const sx_col& kc, int vtype, int naggs, const sx_agg* aggs,
                 int64_t groups_hint, int64_t n, sx_col* out_keys, sx_col* out_aggs, int64_t* out_ngroups) {
  if (sig < 0 || s.nv != 1 || groups_hint > kGtHintMax) return SX_EUNSUPPORTED;
  Scratch scr(ctx);
  // variant and fan-out (measured, see GtWarp): <16, LP> directly up to 16 hinted groups and at ~4
  // groups per partition for 49..1024; <48, !LP> directly for 17..48 and at ~16 per partition above
  // 1024 (SX_GB_K19V=48: <48> above 16, the A/B switch).  A partition's expected groups stay far below the warp's ids (rows of groups beyond them
  // take global atomics: with 16 ids and ~8 groups per partition, the few partitions past 16
  // groups made one warp's chunk 7x slower than the rest, ncu r2u_gb4k).
  bool big = (groups_hint > 16 && groups_hint <= 48) || groups_hint > 1024;
  if (getenv("SX_GB_K19V")) {  // A/B: 48 forces <48> above 16 groups, 16 keeps <16> above 48
    const int v = atoi(getenv("SX_GB_K19V"));
    big = v == 48 ? groups_hint > 16 : (groups_hint > 16 && groups_hint <= 48);
  }
  const int per = big ? 16 : 4, dmax = big ? 48 : 16;
  int bits = 0;
  while (bits < 10 && groups_hint > dmax && ((int64_t)per << bits) < groups_hint) ++bits;
  const int P = 1 << bits;
  std::vector<int64_t> offs{0, n};
  if (P > 1) {
    DCol kd{s.key, s.key_type, 0};
    DCol carry[2] = {kd, DCol{s.val[0], vtype, 0}};
    int width[2] = {s.key_bytes, s.vbytes[0]};
    void* outp[2];
    for (int c = 0; c < 2; ++c) SX_TRY(scr.get((char**)&outp[c], (size_t)n * width[c]));
    offs.assign((size_t)P + 1, 0);
    SX_TRY(radix_partition_carry(ctx, kd, kd, 1, carry, width, 2, nullptr, n, bits, outp, offs.data()));
    s.key = outp[0];
    s.val[0] = outp[1];
  }
  // chunks: ~4 per resident warp (partition tails even out), <= 2^21 rows (exact 64-bit warp
  // sums), never across partitions
  const int nwarps = ctx->num_sms * kGwWarps;
  const int64_t L = std::min<int64_t>(1 << 21, std::max<int64_t>(32 * kGwU, (n + 4 * nwarps - 1) / (4 * nwarps)));
  std::vector<int64_t> clo, chi;
  for (int p = 0; p < (int)offs.size() - 1; ++p)
    for (int64_t a = offs[p]; a < offs[p + 1]; a += L) {
      clo.push_back(a);
      chi.push_back(std::min(a + L, offs[p + 1]));
    }
  const int nch = (int)clo.size();
  int64_t* d_ch;
  SX_TRY(scr.get(&d_ch, (size_t)std::max(1, 2 * nch)));
  if (nch) {
    std::vector<int64_t> both(clo);
    both.insert(both.end(), chi.begin(), chi.end());
    SX_CUDA(cudaMemcpyAsync(d_ch, both.data(), sizeof(int64_t) * 2 * nch, cudaMemcpyHostToDevice, ctx->stream));
  }
  GwChunks ch{d_ch, d_ch + nch, nch};
  // global merge table (load <= 0.5 at the hint) and the outputs (every slot + the side slot)
  GsGlobal g{};
  uint64_t C = 64;
  while (C < (uint64_t)(2 * groups_hint)) C <<= 1;
  SX_TRY(scr.get(&g.keys, C + 1));
  SX_TRY(scr.get(&g.used, C + 1));
  for (int a = 0; a < s.nst; ++a) {
    SX_TRY(scr.get(&g.st[a], C + 1));
    g.hi[a] = nullptr;
    if (s.kind[a] == ST_SUM) SX_TRY(scr.get(&g.hi[a], C + 1));
  }
  g.mask = C - 1;
  const int64_t cap = (int64_t)std::min<uint64_t>((uint64_t)n, C + 1);
  void* okey;
  void* oagg[SX_MAX_AGGS];
  SX_TRY(scr.get((char**)&okey, (size_t)std::max<int64_t>(cap, 1) * s.key_bytes));
  for (int j = 0; j < naggs; ++j)
    SX_TRY(scr.get((char**)&oagg[j], (size_t)std::max<int64_t>(cap, 1) * type_width(agg_out_type(aggs[j].op))));
  s.out_key = okey;
  for (int j = 0; j < naggs; ++j) s.out_agg[j] = oagg[j];
  s.out_cap = cap;
  unsigned long long* cursor = (unsigned long long*)ctx->d_counters;
  s.out_cursor = cursor;
  s.flags = ctx->d_flags;
  SX_CUDA(cudaMemsetAsync(cursor, 0, 8, ctx->stream));
  SX_CUDA(cudaMemsetAsync(s.flags, 0, sizeof(int), ctx->stream));
  k_gbs_init<<<persistent_grid(ctx, 4, (C + kBlock) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(s, g);
  SX_CHECK_LAUNCH();
  SX_TRY(with_sig(sig, [&](auto sg) -> sx_status {
    using SIG = decltype(sg);
    if constexpr (!SIG::kFixed) {
      return SX_EUNSUPPORTED;
    } else {
      auto go = [&](auto kbc, auto vbc) -> sx_status {
        constexpr int KB = decltype(kbc)::value, VB = decltype(vbc)::value;
        auto launch = [&](auto kern, size_t wbytes) -> sx_status {
          const size_t smem = wbytes * kGwWarps;
          SX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          int per_sm = 1;
          SX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGwThreads, smem));
          const unsigned grid = (unsigned)std::max(1, std::min(nch, ctx->num_sms * std::max(1, per_sm)));
          SX_CUDA(cudaMemsetAsync(ctx->d_counters + 16, 0, sizeof(unsigned), ctx->stream));
          kern<<<grid, kGwThreads, smem, SX_STREAM(ctx)>>>(s, ch, g, ctx->d_counters + 16);
          return SX_OK;
        };
        if (big) SX_TRY(launch(k_gbt<SIG, KB, VB, 48, false>, sizeof(GtWarp<48, false>)));
        else SX_TRY(launch(k_gbt<SIG, KB, VB, 16, true>, sizeof(GtWarp<16, true>)));
        SX_CHECK_LAUNCH();
        return SX_OK;
      };
      using I4 = std::integral_constant<int, 4>;
      using I8 = std::integral_constant<int, 8>;
      if (s.key_bytes == 8) return s.vbytes[0] == 8 ? go(I8{}, I8{}) : go(I8{}, I4{});
      return s.vbytes[0] == 8 ? go(I4{}, I8{}) : go(I4{}, I4{});
    }
  }));
  k_gbs_emit<<<persistent_grid(ctx, 4, (C + kBlock) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(s, g);
  SX_CHECK_LAUNCH();
  int64_t ng = 0;
  SX_TRY(read_i64(ctx, cursor, &ng));
  int fl = 0;
  SX_CUDA(cudaMemcpy(&fl, s.flags, sizeof(int), cudaMemcpyDeviceToHost));
  if (fl || ng > cap) return SX_EUNSUPPORTED;  // a warp table / the hinted global table overflowed
  out_keys[0] = sx_col{kc.type, kc.scale, ng, okey, nullptr, nullptr};
  scr.release(okey);
  for (int j = 0; j < naggs; ++j) {
    out_aggs[j] = sx_col{agg_out_type(aggs[j].op), 0, ng, oagg[j], nullptr, nullptr};
    scr.release(oagg[j]);
  }
  *out_ngroups = ng;
  return SX_OK;
}
}  // namespace

namespace sx {

sx_status gb_simple(sx_ctx* ctx, const sx_col* cols, int ncols, const sx_key* keys, int nkeys, const sx_sel* in_sel,
                    int nwhere, const sx_agg* aggs, int naggs, const sx_having* having, int64_t groups_hint,
                    sx_col* out_keys, sx_col* out_aggs, int64_t* out_ngroups) {
  const bool off = getenv("SX_GB_SIMPLE") && getenv("SX_GB_SIMPLE")[0] == '0';
  if (off || nkeys != 1 || in_sel || nwhere || having || naggs < 1 || naggs > SX_MAX_AGGS || groups_hint < 1 ||
      groups_hint > (1 << 27))
    return SX_EUNSUPPORTED;
  if (keys[0].fn != SX_KEY_IDENTITY || keys[0].col < 0 || keys[0].col >= ncols) return SX_EUNSUPPORTED;
  const sx_col& kc = cols[keys[0].col];
  const int kt = kc.type;
  if (!(kt == SX_I32 || kt == SX_DATE32 || kt == SX_I64) || kc.validity) return SX_EUNSUPPORTED;
  const int64_t n = kc.len;
  if (n < (1 << 20) || n > INT32_MAX) return SX_EUNSUPPORTED;
  GsSpec s{};
  s.key = kc.data;
  s.key_bytes = kt == SX_I64 ? 8 : 4;
  s.key_type = kt;
  s.count_state = -1;
  int vcol_of[kGsMaxVals];
  auto vslot = [&](int col) -> int {
    for (int c = 0; c < s.nv; ++c)
      if (vcol_of[c] == col) return c;
    if (s.nv == kGsMaxVals) return -1;
    const sx_col& vc = cols[col];
    if (vc.len != n || vc.validity) return -1;
    const int w = (vc.type == SX_I64 || vc.type == SX_DEC64) ? 8 : (vc.type == SX_I32 || vc.type == SX_DATE32) ? 4 : 0;
    if (!w) return -1;
    vcol_of[s.nv] = col;
    s.val[s.nv] = vc.data;
    s.vbytes[s.nv] = w;
    return s.nv++;
  };
  auto state = [&](int kind, int vc) -> int {
    for (int a = 0; a < s.nst; ++a)
      if (s.kind[a] == kind && s.vc[a] == vc) return a;
    if (s.nst == kGsMaxStates) return -1;
    s.kind[s.nst] = kind;
    s.vc[s.nst] = vc;
    return s.nst++;
  };
  s.naggs = naggs;
  s.count_state = state(ST_COUNT, -1);  // always kept: it marks the side slot (key kEmptyKey) as used
  for (int j = 0; j < naggs; ++j) {
    const int op = aggs[j].op;
    s.agg_op[j] = op;
    s.agg_scale[j] = aggs[j].scale;
    if (op == SX_COUNT) {
      s.agg_state[j] = s.count_state;
      continue;
    }
    int col = -1;
    if (!plain_col_expr(aggs[j].value, &col) || col < 0 || col >= ncols) return SX_EUNSUPPORTED;
    const int vc = vslot(col);
    if (vc < 0) return SX_EUNSUPPORTED;
    const int kind = (op == SX_SUM || op == SX_AVG) ? ST_SUM : op == SX_MIN ? ST_MIN : op == SX_MAX ? ST_MAX : -1;
    if (kind < 0) return SX_EUNSUPPORTED;
    const int a = state(kind, vc);
    if (a < 0) return SX_EUNSUPPORTED;
    s.agg_state[j] = a;
  }
  // the fixed signature (one value column; COUNT, SUM, MIN, MAX at most once each): states in the
  // canonical order COUNT, SUM, MIN, MAX
  int sig = -1;  // bit 0 SUM, bit 1 MIN, bit 2 MAX
  if (s.nv == 1) {
    int seen[4] = {0, 0, 0, 0}, remap[kGsMaxStates];
    bool ok = true;
    for (int a = 0; a < s.nst; ++a) ok = ok && ++seen[s.kind[a]] == 1;
    if (ok) {
      const bool hs = seen[ST_SUM], hm = seen[ST_MIN], hx = seen[ST_MAX];
      const int idx[4] = {1, 0, 1 + hs, 1 + hs + hm};  // by kind: SUM, COUNT, MIN, MAX
      int kind[kGsMaxStates], vc[kGsMaxStates];
      for (int a = 0; a < s.nst; ++a) {
        remap[a] = idx[s.kind[a]];
        kind[remap[a]] = s.kind[a];
        vc[remap[a]] = s.vc[a];
      }
      for (int a = 0; a < s.nst; ++a) {
        s.kind[a] = kind[a];
        s.vc[a] = vc[a];
      }
      for (int j = 0; j < naggs; ++j) s.agg_state[j] = remap[s.agg_state[j]];
      s.count_state = 0;
      sig = (hs ? 1 : 0) | (hm ? 2 : 0) | (hx ? 4 : 0);
    }
  }
  for (int c = 0; c < s.nv; ++c)
    if ((uintptr_t)s.val[c] % 16) return SX_EUNSUPPORTED;
  if ((uintptr_t)s.key % 16) return SX_EUNSUPPORTED;
  // K19 (atomic-free warp tables) for the fixed signature up to 2^18 hinted groups (SX_GB_K19=0: K18)
  if (!(getenv("SX_GB_K19") && getenv("SX_GB_K19")[0] == '0')) {
    const sx_status k19 = gb_k19(ctx, s, sig, kc, s.nv == 1 ? cols[vcol_of[0]].type : 0, naggs, aggs, groups_hint, n,
                                 out_keys, out_aggs, out_ngroups);
    if (k19 != SX_EUNSUPPORTED) return k19;
    ctx->err.clear();
  }
  Scratch scr(ctx);
  // outputs (capacity from the hint; rerun with the exact count if it was low)
  int64_t cap = std::min<int64_t>(n, 2 * groups_hint + 1024);
  unsigned long long* cursor = (unsigned long long*)ctx->d_counters;
  s.out_cursor = cursor;
  s.flags = ctx->d_flags;
  // K18s while one CTA's replicated tables fit ~200 KB of shared memory (S = 2 x hint slots; the
  // partitioned path leaves 1-4 groups per partition for G ~ 2048-4096: every thread of the CTA
  // on the same few shared addresses, 172 ms for G = 2048), else K18p
  uint32_t S_loc = 16;
  while (S_loc < (uint32_t)(2 * groups_hint)) S_loc <<= 1;
  const bool part = (size_t)(S_loc + 1) * 8 * (1 + s.nst) > (200u << 10);
  // K18p partitioning (once, outside the capacity retry)
  int bits = 0;
  std::vector<int64_t> offs;
  int64_t* d_off = nullptr;
  int Pn = 0;  // partitions the shared tables aggregate
  if (part) {
    // fan-out 1024 (the partitioner's maximum): <= 2048 expected groups per shared table, and
    // enough partitions to spread over every SM whatever G is; above 2^21 groups a second level
    // (K18p2) splits every partition 32 ways
    // 512 partitions for 2^17..2^19 hinted groups (256..1024 per partition: 44 vs 57 ms for 2^30
    // rows, the 512-way scatter moves less partial-sector traffic); fewer groups per partition
    // put too many threads on too few shared words (2^13 groups over 512: 172 vs 52 ms), 256
    // partitions leave SMs idle (163-176 ms) — profiles/r02_mb_gb_variants_v3.txt
    bits = (groups_hint >= (1 << 17) && groups_hint <= (1 << 19)) ? 9 : 10;
    if (getenv("SX_GB_PBITS")) bits = std::max(6, std::min(10, atoi(getenv("SX_GB_PBITS"))));
    if ((groups_hint >> bits) > 2048) bits = 10;
    const bool two = (groups_hint >> bits) > 2048;
    if (two && (groups_hint >> (bits + kSubBits)) > 2048) return SX_EUNSUPPORTED;
    const int P = 1 << bits;
    DCol kd{kc.data, kt, 0};
    DCol carry[1 + kGsMaxVals];
    int width[1 + kGsMaxVals];
    void* outp[1 + kGsMaxVals];
    carry[0] = kd;
    width[0] = s.key_bytes;
    for (int c = 0; c < s.nv; ++c) {
      carry[1 + c] = DCol{s.val[c], cols[vcol_of[c]].type, 0};
      width[1 + c] = s.vbytes[c];
    }
    for (int c = 0; c <= s.nv; ++c) SX_TRY(scr.get((char**)&outp[c], (size_t)n * width[c]));
    offs.assign((size_t)P + 1, 0);
    SX_TRY(radix_partition_carry(ctx, kd, kd, 1, carry, width, 1 + s.nv, nullptr, n, bits, outp, offs.data()));
    // a partition sums in one CTA in the shared SUM words: <= 2^22 rows of |v| < 2^40 (skewed keys
    // beyond that take the generic path)
    for (int p = 0; p < P; ++p)
      if (offs[p + 1] - offs[p] > (1 << 22)) return SX_EUNSUPPORTED;
    s.key = outp[0];
    for (int c = 0; c < s.nv; ++c) s.val[c] = outp[1 + c];
    SX_TRY(scr.get(&d_off, (size_t)P + 1));
    SX_CUDA(cudaMemcpyAsync(d_off, offs.data(), sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice, ctx->stream));
    Pn = P;
    if (two) {
      GsSpec d2 = s;
      void* o2[1 + kGsMaxVals];
      for (int c = 0; c <= s.nv; ++c) SX_TRY(scr.get((char**)&o2[c], (size_t)n * width[c]));
      d2.key = o2[0];
      for (int c = 0; c < s.nv; ++c) d2.val[c] = o2[1 + c];
      int64_t* d_off2;
      SX_TRY(scr.get(&d_off2, (size_t)P * kSub + 1));
      k_gbs_subpart<<<persistent_grid(ctx, 2, P), kGsThreads, 0, SX_STREAM(ctx)>>>(s, d_off, P, s.nv, d2, d_off2);
      SX_CHECK_LAUNCH();
      s.key = d2.key;
      for (int c = 0; c < s.nv; ++c) s.val[c] = d2.val[c];
      d_off = d_off2;
      Pn = P * kSub;
    }
  }
  for (int attempt = 0; attempt < 2; ++attempt) {
    void* okey;
    void* oagg[SX_MAX_AGGS];
    SX_TRY(scr.get((char**)&okey, (size_t)std::max<int64_t>(cap, 1) * s.key_bytes));
    for (int j = 0; j < naggs; ++j) SX_TRY(scr.get((char**)&oagg[j], (size_t)std::max<int64_t>(cap, 1) * type_width(agg_out_type(aggs[j].op))));
    s.out_key = okey;
    for (int j = 0; j < naggs; ++j) s.out_agg[j] = oagg[j];
    s.out_cap = cap;
    SX_CUDA(cudaMemsetAsync(cursor, 0, 8, ctx->stream));
    SX_CUDA(cudaMemsetAsync(s.flags, 0, sizeof(int), ctx->stream));
    GsGlobal g{};
    if (part) {
      const int P = Pn;
      // per-partition table: 2 x the expected groups (>= 64 slots, <= kGsPartSlots), replicated
      // up to 16 ways within ~200 KB
      uint32_t Sp = 64;
      while (Sp < (uint32_t)kGsPartSlots && Sp < (uint32_t)(2 * (groups_hint / P + 1))) Sp <<= 1;
      const size_t tabp = (size_t)(Sp + 1) * 8 * (1 + s.nst);
      const int Rp = (int)std::max<size_t>(1, std::min<size_t>(16, (200u << 10) / tabp));
      const size_t smem = tabp * Rp;
      SX_TRY(with_sig(sig, [&](auto sg) -> sx_status {
        using SIG = decltype(sg);
        SX_CUDA(cudaFuncSetAttribute(k_gbs_part<SIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        SX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gbs_part<SIG>, kGsThreads, smem));
        const unsigned grid = (unsigned)std::min<int64_t>(P, (int64_t)ctx->num_sms * std::max(1, per_sm));
        SX_CUDA(cudaMemsetAsync(ctx->d_counters + 16, 0, sizeof(unsigned), ctx->stream));
        k_gbs_part<SIG><<<grid, kGsThreads, smem, SX_STREAM(ctx)>>>(s, d_off, P, Sp, Rp, g, ctx->d_counters + 16);
        SX_CHECK_LAUNCH();
        return SX_OK;
      }));
    } else {
      // global merge table: load <= 0.5
      uint64_t C = 64;
      while (C < (uint64_t)(2 * groups_hint)) C <<= 1;
      SX_TRY(scr.get(&g.keys, C + 1));
      SX_TRY(scr.get(&g.used, C + 1));
      for (int a = 0; a < s.nst; ++a) {
        SX_TRY(scr.get(&g.st[a], C + 1));
        g.hi[a] = nullptr;
        if (s.kind[a] == ST_SUM) SX_TRY(scr.get(&g.hi[a], C + 1));
      }
      g.mask = C - 1;
      k_gbs_init<<<persistent_grid(ctx, 4, (C + kBlock) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(s, g);
      // shared table: S slots (load <= 0.5 at the hint), R replicas in <= 96 KB (one table up to
      // ~200 KB)
      const uint32_t S = S_loc;
      const size_t tab = (size_t)(S + 1) * 8 * (1 + s.nst);
      int R = (int)std::max<size_t>(1, std::min<size_t>(32, (96u << 10) / tab));
      while (32 % R) --R;
      const size_t smem = tab * R;
      SX_TRY(with_sig(sig, [&](auto sg) -> sx_status {
        using SIG = decltype(sg);
        SX_CUDA(cudaFuncSetAttribute(k_gbs_local<SIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        SX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gbs_local<SIG>, kGsThreads, smem));
        const int64_t ctas = (int64_t)ctx->num_sms * std::max(1, per_sm);
        int64_t chunk = (n + ctas - 1) / ctas;
        chunk = std::min<int64_t>(chunk, 1 << 22);  // (<= 2^22 rows per CTA: the shared SUM words)
        const unsigned grid = (unsigned)((n + chunk - 1) / chunk);
        k_gbs_local<SIG><<<grid, kGsThreads, smem, SX_STREAM(ctx)>>>(s, n, chunk, S, R, g);
        SX_CHECK_LAUNCH();
        return SX_OK;
      }));
      k_gbs_emit<<<persistent_grid(ctx, 4, (C + kBlock) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(s, g);
      SX_CHECK_LAUNCH();
    }
    int64_t ng = 0;
    SX_TRY(read_i64(ctx, cursor, &ng));
    int fl = 0;
    SX_CUDA(cudaMemcpy(&fl, s.flags, sizeof(int), cudaMemcpyDeviceToHost));
    if (fl) return SX_EUNSUPPORTED;  // a shared table filled up / a wide value in K18p: generic path
    if (ng > cap) {
      if (!part) return SX_EUNSUPPORTED;  // (the global table was sized from the hint: generic path)
      cap = ng;
      continue;
    }
    out_keys[0] = sx_col{kt, kc.scale, ng, okey, nullptr, nullptr};
    scr.release(okey);
    for (int j = 0; j < naggs; ++j) {
      out_aggs[j] = sx_col{agg_out_type(aggs[j].op), 0, ng, oagg[j], nullptr, nullptr};
      scr.release(oagg[j]);
    }
    *out_ngroups = ng;
    return SX_OK;
  }
  return SX_EUNSUPPORTED;
}

}  // namespace sx
