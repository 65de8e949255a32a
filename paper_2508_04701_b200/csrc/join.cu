// join.cu — H4/H6: open-addressing hash join build (K5) and probe (K6).
//
// PAPER.md P:96 / P:254 (joins via libcudf, here our own kernels)
// (joins dominate join-heavy queries), P:268 ("hash tables" live in the
// processing region).  Table: power-of-two slots, load <= 0.5, linear probing,
// hash = murmur3 fmix64 (reading R14), duplicates kept.
//   key_bytes 4: slot u64 = (row << 32) | key32, claimed by one 64-bit CAS.
//   key_bytes 8: slot {u64 key; u32 row; u32 pad}, claimed by a 32-bit CAS on
//                row, key stored after (probes run in a later kernel).
// EMPTY: row word 0xFFFFFFFF (never a valid int32 row id).
#include <algorithm>

#include "compact.cuh"
#include "filter.cuh"
#include "join.cuh"
#include "radix.cuh"

using namespace sx;

namespace sx {

__device__ __forceinline__ uint64_t key_of(const DCol* cols, int nkeys, int kc0, int kc1, int64_t r) {
  if (nkeys == 1) return (uint64_t)ldv(cols[kc0], r);
  return ((uint64_t)(uint32_t)ldv(cols[kc0], r) << 32) | (uint32_t)ldv(cols[kc1], r);
}

struct BuildArgs {
  DCol cols[SX_MAX_COLS];
  DPred preds[SX_MAX_PREDS];
  int np, nkeys, kc0, kc1, key_bytes;
  const int32_t* sel;
  int64_t n;
  void* slots;
  uint64_t mask;
  unsigned long long* inserted;
  long long* kmin;  // [0] min, [1] max of inserted single-column keys (bitmap filter range)
};

__global__ void __launch_bounds__(kBlock) k_build(const __grid_constant__ BuildArgs a) {
  int64_t cnt = 0;
  long long mn = LLONG_MAX, mx = LLONG_MIN;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < a.n; idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = a.sel ? (int64_t)__ldg(a.sel + idx) : idx;
    if (!eval_conj(a.cols, a.preds, a.np, r)) continue;
    uint64_t key = key_of(a.cols, a.nkeys, a.kc0, a.kc1, r);
    mn = min(mn, (long long)key);
    mx = max(mx, (long long)key);
    uint64_t h = table_hash(key, a.key_bytes) & a.mask;
    if (!a.slots) {  // membership-only build: count and key range only
    } else if (a.key_bytes == 4) {
      unsigned long long* s = (unsigned long long*)a.slots;
      unsigned long long v = ((unsigned long long)(uint32_t)r << 32) | (uint32_t)key;
      while (atomicCAS(s + h, ~0ull, v) != ~0ull) h = (h + 1) & a.mask;
    } else {
      HtSlot8* s = (HtSlot8*)a.slots;
      while (atomicCAS(&s[h].row, 0xffffffffu, (unsigned)r) != 0xffffffffu) h = (h + 1) & a.mask;
      s[h].key = key;
    }
    ++cnt;
  }
  // warp-aggregated count of inserted rows and key range
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(kFull, cnt, o);
    mn = min(mn, __shfl_xor_sync(kFull, mn, o));
    mx = max(mx, __shfl_xor_sync(kFull, mx, o));
  }
  if ((threadIdx.x & 31) == 0 && cnt) {
    atomicAdd(a.inserted, (unsigned long long)cnt);
    atomicMin(a.kmin, mn);
    atomicMax(a.kmin + 1, mx);
  }
}

// Membership builds of a plain key column (no predicate, no selection): count and key range
// only, with 16-byte streaming loads (k_build's per-row interpreted path is 3x slower here).
template <typename KT>
__global__ void __launch_bounds__(kBlock) k_minmax(const KT* __restrict__ p, int64_t n, unsigned long long* inserted,
                                                   long long* kmin) {
  constexpr int V = 16 / sizeof(KT);
  long long mn = LLONG_MAX, mx = LLONG_MIN;
  const int64_t head = (int64_t)(((16 - ((uintptr_t)p & 15)) & 15) / sizeof(KT)) < n
                           ? (int64_t)(((16 - ((uintptr_t)p & 15)) & 15) / sizeof(KT)) : n;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  if (((uintptr_t)p % sizeof(KT)) == 0) {
    for (int64_t i = tid; i < head; i += nt) {
      const long long v = (long long)__ldg(p + i);
      mn = min(mn, v);
      mx = max(mx, v);
    }
    const int64_t nv = (n - head) / V;
    const KT* q = p + head;
    for (int64_t j = tid; j < nv; j += nt) {
      KT x[V];
      *(int4*)x = __ldcs((const int4*)q + j);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        mn = min(mn, (long long)x[k]);
        mx = max(mx, (long long)x[k]);
      }
    }
    for (int64_t i = head + nv * V + tid; i < n; i += nt) {
      const long long v = (long long)__ldg(p + i);
      mn = min(mn, v);
      mx = max(mx, v);
    }
  } else {
    for (int64_t i = tid; i < n; i += nt) {
      const long long v = (long long)p[i];
      mn = min(mn, v);
      mx = max(mx, v);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(kFull, mn, o));
    mx = max(mx, __shfl_xor_sync(kFull, mx, o));
  }
  if ((threadIdx.x & 31) == 0 && mn <= mx) {
    atomicMin(kmin, mn);
    atomicMax(kmin + 1, mx);
  }
  if (tid == 0) atomicAdd(inserted, (unsigned long long)n);
}

// Exact key-range bitmap of the build keys (predicate transfer): bit (key - min).
// Probes test it before touching the table, so misses cost one (L2-resident) word load.
__global__ void __launch_bounds__(kBlock) k_bitmap_set(const __grid_constant__ BuildArgs a, uint32_t* bm,
                                                       long long kmin, int32_t* direct) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < a.n; idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = a.sel ? (int64_t)__ldg(a.sel + idx) : idx;
    if (!eval_conj(a.cols, a.preds, a.np, r)) continue;
    uint64_t off = (uint64_t)((long long)key_of(a.cols, a.nkeys, a.kc0, a.kc1, r) - kmin);
    atomicOr(bm + (off >> 5), 1u << (off & 31));
    if (direct) direct[off] = (int32_t)r;  // unique keys: one writer per entry
  }
}

// Probe functor for the ordered compaction skeleton (semi / anti / inner on a unique build).
struct ProbeFn {
  DCol cols[SX_MAX_COLS];
  DPred preds[SX_MAX_PREDS];
  int np, nkeys, kc0, kc1, key_bytes, anti;
  const void* slots;
  uint64_t mask;
  template <int ITEMS>
  __device__ __forceinline__ void eval(const int32_t (&row)[ITEMS], const bool (&valid)[ITEMS], bool (&alive)[ITEMS],
                                       int32_t (&aux)[ITEMS]) const {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) alive[i] = valid[i];
    for (int p = 0; p < np; ++p) apply_pred<ITEMS>(cols[preds[p].col], preds[p], row, alive);
    uint64_t key[ITEMS], h[ITEMS];
    bool pend[ITEMS], found[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) key[i] = alive[i] ? key_of(cols, nkeys, kc0, kc1, row[i]) : 0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      h[i] = table_hash(key[i], key_bytes) & mask;
      pend[i] = alive[i];
      found[i] = false;
    }
    bool any = true;
    while (any) {
      any = false;
      if (key_bytes == 4) {
        unsigned long long s[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) s[i] = pend[i] ? __ldg((const unsigned long long*)slots + h[i]) : ~0ull;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          if (!pend[i]) continue;
          if ((uint32_t)(s[i] >> 32) == 0xffffffffu) pend[i] = false;
          else if ((uint32_t)s[i] == (uint32_t)key[i]) { found[i] = true; aux[i] = (int32_t)(s[i] >> 32); pend[i] = false; }
          else { h[i] = (h[i] + 1) & mask; any = true; }
        }
      } else {
        longlong2 s[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) s[i] = pend[i] ? __ldg((const longlong2*)slots + h[i]) : make_longlong2(0, -1);
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          if (!pend[i]) continue;
          uint32_t rw = (uint32_t)(unsigned long long)s[i].y;
          if (rw == 0xffffffffu) pend[i] = false;
          else if ((uint64_t)s[i].x == key[i]) { found[i] = true; aux[i] = (int32_t)rw; pend[i] = false; }
          else { h[i] = (h[i] + 1) & mask; any = true; }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) alive[i] = alive[i] && (anti ? !found[i] : found[i]);
  }
};

// INNER join on a non-unique build, typed keys (count -> scan -> expand):
//   1. ordered compaction with ProbeFnT{count_all}: the probe rows with >= 1 match, aux = count;
//   2. exclusive scan of the counts -> each matched row's first output position;
//   3. k_expand walks each matched row's chain again and writes its (probe row, build row)
//      pairs at those positions; payload columns are then gathered densely.
// Output order: probe order; a probe row's matches in table-chain order.
template <typename KT, int NK, int KB>
__global__ void __launch_bounds__(kBlock) k_expand(const __grid_constant__ ProbeFnT<KT, NK, KB, true> f,
                                                   const int32_t* __restrict__ msel, const int64_t* __restrict__ offs,
                                                   int64_t m, int32_t* __restrict__ op, int32_t* __restrict__ ob) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = __ldg(msel + j);
    int64_t o = __ldg(offs + j);
    uint64_t key = (uint64_t)(int64_t)__ldg(f.k0 + r);
    if (NK == 2) key = (key << 32) | (uint32_t)__ldg(f.k1 + r);
    uint32_t h = (uint32_t)(KB == 4 ? hash32((uint32_t)key) : hash64(key)) & f.mask;
    if (KB == 4) {
      bool first = (h & 1u) != 0;
      h &= ~1u;
      for (;;) {
        ulonglong2 s = __ldg((const ulonglong2*)f.slots + (h >> 1));
        uint32_t r0 = (uint32_t)(s.x >> 32), r1 = (uint32_t)(s.y >> 32);
        if (!first) {
          if (r0 == 0xffffffffu) break;
          if ((uint32_t)s.x == (uint32_t)key) { op[o] = r; ob[o] = (int32_t)r0; ++o; }
        }
        if (r1 == 0xffffffffu) break;
        if ((uint32_t)s.y == (uint32_t)key) { op[o] = r; ob[o] = (int32_t)r1; ++o; }
        first = false;
        h = (h + 2) & f.mask;
      }
    } else {
      for (;;) {
        longlong2 s = __ldg((const longlong2*)f.slots + h);
        uint32_t rw = (uint32_t)(unsigned long long)s.y;
        if (rw == 0xffffffffu) break;
        if ((uint64_t)s.x == key) { op[o] = r; ob[o] = (int32_t)rw; ++o; }
        h = (h + 1) & f.mask;
      }
    }
  }
}

// INNER join on a non-unique build, generic keys: every match emitted; output slots by
// warp-aggregated atomics (order not deterministic).
struct InnerArgs {
  DCol cols[SX_MAX_COLS];
  DPred preds[SX_MAX_PREDS];
  int np, nkeys, kc0, kc1, key_bytes;
  const int32_t* sel;
  int64_t n;
  const void* slots;
  uint64_t mask;
  int32_t* out_probe;
  int32_t* out_build;
  int64_t cap;
  unsigned long long* counter;
  const uint32_t* bm;
  long long bm_min;
  unsigned long long bm_bits;
};

__global__ void __launch_bounds__(kBlock) k_probe_inner(const __grid_constant__ InnerArgs a,
                                                        const __grid_constant__ GatherSpec gs) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // iterate so that whole warps stay converged: loop bound uniform per warp
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < a.n; base += stride) {
    int64_t idx = base + lane;
    bool alive = idx < a.n;
    int64_t r = 0;
    if (alive) {
      r = a.sel ? (int64_t)__ldg(a.sel + idx) : idx;
      alive = eval_conj(a.cols, a.preds, a.np, r);
    }
    uint64_t key = alive ? key_of(a.cols, a.nkeys, a.kc0, a.kc1, r) : 0;
    uint64_t h = table_hash(key, a.key_bytes) & a.mask;
    bool pend = alive;
    if (a.bm && pend) {
      unsigned long long off = (unsigned long long)((long long)key - a.bm_min);
      pend = off < a.bm_bits && ((__ldg(a.bm + (off >> 5)) >> (off & 31)) & 1u);
    }
    while (__any_sync(kFull, pend)) {
      bool hit = false;
      int32_t brow = -1;
      if (pend) {
        if (a.key_bytes == 4) {
          unsigned long long s = __ldg((const unsigned long long*)a.slots + h);
          if ((uint32_t)(s >> 32) == 0xffffffffu) pend = false;
          else if ((uint32_t)s == (uint32_t)key) { hit = true; brow = (int32_t)(s >> 32); }
        } else {
          longlong2 s = __ldg((const longlong2*)a.slots + h);
          uint32_t rw = (uint32_t)(unsigned long long)s.y;
          if (rw == 0xffffffffu) pend = false;
          else if ((uint64_t)s.x == key) { hit = true; brow = (int32_t)rw; }
        }
        h = (h + 1) & a.mask;
      }
      unsigned b = __ballot_sync(kFull, hit);
      if (b) {
        unsigned long long base_pos = 0;
        if (lane == __ffs(b) - 1) base_pos = atomicAdd(a.counter, (unsigned long long)__popc(b));
        base_pos = __shfl_sync(kFull, base_pos, __ffs(b) - 1);
        if (hit) {
          int64_t pos = (int64_t)base_pos + __popc(b & lt);
          if (pos < a.cap) {
            a.out_probe[pos] = (int32_t)r;
            a.out_build[pos] = brow;
            for (int g = 0; g < gs.n; ++g) gather_one(gs.g[g], pos, gs.g[g].by_aux ? (int64_t)brow : r);
          }
        }
      }
    }
  }
}

}  // namespace sx

namespace {

sx_status resolve_keys(sx_ctx* ctx, const sx_col* cols, int ncols, const int32_t* key_cols, int nkeys, int* kb,
                       int types[2]) {
  if (nkeys < 1 || nkeys > 2 || !key_cols) return set_err(ctx, SX_EINVAL, "join needs 1 or 2 key columns");
  for (int k = 0; k < nkeys; ++k) {
    if (key_cols[k] < 0 || key_cols[k] >= ncols) return set_err(ctx, SX_EINVAL, "key column out of range");
    int t = cols[key_cols[k]].type;
    if (t != SX_I32 && t != SX_DATE32 && t != SX_I64 && t != SX_U8)
      return set_err(ctx, SX_ETYPE, "join key type %d unsupported", t);
    if (nkeys == 2 && key_bits(t) > 32) return set_err(ctx, SX_ETYPE, "two-column keys must each be <= 32 bits");
    types[k] = t;
  }
  *kb = (nkeys == 1 && key_bits(types[0]) <= 32) ? 4 : 8;
  return SX_OK;
}

}  // namespace

SX_EXPORT sx_status sx_hash_build(sx_ctx* ctx, const sx_col* cols, int ncols, const int32_t* key_cols, int nkeys,
                                  const sx_sel* in_sel, const sx_pred* where, int nwhere, int unique_hint,
                                  sx_ht** out) {
  if (!ctx || !out) return SX_EINVAL;
  *out = nullptr;
  ProfScope ps(ctx, "hash_build");
  BuildArgs a{};
  SX_TRY(to_dcols(ctx, cols, ncols, a.cols));
  SX_TRY(check_preds(ctx, cols, ncols, where, nwhere, a.preds));
  int types[2] = {SX_I32, SX_I32};
  SX_TRY(resolve_keys(ctx, cols, ncols, key_cols, nkeys, &a.key_bytes, types));
  a.np = nwhere;
  a.nkeys = nkeys;
  a.kc0 = key_cols[0];
  a.kc1 = nkeys > 1 ? key_cols[1] : 0;
  int64_t n = in_sel ? in_sel->len : cols[key_cols[0]].len;
  if (n > INT32_MAX) return set_err(ctx, SX_EINDEX, "build side exceeds INT32_MAX rows");
  uint64_t cap = 64;
  while (cap < (uint64_t)(2 * n)) cap <<= 1;
  size_t slot_bytes = a.key_bytes == 4 ? 8 : 16;
  if (cap * slot_bytes * 2 <= (32ull << 20)) cap <<= 1;  // small (L2-resident) tables: load <= 0.25
  // unique_hint bit 1 (SX_BUILD_MEMBERSHIP): only semi/anti probes will follow; when the exact
  // key-range bitmap can be built (one key column, range <= 2^30) the table itself is omitted
  const bool membership = (unique_hint & 2) != 0 && nkeys == 1;
  // a unique single-column build whose table would not be L2-resident may become a direct-address
  // array (decided after the key range is known): bitmap + row per key, no table and no CAS
  const bool direct_off = getenv("SX_DIRECT") && getenv("SX_DIRECT")[0] == '0';
  const bool direct_cand = !direct_off && !membership && (unique_hint & 1) && nkeys == 1 &&
                           (types[0] == SX_I32 || types[0] == SX_DATE32 || types[0] == SX_I64) &&
                           cap * slot_bytes >= (8u << 20);
  sx_ht* ht = new sx_ht();
  ht->key_bytes = a.key_bytes;
  ht->key_types[0] = types[0];
  ht->key_types[1] = types[1];
  ht->nkeys = nkeys;
  ht->unique = (unique_hint & 1) != 0;
  ht->cap = cap;
  sx_status s = SX_OK;
  if (!membership && !direct_cand) {
    s = alloc(ctx, (char**)&ht->slots, cap * slot_bytes);
    if (s != SX_OK) {
      delete ht;
      return s;
    }
    cudaMemsetAsync(ht->slots, 0xff, cap * slot_bytes, ctx->stream);
  }
  // counters: [0] inserted rows, [1] min key, [2] max key
  unsigned long long* ins = (unsigned long long*)ctx->d_counters;
  int64_t* init = ctx->h_pinned + 8;
  init[0] = 0;
  init[1] = LLONG_MAX;
  init[2] = LLONG_MIN;
  cudaMemcpyAsync(ins, init, 3 * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream);
  a.sel = in_sel ? in_sel->idx : nullptr;
  a.n = n;
  a.slots = ht->slots;
  a.mask = cap - 1;
  a.inserted = ins;
  a.kmin = (long long*)(ins + 1);
  const bool plain = !a.slots && a.np == 0 && !a.sel && nkeys == 1 && !cols[key_cols[0]].validity;
  if (n > 0 && plain && (types[0] == SX_I32 || types[0] == SX_DATE32))
    k_minmax<int32_t><<<persistent_grid(ctx, 8, (n / 4 + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
        (const int32_t*)cols[key_cols[0]].data, n, ins, a.kmin);
  else if (n > 0 && plain && types[0] == SX_I64)
    k_minmax<long long><<<persistent_grid(ctx, 8, (n / 2 + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
        (const long long*)cols[key_cols[0]].data, n, ins, a.kmin);
  else if (n > 0)
    k_build<<<persistent_grid(ctx, 8, (n + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(a);
  cudaError_t e = cudaGetLastError();
  int64_t stats[3] = {0, 0, 0};
  if (e == cudaSuccess) s = read_i64(ctx, ins, stats, 3);
  if (e != cudaSuccess || s != SX_OK) {
    dfree(ctx, ht->slots);
    delete ht;
    return e != cudaSuccess ? set_err(ctx, SX_ECUDA, "build: %s", cudaGetErrorString(e)) : s;
  }
  ht->rows = stats[0];
  const bool bm_ok = nkeys == 1 && stats[0] > 0 && stats[2] >= stats[1] &&
                     (unsigned long long)(stats[2] - stats[1]) + 1 <= (1ull << 30);
  const unsigned long long krange = bm_ok ? (unsigned long long)(stats[2] - stats[1]) + 1 : 0;
  const bool use_direct = direct_cand && bm_ok && krange <= 64ull * (unsigned long long)stats[0] &&
                          krange * 4 <= (4ull << 30);
  if (use_direct) {
    s = alloc(ctx, &ht->direct, (size_t)krange);
    if (s != SX_OK) {
      ctx->err.clear();
      ht->direct = nullptr;
    }
  }
  if ((membership || direct_cand) && !ht->direct && !(membership && bm_ok) && stats[0] > 0) {
    // no bitmap / direct array possible: build the table after all
    s = alloc(ctx, (char**)&ht->slots, cap * slot_bytes);
    if (s != SX_OK) {
      delete ht;
      return s;
    }
    cudaMemsetAsync(ht->slots, 0xff, cap * slot_bytes, ctx->stream);
    a.slots = ht->slots;
    cudaMemcpyAsync(ins, init, 3 * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream);
    k_build<<<persistent_grid(ctx, 8, (n + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(a);
    SX_CHECK_LAUNCH();
  }
  if ((membership || ht->direct) && !ht->slots) ht->cap = 0;
  // exact bitmap filter over the key range when it is small enough to stay cache-resident-ish
  if (nkeys == 1 && stats[0] > 0) {
    unsigned long long range = (unsigned long long)(stats[2] - stats[1]) + 1;
    if (stats[2] >= stats[1] && range <= (1ull << 30)) {
      size_t words = (size_t)((range + 31) / 32);
      if (alloc(ctx, &ht->bm, words) == SX_OK) {
        cudaMemsetAsync(ht->bm, 0, words * sizeof(uint32_t), ctx->stream);
        ht->bm_min = stats[1];
        ht->bm_bits = range;
        k_bitmap_set<<<persistent_grid(ctx, 8, (n + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(a, ht->bm, stats[1],
                                                                                                     ht->direct);
        e = cudaGetLastError();
        if (e != cudaSuccess) {
          dfree(ctx, ht->slots);
          dfree(ctx, ht->bm);
          delete ht;
          return set_err(ctx, SX_ECUDA, "bitmap: %s", cudaGetErrorString(e));
        }
      } else {
        ctx->err.clear();
        ht->bm = nullptr;
        if (ht->direct) {  // the direct array needs the bitmap
          dfree(ctx, ht->direct);
          dfree(ctx, ht->slots);
          delete ht;
          return set_err(ctx, SX_ENOMEM, "device pool exhausted (key bitmap)");
        }
      }
    }
  }
  *out = ht;
  if (ps.on()) {  // key (+ predicate) columns of the scanned rows, selection, one slot per inserted row
    RefCols rc;
    for (int k = 0; k < nkeys; ++k) rc.add(key_cols[k]);
    for (int p = 0; p < nwhere; ++p) rc.add(where[p].col);
    ps.set_bytes((rc.row_bytes(cols, ncols) + (in_sel ? 4.0 : 0.0)) * n + (double)slot_bytes * ht->rows);
  }
  return SX_OK;
}

SX_EXPORT int64_t sx_ht_rows(const sx_ht* ht) { return ht ? ht->rows : 0; }

SX_EXPORT void sx_ht_destroy(sx_ctx* ctx, sx_ht* ht) {
  if (!ht) return;
  if (ctx) {
    dfree(ctx, ht->slots);
    dfree(ctx, ht->bm);
    dfree(ctx, ht->direct);
  }
  delete ht;
}

SX_EXPORT sx_status sx_hash_probe(sx_ctx* ctx, const sx_ht* ht, const sx_col* probe_cols, int nprobe_cols,
                                  const int32_t* key_cols, int nkeys, const sx_sel* in_sel, const sx_pred* where,
                                  int nwhere, int join_type, const sx_col* build_cols, int nbuild_cols,
                                  const int32_t* bp, int nbp, const int32_t* pp, int npp, sx_sel* out_probe,
                                  sx_sel* out_build, sx_col* out_payload) {
  if (!ctx || !ht || !out_probe) return SX_EINVAL;
  *out_probe = sx_sel{0, nullptr};
  if (out_build) *out_build = sx_sel{0, nullptr};
  for (int i = 0; out_payload && i < nbp + npp && i < kMaxGather; ++i) out_payload[i] = sx_col{};
  ProfScope ps(ctx, join_type == SX_INNER ? "probe_inner" : (join_type == SX_SEMI ? "probe_semi" : "probe_anti"));
  if (join_type < SX_INNER || join_type > SX_ANTI) return set_err(ctx, SX_EINVAL, "join type %d", join_type);
  if (join_type == SX_INNER && !out_build) return set_err(ctx, SX_EINVAL, "INNER join needs out_build");
  if (!ht->slots && !ht->direct && (join_type == SX_INNER || !ht->bm))
    return set_err(ctx, SX_EINVAL, "membership-only table: SEMI/ANTI probes only");
  if (join_type != SX_INNER && nbp > 0) return set_err(ctx, SX_EINVAL, "build payload only for INNER joins");
  if (nbp + npp > kMaxGather || nbp < 0 || npp < 0) return set_err(ctx, SX_EINVAL, "too many payload columns");
  if ((nbp + npp) > 0 && !out_payload) return set_err(ctx, SX_EINVAL, "out_payload is NULL");
  DCol pcols[SX_MAX_COLS], bcols[SX_MAX_COLS];
  SX_TRY(to_dcols(ctx, probe_cols, nprobe_cols, pcols));
  if (nbp > 0) SX_TRY(to_dcols(ctx, build_cols, nbuild_cols, bcols));
  DPred preds[SX_MAX_PREDS];
  SX_TRY(check_preds(ctx, probe_cols, nprobe_cols, where, nwhere, preds));
  int kb = 4, types[2];
  SX_TRY(resolve_keys(ctx, probe_cols, nprobe_cols, key_cols, nkeys, &kb, types));
  if (nkeys != ht->nkeys || kb != ht->key_bytes)
    return set_err(ctx, SX_ETYPE, "probe key shape (%d keys, %d bytes) differs from the build (%d, %d)", nkeys, kb,
                   ht->nkeys, ht->key_bytes);
  int64_t n = in_sel ? in_sel->len : probe_cols[key_cols[0]].len;
  if (n > INT32_MAX) return set_err(ctx, SX_EINDEX, "probe side exceeds INT32_MAX rows");
  Scratch scr(ctx);
  GatherSpec gs;
  gs.n = nbp + npp;
  for (int g = 0; g < nbp; ++g) {
    if (bp[g] < 0 || bp[g] >= nbuild_cols) return set_err(ctx, SX_EINVAL, "build payload column out of range");
    gs.g[g].src = bcols[bp[g]];
    gs.g[g].by_aux = 1;
    gs.g[g].width = type_width(build_cols[bp[g]].type);
    if (!gs.g[g].width) return set_err(ctx, SX_ETYPE, "payload must be fixed-width");
  }
  for (int g = 0; g < npp; ++g) {
    if (pp[g] < 0 || pp[g] >= nprobe_cols) return set_err(ctx, SX_EINVAL, "probe payload column out of range");
    gs.g[nbp + g].src = pcols[pp[g]];
    gs.g[nbp + g].by_aux = 0;
    gs.g[nbp + g].width = type_width(probe_cols[pp[g]].type);
    if (!gs.g[nbp + g].width) return set_err(ctx, SX_ETYPE, "payload must be fixed-width");
  }
  const int32_t* isel = in_sel ? in_sel->idx : nullptr;
  int64_t count = 0;
  int32_t *op = nullptr, *ob = nullptr;
  auto is32 = [&](int c) { int t = probe_cols[key_cols[c]].type; return t == SX_I32 || t == SX_DATE32; };
  auto fill_t = [&](auto& ft) {
    for (int i = 0; i < nprobe_cols; ++i) ft.cols[i] = pcols[i];
    for (int i = 0; i < nwhere; ++i) ft.preds[i] = preds[i];
    ft.np = nwhere;
    ft.k0 = (decltype(ft.k0))probe_cols[key_cols[0]].data;
    ft.k1 = nkeys > 1 ? (const int32_t*)probe_cols[key_cols[1]].data : nullptr;
    ft.slots = ht->slots;
    ft.mask = (uint32_t)(ht->cap - 1);
    ft.anti = join_type == SX_ANTI;
    ft.member_only = join_type != SX_INNER;
    ft.bm = ht->bm;
    ft.bm_min = ht->bm_min;
    ft.bm_bits = ht->bm_bits;
    ft.direct = ht->direct;
  };
  // non-unique INNER with typed keys: count -> scan -> expand (see k_expand)
  auto run_expand = [&](auto ft) -> sx_status {
    fill_t(ft);
    int32_t *msel = nullptr, *mcnt = nullptr;
    int64_t m = 0;
    GatherSpec none;
    none.n = 0;
    SX_TRY((run_compact<decltype(ft), 4>(ctx, ft, n, isel, &msel, &mcnt, none, &m)));
    scr.ptrs.push_back(msel);
    scr.ptrs.push_back(mcnt);
    int64_t* offs;
    SX_TRY(scr.get(&offs, (size_t)m + 1));
    SX_TRY(scan_counts(ctx, mcnt, m, offs, &count));
    if (count > INT32_MAX) return set_err(ctx, SX_EINDEX, "join output exceeds INT32_MAX rows");
    const size_t c = (size_t)(count > 0 ? count : 1);
    SX_TRY(scr.get(&op, c));
    SX_TRY(scr.get(&ob, c));
    for (int g = 0; g < gs.n; ++g) SX_TRY(scr.get((char**)&gs.g[g].dst, c * gs.g[g].width));
    if (m > 0) {
      k_expand<<<persistent_grid(ctx, 8, (m + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(ft, msel, offs, m, op,
                                                                                                ob);
      SX_CHECK_LAUNCH();
    }
    if (count > 0 && gs.n > 0) {
      k_gather_multi<<<persistent_grid(ctx, 8, (count + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(op, ob,
                                                                                                          count, gs);
      SX_CHECK_LAUNCH();
    }
    return SX_OK;
  };
  const bool typed = ht->cap <= (1ull << 32) &&
                     ((nkeys == 1 && kb == 4 && is32(0)) || (nkeys == 1 && kb == 8 && probe_cols[key_cols[0]].type == SX_I64) ||
                      (nkeys == 2 && is32(0) && is32(1)));
  if (join_type == SX_INNER && !ht->unique && typed) {
    if (nkeys == 2) SX_TRY((run_expand(ProbeFnT<int32_t, 2, 8, true>{})));
    else if (kb == 4) SX_TRY((run_expand(ProbeFnT<int32_t, 1, 4, true>{})));
    else SX_TRY((run_expand(ProbeFnT<long long, 1, 8, true>{})));
  } else if (join_type != SX_INNER || ht->unique) {
    // ordered compaction: each probe row emits at most one output
    ProbeFn f;
    for (int i = 0; i < nprobe_cols; ++i) f.cols[i] = pcols[i];
    for (int i = 0; i < nwhere; ++i) f.preds[i] = preds[i];
    f.np = nwhere;
    f.nkeys = nkeys;
    f.kc0 = key_cols[0];
    f.kc1 = nkeys > 1 ? key_cols[1] : 0;
    f.key_bytes = kb;
    f.anti = join_type == SX_ANTI;
    f.slots = ht->slots;
    f.mask = ht->cap - 1;
    for (int g = 0; g < gs.n; ++g) gs.g[g].dst = nullptr;  // allocated at the exact output count
    int32_t** pob = join_type == SX_INNER ? &ob : nullptr;
    // bitmap-only membership functor for one key column (semi/anti answer, or INNER phase 1)
    auto make_bm = [&](auto* kt) {
      using KT = std::remove_pointer_t<decltype(kt)>;
      BitmapFn<KT> b;
      for (int i = 0; i < nprobe_cols; ++i) b.cols[i] = pcols[i];
      for (int i = 0; i < nwhere; ++i) b.preds[i] = preds[i];
      b.np = nwhere;
      b.k0 = (const KT*)probe_cols[key_cols[0]].data;
      b.bm = ht->bm;
      b.bm_min = ht->bm_min;
      b.bm_bits = ht->bm_bits;
      b.anti = join_type == SX_ANTI;
      return b;
    };
    auto run_t = [&](auto ft) -> sx_status {
      fill_t(ft);
      if (ft.bm && nkeys == 1 && join_type != SX_INNER) {  // the exact bitmap is the answer
        if (probe_cols[key_cols[0]].type == SX_I64)
          return run_compact<BitmapFn<long long>, 8>(ctx, make_bm((long long*)nullptr), n, isel, &op, nullptr, gs,
                                                     &count);
        return run_compact<BitmapFn<int32_t>, 8>(ctx, make_bm((int32_t*)nullptr), n, isel, &op, nullptr, gs, &count);
      }
      if (join_type == SX_INNER && ft.bm && (ht->slots || ht->direct) && nkeys == 1) {
        // Two phases: the exact bitmap selects the matching probe rows (a streaming scan whose
        // only lookups are bitmap words), then only those rows probe the table for their build
        // row.  The scan's tiles never wait on a random HBM table access.
        int32_t* cand = nullptr;
        int64_t nc = 0;
        GatherSpec none;
        none.n = 0;
        auto bmf = make_bm((decltype(ft.k0))nullptr);
        bmf.anti = 0;
        SX_TRY((run_compact<decltype(bmf), 8>(ctx, bmf, n, isel, &cand, nullptr, none, &nc)));
        scr.ptrs.push_back(cand);
        auto fl = ft;
        fl.np = 0;  // predicates already applied
        fl.bm = nullptr;
        return run_compact<decltype(fl), 4>(ctx, fl, nc, cand, &op, pob, gs, &count);
      }
      if (join_type == SX_INNER && ft.bm && ht->slots) {
        // Two phases: the exact bitmap selects the matching probe rows (a streaming scan whose
        // only lookups are bitmap words), then only those rows probe the table for their build
        // row.  The scan's tiles never wait on a random HBM table access.
        auto fm = ft;
        fm.member_only = 1;
        fm.anti = 0;
        int32_t* cand = nullptr;
        int64_t nc = 0;
        GatherSpec none;
        none.n = 0;
        SX_TRY((run_compact<decltype(fm), 4>(ctx, fm, n, isel, &cand, nullptr, none, &nc)));
        scr.ptrs.push_back(cand);
        auto fl = ft;
        fl.np = 0;  // predicates already applied
        fl.bm = nullptr;
        return run_compact<decltype(fl), 4>(ctx, fl, nc, cand, &op, pob, gs, &count);
      }
      return run_compact<decltype(ft), 4>(ctx, ft, n, isel, &op, pob, gs, &count);
    };
    if (ht->cap <= (1ull << 32) && nkeys == 1 && kb == 4 && is32(0)) {
      SX_TRY(run_t(ProbeFnT<int32_t, 1, 4>{}));
    } else if (ht->cap <= (1ull << 32) && nkeys == 1 && kb == 8 && probe_cols[key_cols[0]].type == SX_I64) {
      SX_TRY(run_t(ProbeFnT<long long, 1, 8>{}));
    } else if (ht->cap <= (1ull << 32) && nkeys == 2 && is32(0) && is32(1)) {
      SX_TRY(run_t(ProbeFnT<int32_t, 2, 8>{}));
    } else {
      SX_TRY((run_compact<ProbeFn, 4>(ctx, f, n, isel, &op, pob, gs, &count)));
    }
  } else {
    InnerArgs a{};
    for (int i = 0; i < nprobe_cols; ++i) a.cols[i] = pcols[i];
    for (int i = 0; i < nwhere; ++i) a.preds[i] = preds[i];
    a.np = nwhere;
    a.nkeys = nkeys;
    a.kc0 = key_cols[0];
    a.kc1 = nkeys > 1 ? key_cols[1] : 0;
    a.key_bytes = kb;
    a.sel = isel;
    a.n = n;
    a.slots = ht->slots;
    a.mask = ht->cap - 1;
    a.counter = (unsigned long long*)ctx->d_counters;
    a.bm = ht->bm;
    a.bm_min = ht->bm_min;
    a.bm_bits = ht->bm_bits;
    // first guess: one output per build row (FK side built, PK side probed); exact retry if more
    int64_t cap = std::max<int64_t>(std::min<int64_t>(n, std::max<int64_t>(ht->rows, n / 16)), 1024);
    for (int attempt = 0; attempt < 2; ++attempt) {
      SX_TRY(scr.get(&op, (size_t)cap));
      SX_TRY(scr.get(&ob, (size_t)cap));
      for (int g = 0; g < gs.n; ++g) SX_TRY(scr.get((char**)&gs.g[g].dst, (size_t)cap * gs.g[g].width));
      a.out_probe = op;
      a.out_build = ob;
      a.cap = cap;
      SX_CUDA(cudaMemsetAsync(a.counter, 0, 8, ctx->stream));
      if (n > 0) k_probe_inner<<<persistent_grid(ctx, 8, (n + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(a, gs);
      SX_CHECK_LAUNCH();
      SX_TRY(read_i64(ctx, a.counter, &count));
      if (count <= cap) break;
      if (count > INT32_MAX) return set_err(ctx, SX_EINDEX, "join output exceeds INT32_MAX rows");
      // too small: release and retry at the exact size
      dfree(ctx, op); scr.release(op);
      dfree(ctx, ob); scr.release(ob);
      for (int g = 0; g < gs.n; ++g) { dfree(ctx, gs.g[g].dst); scr.release(gs.g[g].dst); }
      cap = count;
    }
  }
  out_probe->len = count;
  out_probe->idx = op;
  scr.release(op);
  if (join_type == SX_INNER) {
    out_build->len = count;
    out_build->idx = ob;
    scr.release(ob);
  }
  for (int g = 0; g < gs.n; ++g) {
    const sx_col& src = g < nbp ? build_cols[bp[g]] : probe_cols[pp[g - nbp]];
    out_payload[g] = src;
    out_payload[g].len = count;
    out_payload[g].data = gs.g[g].dst;
    out_payload[g].offsets = nullptr;
    scr.release(gs.g[g].dst);
  }
  if (ps.on()) {  // probe keys (+ predicate columns) + selection in; row ids out; payload read + written
    RefCols rc;
    for (int k = 0; k < nkeys; ++k) rc.add(key_cols[k]);
    for (int p = 0; p < nwhere; ++p) rc.add(where[p].col);
    double b = (rc.row_bytes(probe_cols, nprobe_cols) + (in_sel ? 4.0 : 0.0)) * n;
    b += (join_type == SX_INNER ? 8.0 : 4.0) * count;
    for (int g = 0; g < gs.n; ++g) b += 2.0 * gs.g[g].width * count;
    ps.set_bytes(b);
  }
  return SX_OK;
}

// ------------------------------------------------------------------ payload tables (internal)
namespace sx {
namespace {
struct PtArgs {
  DCol k0, k1, pay;
  int nkeys, kb, compact;
  const int32_t* sel;
  int64_t lo, n;  // rows [lo, n) (of sel, else of the columns)
  ulonglong2* slots;
  uint32_t mask;
  int pbits;
  int* bad;  // duplicate or reserved key
};

__global__ void __launch_bounds__(kBlock) k_pt_build(const __grid_constant__ PtArgs a) {
  for (int64_t i = a.lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = a.sel ? (int64_t)__ldg(a.sel + i) : i;
    uint64_t key = (uint64_t)ldv(a.k0, r);
    if (a.nkeys == 2) key = (key << 32) | (uint32_t)ldv(a.k1, r);
    const uint64_t base = pt_region_base(key, a.pbits, a.mask);
    const uint64_t x = a.kb == 4 ? (uint64_t)(uint32_t)key : key;
    if (x == ~0ull) {
      atomicExch(a.bad, 1);
      continue;
    }
    uint32_t h = (uint32_t)(a.kb == 4 ? hash32((uint32_t)key) : hash64(key)) & a.mask;
    if (a.compact) {  // 8-byte slots: (payload32 << 32) | key32 in one CAS
      const unsigned long long e = ((unsigned long long)(uint32_t)ldv(a.pay, r) << 32) | (uint32_t)key;
      if (e == ~0ull) {
        atomicExch(a.bad, 1);
        continue;
      }
      unsigned long long* sl = (unsigned long long*)a.slots + base;
      for (;;) {
        const unsigned long long old = atomicCAS(sl + h, ~0ull, e);
        if (old == ~0ull) break;
        if ((uint32_t)old == (uint32_t)key) {
          atomicExch(a.bad, 1);
          break;
        }
        h = (h + 1) & a.mask;
      }
      continue;
    }
    ulonglong2* sl = a.slots + base;
    for (;;) {
      const unsigned long long old = atomicCAS(&sl[h].x, ~0ull, (unsigned long long)x);
      if (old == ~0ull) {
        sl[h].y = (unsigned long long)ldv(a.pay, r);
        break;
      }
      if (old == x) {  // a repeated key: not a PK side
        atomicExch(a.bad, 1);
        break;
      }
      h = (h + 1) & a.mask;
    }
  }
}
}  // namespace

sx_status build_payload_table(sx_ctx* ctx, const sx_col* keys, int nkeys, const sx_col& pay, const sx_sel* sel,
                              PayloadTable* out, bool allow_compact) {
  *out = PayloadTable{};
  if (nkeys < 1 || nkeys > 2) return set_err(ctx, SX_EINVAL, "payload table: nkeys %d", nkeys);
  for (int k = 0; k < nkeys; ++k)
    if (!(keys[k].type == SX_I32 || keys[k].type == SX_DATE32 || (nkeys == 1 && keys[k].type == SX_I64)))
      return set_err(ctx, SX_ETYPE, "payload table: key type %d", keys[k].type);
  if (!is_int_type(pay.type)) return set_err(ctx, SX_ETYPE, "payload table: payload type %d", pay.type);
  const int64_t n = sel ? sel->len : keys[0].len;
  uint64_t cap = 64;
  while (cap < (uint64_t)(n + n / 2)) cap <<= 1;  // load <= 2/3: a smaller table stays more L2-resident
  if (cap > (1ull << 32)) return set_err(ctx, SX_EINDEX, "payload table too large");
  PtArgs a{};
  a.k0 = DCol{keys[0].data, keys[0].type, 0};
  a.k1 = DCol{keys[nkeys - 1].data, keys[nkeys - 1].type, 0};
  a.pay = DCol{pay.data, pay.type, 0};
  a.nkeys = nkeys;
  a.kb = (nkeys == 1 && keys[0].type != SX_I64) ? 4 : 8;
  a.compact = allow_compact && a.kb == 4 && (pay.type == SX_I32 || pay.type == SX_DATE32 || pay.type == SX_U8);
  a.sel = sel ? sel->idx : nullptr;
  a.n = n;
  a.mask = (uint32_t)(cap - 1);
  a.bad = ctx->d_flags + 2;
  const size_t sb = a.compact ? 8 : 16;
  Scratch scr(ctx);
  // much larger than the L2: radix-partition (key, payload) and build region by region in waves
  // that stay L2-resident (random CAS hits L2 instead of HBM)
  // SX_PT_PARTITION: 0 never, 2 always (tests), else when the table exceeds half the L2
  const char* pe = getenv("SX_PT_PARTITION");
  const int pmode = pe ? pe[0] - '0' : 1;
  std::vector<int64_t> off;
  // (measured at SF100: 268 MB partsupp' table 0.35 -> 0.55 ms partitioned, 512 MB orders' 2.1 -> 1.9 ms:
  // the partition pass pays off only well above the L2 size)
  if (pmode != 0 && n > 0 && (pmode == 2 || cap * sb > 4 * ctx->l2_bytes)) {
    int bits = 1;
    while (bits < 10 && ((cap * sb) >> bits) > (8u << 20)) ++bits;
    if (pmode == 2 && cap * sb <= (8u << 20)) bits = 3;  // forced: a few regions even for small tables
    const int P = 1 << bits;
    DCol carry[3];
    int width[3];
    void* outp[3];
    int nc = 0;
    for (int k = 0; k < nkeys; ++k) {
      carry[nc] = DCol{keys[k].data, keys[k].type, 0};
      width[nc] = type_width(keys[k].type);
      ++nc;
    }
    carry[nc] = a.pay;
    width[nc] = type_width(pay.type);
    ++nc;
    for (int c = 0; c < nc; ++c) SX_TRY(scr.get((char**)&outp[c], (size_t)n * width[c]));
    off.assign((size_t)P + 1, 0);
    SX_TRY(radix_partition_carry(ctx, a.k0, a.k1, nkeys, carry, width, nc, a.sel, n, bits, outp, off.data()));
    int64_t maxp = 1;
    for (int p = 0; p < P; ++p) maxp = std::max<int64_t>(maxp, off[p + 1] - off[p]);
    uint64_t capp = 64;
    while (capp < (uint64_t)(2 * maxp)) capp <<= 1;
    a.pbits = bits;
    a.mask = (uint32_t)(capp - 1);
    cap = capp * P;
    a.k0 = DCol{outp[0], keys[0].type, 0};
    a.k1 = DCol{outp[nkeys - 1], keys[nkeys - 1].type, 0};
    a.pay = DCol{outp[nc - 1], pay.type, 0};
    a.sel = nullptr;
  }
  SX_TRY(alloc(ctx, (char**)&a.slots, (size_t)cap * sb));
  SX_CUDA(cudaMemsetAsync(a.slots, 0xff, cap * sb, ctx->stream));
  SX_CUDA(cudaMemsetAsync(a.bad, 0, sizeof(int), ctx->stream));
  if (n > 0 && a.pbits == 0) {
    k_pt_build<<<persistent_grid(ctx, 8, (n + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(a);
  } else if (n > 0) {
    const int P = 1 << a.pbits;
    const size_t region = ((size_t)a.mask + 1) * sb;
    const int W = (int)std::max<size_t>(1, (ctx->l2_bytes / 3) / region);
    for (int p0 = 0; p0 < P; p0 += W) {
      const int p1 = std::min(P, p0 + W);
      a.lo = off[p0];
      a.n = off[p1];
      if (a.n > a.lo)
        k_pt_build<<<persistent_grid(ctx, 8, (a.n - a.lo + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(a);
    }
  }
  cudaError_t e = cudaGetLastError();
  int bad = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, a.bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess || bad) {
    dfree(ctx, a.slots);
    return e != cudaSuccess ? set_err(ctx, SX_ECUDA, "payload table: %s", cudaGetErrorString(e))
                            : set_err(ctx, SX_EINVAL, "payload table: repeated or reserved key");
  }
  out->slots = a.slots;
  out->mask = a.mask;
  out->pbits = a.pbits;
  out->kb = a.kb;
  out->compact = a.compact;
  out->rows = n;
  return SX_OK;
}

void free_payload_table(sx_ctx* ctx, PayloadTable* t) {
  if (t && t->slots) dfree(ctx, t->slots);
  if (t) *t = PayloadTable{};
}
}  // namespace sx
