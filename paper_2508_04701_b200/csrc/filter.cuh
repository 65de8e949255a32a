// filter.cuh — row functors for the compaction skeleton: conjunctive
// fixed-width predicates (K1, lazy column loads) and string CONTAINS (K4).
#pragma once
#include "common.cuh"

namespace sx {

// Apply one predicate to a thread's ITEMS rows.  Loads are predicated on the row still
// being alive (short-circuit at row granularity: sectors of dead rows are never fetched)
// and issued back to back for memory-level parallelism; type and op switches are uniform.
template <int ITEMS>
__device__ __forceinline__ void apply_pred(const DCol& c, const DPred& q, const int32_t (&row)[ITEMS],
                                           bool (&alive)[ITEMS]) {
  int64_t x[ITEMS];
  switch (c.type) {
    case SX_U8: {
      const uint8_t* p = (const uint8_t*)c.p;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) x[i] = alive[i] ? (int64_t)__ldg(p + row[i]) : 0;
      break;
    }
    case SX_I32:
    case SX_DATE32: {
      const int32_t* p = (const int32_t*)c.p;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) x[i] = alive[i] ? (int64_t)__ldg(p + row[i]) : 0;
      break;
    }
    default: {
      const long long* p = (const long long*)c.p;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) x[i] = alive[i] ? (int64_t)__ldg(p + row[i]) : 0;
      break;
    }
  }
  const int64_t lo = q.lo, hi = q.hi;
  switch (q.op) {
#define SX_APPLY(OPC, EXPR)                                       \
  case OPC:                                                       \
    _Pragma("unroll") for (int i = 0; i < ITEMS; ++i) alive[i] = alive[i] && (EXPR); \
    break;
    SX_APPLY(SX_LT, x[i] < lo)
    SX_APPLY(SX_LE, x[i] <= lo)
    SX_APPLY(SX_GT, x[i] > lo)
    SX_APPLY(SX_GE, x[i] >= lo)
    SX_APPLY(SX_EQ, x[i] == lo)
    SX_APPLY(SX_NE, x[i] != lo)
    default:
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) alive[i] = alive[i] && lo <= x[i] && x[i] <= hi;
#undef SX_APPLY
  }
}

// ---- dense (selection-free) evaluation: a thread owns ITEMS consecutive rows r0.. (r0 % ITEMS == 0)
// and loads each column with 128-bit vector loads (column buffers are 16-byte aligned) marked
// streaming (ld.global.cs: evict-first, so scanned columns do not push the probed hash tables and
// bitmaps out of L2); `full`
// means all ITEMS rows exist (else the tail is loaded row by row).  Results are bit masks.
template <int ITEMS>
__device__ __forceinline__ void dense_load(const DCol& c, int64_t r0, int64_t n, bool full, int64_t (&x)[ITEMS]) {
  static_assert(ITEMS % 4 == 0, "dense rows come in groups of 4");
  if (full) {
    switch (c.type) {
      case SX_U8: {
#pragma unroll
        for (int j = 0; j < ITEMS / 4; ++j) {
          const uint32_t v = __ldcs((const unsigned int*)((const uint8_t*)c.p + r0) + j);
#pragma unroll
          for (int b = 0; b < 4; ++b) x[4 * j + b] = (int64_t)((v >> (8 * b)) & 0xffu);
        }
        return;
      }
      case SX_I32:
      case SX_DATE32: {
#pragma unroll
        for (int j = 0; j < ITEMS / 4; ++j) {
          const int4 v = __ldcs((const int4*)((const int32_t*)c.p + r0) + j);
          x[4 * j] = v.x; x[4 * j + 1] = v.y; x[4 * j + 2] = v.z; x[4 * j + 3] = v.w;
        }
        return;
      }
      default: {
#pragma unroll
        for (int j = 0; j < ITEMS / 2; ++j) {
          const longlong2 v = __ldcs((const longlong2*)((const long long*)c.p + r0) + j);
          x[2 * j] = v.x; x[2 * j + 1] = v.y;
        }
        return;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) x[i] = r0 + i < n ? ldv(c, r0 + i) : 0;
}

template <int ITEMS>
__device__ __forceinline__ uint32_t dense_valid(int64_t r0, int64_t n) {
  const int64_t m = n - r0;
  return m >= ITEMS ? (ITEMS == 32 ? 0xffffffffu : ((1u << ITEMS) - 1u)) : (m <= 0 ? 0u : ((1u << m) - 1u));
}

// 32-bit column values of ITEMS rows (kept 32-bit: half the registers, 32-bit compares)
template <int ITEMS>
__device__ __forceinline__ void dense_load32(const int32_t* p, int64_t r0, int64_t n, bool full, int32_t (&x)[ITEMS]) {
  if (full) {
#pragma unroll
    for (int j = 0; j < ITEMS / 4; ++j) {
      const int4 v = __ldcs((const int4*)(p + r0) + j);
      x[4 * j] = v.x; x[4 * j + 1] = v.y; x[4 * j + 2] = v.z; x[4 * j + 3] = v.w;
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) x[i] = r0 + i < n ? __ldg(p + r0 + i) : 0;
}

// A predicate on a 32-bit column with 32-bit compares: constants outside the int32 range make a
// comparison uniformly true or false, else they are exact as int32.
template <int ITEMS>
__device__ __forceinline__ uint32_t dense_pred32(const int32_t (&x)[ITEMS], const DPred& q) {
  const long long lo = q.lo, hi = q.hi;
  const bool lo_big = lo > INT32_MAX, lo_small = lo < INT32_MIN;
  const bool hi_big = hi > INT32_MAX, hi_small = hi < INT32_MIN;
  const int32_t l = (int32_t)(lo_big ? INT32_MAX : lo_small ? INT32_MIN : lo);
  const int32_t h = (int32_t)(hi_big ? INT32_MAX : hi_small ? INT32_MIN : hi);
  constexpr uint32_t all = ITEMS == 32 ? 0xffffffffu : ((1u << ITEMS) - 1u);
  uint32_t m = 0;
  switch (q.op) {  // uniform
    case SX_LT:
      if (lo_big) return all;
      if (lo_small) return 0;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) m |= (x[i] < l ? 1u : 0u) << i;
      return m;
    case SX_LE:
      if (lo_big) return all;
      if (lo_small) return 0;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) m |= (x[i] <= l ? 1u : 0u) << i;
      return m;
    case SX_GT:
      if (lo_small) return all;
      if (lo_big) return 0;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) m |= (x[i] > l ? 1u : 0u) << i;
      return m;
    case SX_GE:
      if (lo_small) return all;
      if (lo_big) return 0;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) m |= (x[i] >= l ? 1u : 0u) << i;
      return m;
    case SX_EQ:
      if (lo_big || lo_small) return 0;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) m |= (x[i] == l ? 1u : 0u) << i;
      return m;
    case SX_NE:
      if (lo_big || lo_small) return all;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) m |= (x[i] != l ? 1u : 0u) << i;
      return m;
    default:  // BETWEEN lo..hi
      if (lo_big || hi_small || lo > hi) return 0;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) m |= (x[i] >= l && x[i] <= h ? 1u : 0u) << i;
      return m;
  }
}

template <int ITEMS>
__device__ __forceinline__ void dense_pred(const DCol& c, const DPred& q, int64_t r0, int64_t n, bool full,
                                           uint32_t& mask) {
  if (c.type == SX_I32 || c.type == SX_DATE32) {
    int32_t x32[ITEMS];
    dense_load32<ITEMS>((const int32_t*)c.p, r0, n, full, x32);
    mask &= dense_pred32<ITEMS>(x32, q);
    return;
  }
  int64_t x[ITEMS];
  dense_load<ITEMS>(c, r0, n, full, x);
  uint32_t m = 0;
  const int64_t lo = q.lo, hi = q.hi;
  switch (q.op) {  // uniform
#define SX_DENSE(OPC, EXPR)                                                     \
  case OPC:                                                                     \
    _Pragma("unroll") for (int i = 0; i < ITEMS; ++i) m |= ((EXPR) ? 1u : 0u) << i; \
    break;
    SX_DENSE(SX_LT, x[i] < lo)
    SX_DENSE(SX_LE, x[i] <= lo)
    SX_DENSE(SX_GT, x[i] > lo)
    SX_DENSE(SX_GE, x[i] >= lo)
    SX_DENSE(SX_EQ, x[i] == lo)
    SX_DENSE(SX_NE, x[i] != lo)
    default:
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) m |= ((lo <= x[i] && x[i] <= hi) ? 1u : 0u) << i;
#undef SX_DENSE
  }
  mask &= m;
}

struct ConjFn {
  static constexpr int kDenseItems = 16;
  template <int ITEMS>
  __device__ __forceinline__ void eval_dense(int64_t r0, int64_t n, uint32_t& mask, int32_t (&)[ITEMS]) const {
    const bool full = r0 + ITEMS <= n;
    mask = dense_valid<ITEMS>(r0, n);
    for (int p = 0; p < np; ++p) dense_pred<ITEMS>(cols[preds[p].col], preds[p], r0, n, full, mask);
  }
  DCol cols[SX_MAX_COLS];
  DPred preds[SX_MAX_PREDS];
  int np;
  template <int ITEMS>
  __device__ __forceinline__ void eval(const int32_t (&row)[ITEMS], const bool (&valid)[ITEMS], bool (&alive)[ITEMS],
                                       int32_t (&aux)[ITEMS]) const {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) alive[i] = valid[i];
    for (int p = 0; p < np; ++p) apply_pred<ITEMS>(cols[preds[p].col], preds[p], row, alive);
  }
};

// LIKE '%pattern%' as a byte-substring test on an Arrow large-string column (reading R9).
struct ContainsFn {
  static constexpr int kMaxPat = 32;
  const int64_t* offsets;
  const uint8_t* chars;
  int plen;
  uint8_t pat[kMaxPat];
  __device__ __forceinline__ bool contains(int64_t r) const {
    int64_t s = __ldg(offsets + r), e = __ldg(offsets + r + 1);
    if (plen == 0) return true;
    const uint8_t p0 = pat[0];
    for (int64_t st = s; st + plen <= e; ++st) {
      if (__ldg(chars + st) != p0) continue;
      bool m = true;
      for (int j = 1; j < plen; ++j)
        if (__ldg(chars + st + j) != pat[j]) { m = false; break; }
      if (m) return true;
    }
    return false;
  }
  template <int ITEMS>
  __device__ __forceinline__ void eval(const int32_t (&row)[ITEMS], const bool (&valid)[ITEMS], bool (&alive)[ITEMS],
                                       int32_t (&aux)[ITEMS]) const {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) alive[i] = valid[i] && contains(row[i]);
  }
  // Dense (no input selection), warp-cooperative: the 32 x ITEMS consecutive strings of a warp
  // occupy one contiguous byte span [offsets[wr0], offsets[wr1]), which the warp streams with
  // coalesced 16-byte loads (lane l reads bytes 16l.. of each 512-byte step).  Bytes equal to the
  // pattern's first byte are candidates; a candidate is verified byte by byte (L1/L2 hits) and,
  // if the whole pattern lies inside one string, that string's row is found by binary search
  // over the warp's offsets and its bit set in the owning thread's mask (shared memory).  Every
  // lane of the warp must call this (k_compact_dense: warp_coop).
  static constexpr int kDenseItems = 16;
  static constexpr int kMinBlocks = 4;
  static constexpr bool kWarpCoop = true;
  template <int ITEMS>
  __device__ __forceinline__ void eval_dense(int64_t r0, int64_t n, uint32_t& mask, int32_t (&)[ITEMS]) const {
    __shared__ uint32_t s_hit[kBlock];
    const int lane = threadIdx.x & 31;
    const int64_t wr0 = r0 - (int64_t)lane * ITEMS;
    mask = 0;
    if (wr0 >= n) return;  // warp-uniform
    const uint32_t valid = dense_valid<ITEMS>(r0, n);
    if (plen == 0) {
      mask = valid;
      return;
    }
    const int64_t wr1 = wr0 + 32 * ITEMS < n ? wr0 + 32 * ITEMS : n;
    s_hit[threadIdx.x] = 0;
    const int64_t S = __ldg(offsets + wr0), E = __ldg(offsets + wr1);
    // the warp's string offsets relative to S, staged once with coalesced loads (the row search
    // of each match then runs in shared memory instead of chasing offsets lines in HBM)
    __shared__ int32_t s_off[kBlock / 32][32 * ITEMS + 1];
    int32_t* wo = s_off[threadIdx.x >> 5];
    const int nr = (int)(wr1 - wr0);
    for (int k = lane; k <= nr; k += 32) wo[k] = (int32_t)(__ldg(offsets + wr0 + k) - S);
    __syncwarp();
    // Candidates are 4-byte windows equal to the pattern's first min(plen, 4) bytes: each lane
    // forms the 16 windows that start in its 16 bytes (funnel shifts over its 4 words plus the
    // next lane's first word), so only true prefix matches reach the byte-wise verification.
    uint32_t p4 = 0, pm = 0;
    for (int k = 0; k < 4 && k < plen; ++k) {
      p4 |= (uint32_t)pat[k] << (8 * k);
      pm |= 0xFFu << (8 * k);
    }
    const uintptr_t a0 = ((uintptr_t)(chars + S)) & ~(uintptr_t)15;
    const uintptr_t aE = (uintptr_t)(chars + E);
    constexpr int kSteps = 4;  // 512-byte warp steps per trip (16 B in flight per lane and step)
    for (uintptr_t cb = a0; cb < aE; cb += 512 * kSteps) {  // warp-uniform
      uint4 v[kSteps];
#pragma unroll
      for (int h = 0; h < kSteps; ++h) {
        const uintptr_t p = cb + 512 * h + 16 * lane;
        v[h] = p < aE ? __ldg((const uint4*)p) : make_uint4(0u, 0u, 0u, 0u);
      }
      uint32_t cm[kSteps];
#pragma unroll
      for (int h = 0; h < kSteps; ++h) {
        // bytes 16..19 after this lane's chunk: the next lane's first word (lane 31: the next
        // step's lane 0, or a load past the trip)
        uint32_t nx = __shfl_down_sync(0xffffffffu, v[h].x, 1);
        const uint32_t n0 = __shfl_sync(0xffffffffu, h + 1 < kSteps ? v[h + 1 < kSteps ? h + 1 : h].x : 0u, 0);
        if (lane == 31) {
          if (h + 1 < kSteps) {
            nx = n0;
          } else {
            const uintptr_t p = cb + 512 * kSteps;
            nx = p < aE ? __ldg((const uint32_t*)p) : 0u;
          }
        }
        const uint32_t w[5] = {v[h].x, v[h].y, v[h].z, v[h].w, nx};
        uint32_t c = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          c |= (((w[i] & pm) == p4) ? 1u : 0u) << (4 * i);
#pragma unroll
          for (int o = 1; o < 4; ++o) c |= (((__funnelshift_r(w[i], w[i + 1], 8 * o) & pm) == p4) ? 1u : 0u) << (4 * i + o);
        }
        cm[h] = c;
      }
#pragma unroll
      for (int h = 0; h < kSteps; ++h) {
        uint32_t c = cm[h];
        while (c) {
          const int j = __ffs(c) - 1;
          c &= c - 1;
          const int64_t q = (int64_t)((const uint8_t*)(cb + 512 * h + 16 * lane) - chars) + j;
          if (q < S || q + plen > E) continue;
          bool ok = true;
          for (int k = 4; k < plen && ok; ++k) ok = __ldg(chars + q + k) == pat[k];
          if (!ok) continue;
          const int32_t qr = (int32_t)(q - S);
          int lo = 0, hi = nr - 1;  // last row whose string starts at or before q
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (wo[mid] <= qr) lo = mid;
            else hi = mid - 1;
          }
          if (qr + plen <= wo[lo + 1]) atomicOr(&s_hit[(threadIdx.x & ~31) + lo / ITEMS], 1u << (lo % ITEMS));
        }
      }
    }
    __syncwarp();
    mask = s_hit[threadIdx.x] & valid;
  }
};

sx_status filter_internal(sx_ctx* ctx, const sx_col* cols, int ncols, const sx_pred* conj, int npred,
                          const sx_sel* in_sel, const int32_t* gather_cols, int ngather, sx_sel* out_sel,
                          sx_col* out_cols);

}  // namespace sx
