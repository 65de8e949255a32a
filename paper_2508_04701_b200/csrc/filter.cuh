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

struct ConjFn {
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
};

sx_status filter_internal(sx_ctx* ctx, const sx_col* cols, int ncols, const sx_pred* conj, int npred,
                          const sx_sel* in_sel, const int32_t* gather_cols, int ngather, sx_sel* out_sel,
                          sx_col* out_cols);

}  // namespace sx
