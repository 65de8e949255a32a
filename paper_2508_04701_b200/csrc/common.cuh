// common.cuh — libsx internals: context, errors, stream-ordered allocation,
// device-side column access, expression evaluation, hashing, int128 atomics,
// warp helpers and the decoupled look-back tile scan.
//
// Nothing here is shared with oracle/ (task rule ③).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "sx.h"

#define SX_EXPORT extern "C" __attribute__((visibility("default")))

namespace sx {

constexpr int kBlock = 256;  // threads per CTA for streaming kernels
constexpr unsigned kFull = 0xffffffffu;

}  // namespace sx

// ---------------------------------------------------------------------------- context
struct sx_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  size_t l2_bytes = 0;
  std::string err;
  int* d_flags = nullptr;          // [0] expression overflow, [1] table full, [2..] scratch
  unsigned int* d_counters = nullptr;  // tile counters etc. (64 entries)
  int64_t* h_pinned = nullptr;     // pinned host scratch for size reads (64 entries)
  void* h_stage = nullptr;         // pinned host staging for result rows (grown on demand)
  size_t h_stage_bytes = 0;
  bool profile = false;
  int64_t launches = 0;            // kernels launched by libsx on this ctx (sx_launch_count)
  struct Prof { char name[32]; cudaEvent_t a, b; double bytes; };
  std::vector<Prof> prof;
};

struct sx_ht {
  int key_bytes = 4;       // 4: slot {u32 key, u32 row}; 8: slot {u64 key, u32 row, u32 pad}
  int key_types[2] = {SX_I32, SX_I32};
  int nkeys = 1;
  int unique = 0;
  uint64_t cap = 0;        // slots (power of two)
  void* slots = nullptr;
  int64_t rows = 0;        // inserted build rows
  uint32_t* bm = nullptr;  // exact bitmap over [bm_min, bm_min + bm_bits) of the build keys (or null)
  int32_t* direct = nullptr;  // unique builds over a small key range: build row at [key - bm_min] (no table)
  long long bm_min = 0;
  unsigned long long bm_bits = 0;
};

namespace sx {

// ---------------------------------------------------------------------------- errors
inline sx_status set_err(sx_ctx* c, sx_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return s;
}

#define SX_CUDA(call)                                                                              \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) return ::sx::set_err(ctx, SX_ECUDA, "%s: %s (%s:%d)", #call,           \
                                                cudaGetErrorString(e_), __FILE__, __LINE__);       \
  } while (0)

#define SX_CHECK_LAUNCH() SX_CUDA(cudaGetLastError())

// Launch-configuration stream argument that also counts the launch (evaluated only when the
// launch statement executes).
#define SX_STREAM(c) ((++(c)->launches), (c)->stream)

#define SX_TRY(expr)                    \
  do {                                  \
    sx_status s_ = (expr);              \
    if (s_ != SX_OK) return s_;         \
  } while (0)

// ---------------------------------------------------------------------------- allocation
// Stream-ordered pool allocation (the paper's RMM "processing region").
template <class T>
inline sx_status alloc(sx_ctx* ctx, T** p, size_t n) {
  *p = nullptr;
  size_t bytes = n * sizeof(T);
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMallocAsync((void**)p, bytes, ctx->stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return set_err(ctx, SX_ENOMEM, "device pool exhausted allocating %zu bytes", bytes);
  }
  return SX_OK;
}
inline void dfree(sx_ctx* ctx, void* p) {
  if (p) cudaFreeAsync(p, ctx->stream);
}

// Frees every registered temporary at scope exit (stream-ordered).
struct Scratch {
  sx_ctx* ctx;
  std::vector<void*> ptrs;
  explicit Scratch(sx_ctx* c) : ctx(c) {}
  template <class T>
  sx_status get(T** p, size_t n) {
    sx_status s = alloc(ctx, p, n);
    if (s == SX_OK) ptrs.push_back(*p);
    return s;
  }
  void release(void* p) {  // ownership moves to the caller
    for (auto& q : ptrs)
      if (q == p) q = nullptr;
  }
  ~Scratch() {
    for (void* q : ptrs) dfree(ctx, q);
  }
};

// Scoped per-operator timing (sx_profile_enable).
struct ProfScope {
  sx_ctx* ctx;
  int idx = -1;
  ProfScope(sx_ctx* c, const char* name) : ctx(c) {
    if (!c->profile) return;
    sx_ctx::Prof p;
    snprintf(p.name, sizeof p.name, "%s", name);
    p.bytes = 0;
    cudaEventCreate(&p.a);
    cudaEventCreate(&p.b);
    cudaEventRecord(p.a, c->stream);
    c->prof.push_back(p);
    idx = (int)c->prof.size() - 1;
  }
  ~ProfScope() {
    if (idx >= 0) cudaEventRecord(ctx->prof[idx].b, ctx->stream);
  }
  bool on() const { return idx >= 0; }
  // Algorithmic bytes of this call (SURVEY §8(d) "Bytes definitions" 1).
  void set_bytes(double b) {
    if (idx >= 0) ctx->prof[idx].bytes = b;
  }
};

inline int type_width(int t) {
  switch (t) {
    case SX_U8: return 1;
    case SX_I32: case SX_DATE32: return 4;
    case SX_I64: case SX_DEC64: case SX_F64: return 8;
    case SX_I128: return 16;
    default: return 0;
  }
}
// Referenced-column set of one call, for its algorithmic bytes (SURVEY §8(d) definition 1:
// each referenced input column read once at its stored width).
struct RefCols {
  bool used[SX_MAX_COLS] = {};
  void add(int c) {
    if (c >= 0 && c < SX_MAX_COLS) used[c] = true;
  }
  double row_bytes(const sx_col* cols, int ncols) const {
    double b = 0;
    for (int c = 0; c < ncols && c < SX_MAX_COLS; ++c)
      if (used[c]) b += cols[c].type == SX_STR ? 8.0 : (double)type_width(cols[c].type);
    return b;
  }
};

inline bool is_int_type(int t) {
  return t == SX_U8 || t == SX_I32 || t == SX_DATE32 || t == SX_I64 || t == SX_DEC64;
}
inline int key_bits(int t) { return (t == SX_I64 || t == SX_DEC64) ? 64 : (t == SX_U8 ? 8 : 32); }

// ---------------------------------------------------------------------------- device columns
struct DCol {
  const void* p;
  int32_t type;
  int32_t pad;
};

struct DPred {
  int32_t col, op;
  int64_t lo, hi;
};

__device__ __forceinline__ int64_t ldv(const DCol& c, int64_t r) {
  switch (c.type) {
    case SX_U8: return (int64_t)__ldg((const uint8_t*)c.p + r);
    case SX_I32:
    case SX_DATE32: return (int64_t)__ldg((const int32_t*)c.p + r);
    default: return (int64_t)__ldg((const long long*)c.p + r);
  }
}

__device__ __forceinline__ bool cmp(int op, int64_t x, int64_t lo, int64_t hi) {
  switch (op) {
    case SX_LT: return x < lo;
    case SX_LE: return x <= lo;
    case SX_GT: return x > lo;
    case SX_GE: return x >= lo;
    case SX_EQ: return x == lo;
    case SX_NE: return x != lo;
    default: return lo <= x && x <= hi;  // SX_BETWEEN
  }
}

// Conjunction of predicates, column loads only while the row is still alive (lazy / short-circuit).
__device__ __forceinline__ bool eval_conj(const DCol* cols, const DPred* preds, int np, int64_t r) {
  bool ok = true;
  for (int i = 0; i < np; ++i) {
    if (!ok) break;
    ok = cmp(preds[i].op, ldv(cols[preds[i].col], r), preds[i].lo, preds[i].hi);
  }
  return ok;
}

// ---------------------------------------------------------------------------- exact int64 arithmetic
__device__ __forceinline__ bool fits_i32(int64_t a) { return (uint64_t)(a + 0x80000000ll) < 0x100000000ull; }

__device__ __forceinline__ int64_t mul_ck(int64_t a, int64_t b, bool& ovf) {
  // fast path: both operands in int32 range -> one IMAD.WIDE, cannot overflow int64
  if (fits_i32(a) && fits_i32(b)) return (int64_t)(int32_t)a * (int64_t)(int32_t)b;
  int64_t lo = (int64_t)((uint64_t)a * (uint64_t)b);
  int64_t hi = __mul64hi(a, b);
  ovf |= (hi != (lo >> 63));
  return lo;
}
__device__ __forceinline__ int64_t add_ck(int64_t a, int64_t b, bool& ovf) {
  int64_t s = (int64_t)((uint64_t)a + (uint64_t)b);
  ovf |= ((a ^ s) & (b ^ s)) < 0;
  return s;
}

__device__ __forceinline__ int64_t eval_expr(const sx_expr& e, const DCol* cols, int64_t r, bool& ovf) {
  int64_t v = 0;
  for (int t = 0; t < e.nterms; ++t) {
    const sx_term& tm = e.t[t];
    int64_t p = tm.coef;
    for (int f = 0; f < tm.nf; ++f) {
      int64_t x = ldv(cols[tm.f[f].col], r);
      if (tm.f[f].mul != 1) x = mul_ck(tm.f[f].mul, x, ovf);
      if (tm.f[f].add != 0) x = add_ck(x, tm.f[f].add, ovf);
      p = (f == 0 && tm.coef == 1) ? x : mul_ck(p, x, ovf);
    }
    v = (t == 0) ? p : add_ck(v, p, ovf);
  }
  return v;
}

// ---------------------------------------------------------------------------- hashing
// murmur3 fmix64: bijective mixer; slot = low bits, shard rank = high bits (disjoint fields, reading R14).
__host__ __device__ __forceinline__ uint64_t hash64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

// proleptic Gregorian year of a day number (days since 1970-01-01); closed-form civil-from-days.
__host__ __device__ __forceinline__ int32_t civil_year(int32_t z) {
  z += 719468;
  int32_t era = (z >= 0 ? z : z - 146096) / 146097;
  int32_t doe = z - era * 146097;
  int32_t yoe = (doe - doe / 1460 + doe / 36524 - doe / 146096) / 365;
  int32_t y = yoe + era * 400;
  int32_t doy = doe - (365 * yoe + yoe / 4 - yoe / 100);
  int32_t mp = (5 * doy + 2) / 153;
  int32_t m = mp < 10 ? mp + 3 : mp - 9;
  return y + (m <= 2);
}

// ---------------------------------------------------------------------------- atomics / memory order
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// int128 sum kept as {u64 lo; i32 hi} (96 bits suffice: <= 2^31 rows x |v| < 2^63 < 2^94).
// Carry-propagating pair of atomics: correct under any interleaving because each lo add
// reports its own carry-out.
__device__ __forceinline__ void atomic_add_sum96(unsigned long long* lo, int* hi, int64_t vlo_signed_hi_ext,
                                                 int32_t vhi) {
  unsigned long long v = (unsigned long long)vlo_signed_hi_ext;
  unsigned long long old = atomicAdd(lo, v);
  int carry = (old + v) < old ? 1 : 0;
  int h = vhi + carry;
  if (h) atomicAdd(hi, h);
}
// add a signed int64 to a sum96
__device__ __forceinline__ void atomic_add_i64_to_sum96(unsigned long long* lo, int* hi, int64_t v) {
  atomic_add_sum96(lo, hi, v, v < 0 ? -1 : 0);
}

// ---------------------------------------------------------------------------- warp helpers
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// ---------------------------------------------------------------------------- decoupled look-back
// Tile prefix over per-tile counts in one pass (Merrill & Garland's chained scan).
// status word: [63:62] flag (0 invalid, 1 aggregate, 2 inclusive) | [61:0] value.
// Must be called by ALL 32 lanes of exactly one warp per tile; returns the exclusive prefix.
__device__ __forceinline__ int64_t lookback_exclusive(unsigned long long* status, int64_t tile, int64_t count) {
  const unsigned long long AGG = 1ull << 62, INC = 2ull << 62, VMASK = (1ull << 62) - 1;
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed(&status[0], INC | (unsigned long long)count);
    return 0;
  }
  if (lane == 0) st_relaxed(&status[tile], AGG | (unsigned long long)count);
  int64_t excl = 0;
  int64_t j = tile - 1;
  while (true) {
    int64_t idx = j - lane;
    unsigned long long w;
    do {
      w = idx >= 0 ? ld_relaxed(&status[idx]) : INC;
    } while (__any_sync(kFull, (w >> 62) == 0));
    unsigned inc = __ballot_sync(kFull, (w >> 62) == 2);
    int first = inc ? __ffs(inc) - 1 : 32;
    int64_t v = (lane <= first) ? (int64_t)(w & VMASK) : 0;
    excl += warp_sum64(v);
    if (inc) break;
    j -= 32;
  }
  if (lane == 0) st_relaxed(&status[tile], INC | (unsigned long long)(excl + count));
  return excl;
}

// ---------------------------------------------------------------------------- launch sizing
inline unsigned persistent_grid(sx_ctx* ctx, int blocks_per_sm, int64_t work_tiles) {
  int64_t g = (int64_t)ctx->num_sms * blocks_per_sm;
  if (work_tiles < g) g = work_tiles;
  return (unsigned)(g < 1 ? 1 : g);
}

// The ABI's alignment rule (sx.h "Conventions"): the dense kernels load 16 bytes at a time
// (Q1/Q6 programs, K10w, unselected compaction), so a misaligned buffer would fault (a sticky
// error that kills the context) and a strided view would be misread: reject both up front.
inline sx_status check_aligned(sx_ctx* ctx, const sx_col& c, int i) {
  // (string bytes may start anywhere: the CONTAINS scan aligns its own windows)
  if (c.len > 0 && c.type != SX_STR && ((uintptr_t)c.data & 15u))
    return set_err(ctx, SX_EINVAL, "column %d data %p is not 16-byte aligned", i, c.data);
  if (c.type == SX_STR && c.offsets && ((uintptr_t)c.offsets & 7u))
    return set_err(ctx, SX_EINVAL, "column %d offsets %p are not 8-byte aligned", i, (const void*)c.offsets);
  return SX_OK;
}

// Validate a column array for device kernels; fills DCol[].
inline sx_status to_dcols(sx_ctx* ctx, const sx_col* cols, int ncols, DCol* out) {
  if (ncols < 0 || ncols > SX_MAX_COLS) return set_err(ctx, SX_EINVAL, "ncols %d out of range", ncols);
  if (ncols > 0 && !cols) return set_err(ctx, SX_EINVAL, "cols is NULL");
  for (int i = 0; i < ncols; ++i) {
    SX_TRY(check_aligned(ctx, cols[i], i));
    if (cols[i].validity) return set_err(ctx, SX_EUNSUPPORTED, "column %d has a validity bitmap (null-free v1)", i);
    if (cols[i].len > 0 && !cols[i].data) return set_err(ctx, SX_EINVAL, "column %d data is NULL", i);
    if (cols[i].len > INT32_MAX) return set_err(ctx, SX_EINDEX, "column %d has %lld rows > INT32_MAX", i, (long long)cols[i].len);
    out[i].p = cols[i].data;
    out[i].type = cols[i].type;
    out[i].pad = 0;
  }
  return SX_OK;
}

inline sx_status check_preds(sx_ctx* ctx, const sx_col* cols, int ncols, const sx_pred* p, int np, DPred* out) {
  if (np < 0 || np > SX_MAX_PREDS) return set_err(ctx, SX_EINVAL, "npred %d out of range", np);
  for (int i = 0; i < np; ++i) {
    if (p[i].col < 0 || p[i].col >= ncols) return set_err(ctx, SX_EINVAL, "predicate %d column %d out of range", i, p[i].col);
    if (p[i].op < SX_LT || p[i].op > SX_BETWEEN) return set_err(ctx, SX_EINVAL, "predicate %d: op %d not a fixed-width comparison", i, p[i].op);
    if (!is_int_type(cols[p[i].col].type)) return set_err(ctx, SX_ETYPE, "predicate %d on non-integer column", i);
    out[i].col = p[i].col;
    out[i].op = p[i].op;
    out[i].lo = p[i].lo;
    out[i].hi = p[i].hi;
  }
  return SX_OK;
}

inline sx_status check_expr(sx_ctx* ctx, const sx_col* cols, int ncols, const sx_expr& e) {
  if (e.nterms < 0 || e.nterms > 2) return set_err(ctx, SX_EINVAL, "expression has %d terms (max 2)", e.nterms);
  for (int t = 0; t < e.nterms; ++t) {
    if (e.t[t].nf < 0 || e.t[t].nf > 3) return set_err(ctx, SX_EINVAL, "term has %d factors (max 3)", e.t[t].nf);
    for (int f = 0; f < e.t[t].nf; ++f) {
      int c = e.t[t].f[f].col;
      if (c < 0 || c >= ncols) return set_err(ctx, SX_EINVAL, "expression column %d out of range", c);
      if (!is_int_type(cols[c].type)) return set_err(ctx, SX_ETYPE, "expression column %d is not an integer type", c);
    }
  }
  return SX_OK;
}

// Read one int64 from device (stream-ordered, synchronises the ctx stream once).
inline sx_status read_i64(sx_ctx* ctx, const void* dptr, int64_t* out, int count = 1) {
  SX_CUDA(cudaMemcpyAsync(ctx->h_pinned, dptr, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, ctx->stream));
  SX_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < count; ++i) out[i] = ctx->h_pinned[i];
  return SX_OK;
}

// Internal (C++) entry points shared between operator files and the executor.
struct GatherCol {
  DCol src;
  void* dst;
  int32_t by_aux;  // 0: gather at the output row id; 1: at the aux id (matched build row)
  int32_t width;
};
constexpr int kMaxGather = 16;
struct GatherSpec {
  GatherCol g[kMaxGather];
  int n;
};

__device__ __forceinline__ void gather_one(const GatherCol& g, int64_t pos, int64_t row) {
  switch (g.width) {
    case 1: ((uint8_t*)g.dst)[pos] = __ldg((const uint8_t*)g.src.p + row); break;
    case 4: ((int32_t*)g.dst)[pos] = __ldg((const int32_t*)g.src.p + row); break;
    case 8: ((long long*)g.dst)[pos] = __ldg((const long long*)g.src.p + row); break;
    default: ((longlong2*)g.dst)[pos] = __ldg((const longlong2*)g.src.p + row); break;
  }
}

}  // namespace sx
