// join.cuh — hash-table slot layout, the table hash and the specialised probe functors.
#pragma once
#include <stdint.h>

#include "common.cuh"
#include "filter.cuh"

namespace sx {

struct __align__(16) HtSlot8 {
  unsigned long long key;
  unsigned int row;  // 0xFFFFFFFF = empty
  unsigned int pad;
};

// murmur3 fmix32 (bijective on u32): the slot hash for 32-bit keys (tables <= 2^32 slots).
__host__ __device__ __forceinline__ uint32_t hash32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}

// Slot hash used by build and every probe path: 32-bit keys hash in 32 bits, others in 64.
__device__ __forceinline__ uint64_t table_hash(uint64_t key, int key_bytes) {
  return key_bytes == 4 ? (uint64_t)hash32((uint32_t)key) : hash64(key);
}

// ---- payload tables (executor-internal): unique keys with an inline 8-byte payload -----------
// 16-byte slots {x, y}: KB 4: x = key32 (high word 0) or ~0 = EMPTY; KB 8: x = key64 (~0 reserved
// for EMPTY); y = the payload (any fixed-width integer column value, sign-extended).  A lookup is
// one 16-byte load per probe step: the payload comes with the key, no second random access.
// Compact form (32-bit key and a payload that fits 32 bits): 8-byte slots (payload32 << 32) | key32
// claimed by one 64-bit CAS; ~0 = EMPTY (the entry key = payload = -1 is refused at build).
// Tables larger than L2 are built radix-partitioned (pbits > 0): region r = hash64(key) bits 48..
// (the H5 partition function of the key as a signed 64-bit value) holds that partition's keys in
// its own mask+1 slots, and each wave of regions is built while it is L2-resident.
struct PayloadTable {
  ulonglong2* slots = nullptr;
  uint32_t mask = 0;  // slots per region - 1
  int pbits = 0;      // 0: one region
  int kb = 4;
  int compact = 0;    // 8-byte slots
  int64_t rows = 0;
};

__device__ __forceinline__ uint64_t pt_region_base(uint64_t pkey, int pbits, uint32_t mask) {
  return pbits ? (uint64_t)((uint32_t)(hash64(pkey) >> 48) & ((1u << pbits) - 1u)) * ((uint64_t)mask + 1) : 0ull;
}

// pkey: the key as a signed 64-bit value (region choice); key: the 32-bit key stored in the slot
__device__ __forceinline__ bool pt_find_compact(const unsigned long long* __restrict__ slots, uint32_t mask, int pbits,
                                                uint64_t pkey, uint32_t key, int64_t& payload) {
  const unsigned long long* reg = slots + pt_region_base(pkey, pbits, mask);
  uint32_t h = hash32(key) & mask;
  for (;;) {
    const unsigned long long v = __ldg(reg + h);
    if (v == ~0ull) return false;
    if ((uint32_t)v == key) {
      payload = (int64_t)(int32_t)(v >> 32);
      return true;
    }
    h = (h + 1) & mask;
  }
}

template <int KB>
__device__ __forceinline__ bool pt_find(const ulonglong2* __restrict__ slots, uint32_t mask, int pbits, uint64_t key,
                                        int64_t& payload) {
  const uint64_t want = KB == 4 ? (uint64_t)(uint32_t)key : key;
  const ulonglong2* reg = slots + pt_region_base(key, pbits, mask);
  uint32_t h = (uint32_t)(KB == 4 ? hash32((uint32_t)key) : hash64(key)) & mask;
  for (;;) {
    const ulonglong2 v = __ldg(reg + h);
    if (v.x == ~0ull) return false;
    if (v.x == want) {
      payload = (int64_t)v.y;
      return true;
    }
    h = (h + 1) & mask;
  }
}

// Builds a PayloadTable over the selected rows (sel or all n rows of the key columns): key = one
// 32/64-bit column or two 32-bit columns packed (k0 << 32) | k1; payload = column `pay`.
// SX_EINVAL if a key repeats (the table is for PK sides) or equals the reserved EMPTY value.
sx_status build_payload_table(sx_ctx* ctx, const sx_col* keys, int nkeys, const sx_col& pay, const sx_sel* sel,
                              PayloadTable* out, bool allow_compact = true);
void free_payload_table(sx_ctx* ctx, PayloadTable* t);

// Semi / anti membership through the build's exact key-range bitmap only (one key column of type
// KT): no table code, so 16 rows per thread fit the registers and the scan keeps more loads in
// flight.  Also phase 1 of the two-phase unique INNER probe.
template <typename KT>
struct BitmapFn {
  DCol cols[SX_MAX_COLS];
  DPred preds[SX_MAX_PREDS];
  int np;
  const KT* k0;
  const uint32_t* bm;
  long long bm_min;
  unsigned long long bm_bits;
  int anti;
  static constexpr int kDenseItems = 16;
  static constexpr int kMinBlocks = 4;  // light functor: 4 CTAs (32 warps) per SM
  template <int ITEMS>
  __device__ __forceinline__ bool hit(int64_t key, bool live) const {
    const unsigned long long off = (unsigned long long)(key - bm_min);
    const bool in = live && off < bm_bits;
    const uint32_t w = in ? __ldg(bm + (off >> 5)) : 0u;
    return in && ((w >> (off & 31)) & 1u);
  }
  template <int ITEMS>
  __device__ __forceinline__ void eval(const int32_t (&row)[ITEMS], const bool (&valid)[ITEMS], bool (&alive)[ITEMS],
                                       int32_t (&)[ITEMS]) const {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) alive[i] = valid[i];
    for (int p = 0; p < np; ++p) apply_pred<ITEMS>(cols[preds[p].col], preds[p], row, alive);
    int64_t key[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) key[i] = alive[i] ? (int64_t)__ldg(k0 + row[i]) : 0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const bool h = hit<ITEMS>(key[i], alive[i]);
      alive[i] = alive[i] && (anti ? !h : h);
    }
  }
  template <int ITEMS>
  __device__ __forceinline__ void eval_dense(int64_t r0, int64_t n, uint32_t& mask, int32_t (&)[ITEMS]) const {
    const bool full = r0 + ITEMS <= n;
    mask = dense_valid<ITEMS>(r0, n);
    for (int p = 0; p < np; ++p) dense_pred<ITEMS>(cols[preds[p].col], preds[p], r0, n, full, mask);
    uint32_t m = 0;
    if constexpr (sizeof(KT) == 4) {  // 32-bit keys stay 32-bit until the bitmap offset
      int32_t k[ITEMS];
      dense_load32<ITEMS>((const int32_t*)k0, r0, n, full, k);
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const bool live = (mask >> i) & 1u;
        const bool h = hit<ITEMS>((int64_t)k[i], live);
        m |= ((live && (anti ? !h : h)) ? 1u : 0u) << i;
      }
    } else {
      int64_t k[ITEMS];
      dense_load<ITEMS>(DCol{k0, SX_I64, 0}, r0, n, full, k);
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const bool live = (mask >> i) & 1u;
        const bool h = hit<ITEMS>(k[i], live);
        m |= ((live && (anti ? !h : h)) ? 1u : 0u) << i;
      }
    }
    mask = m;
  }
};

// Probe functor specialised on the key column type KT (int32_t / long long), the number of key
// columns NK (2: two int32 columns packed (k0 << 32) | k1, reading R11) and the table layout KB.
// All ITEMS key loads are issued back to back, then all first-slot loads, then the (rare) longer
// chains; semi/anti/unique-inner emit at most one output per probe row (ordered compaction).
template <typename KT, int NK, int KB, bool CNT = false>
struct ProbeFnT {
  DCol cols[SX_MAX_COLS];
  DPred preds[SX_MAX_PREDS];
  int np;
  const KT* k0;
  const int32_t* k1;
  const void* slots;
  uint32_t mask;
  int anti;
  int member_only;     // semi/anti: membership is the whole answer
  // CNT: inner join on a non-unique build: aux = number of matches (scan to the first EMPTY)
  static constexpr bool count_all = CNT;
  const uint32_t* bm;  // optional exact key-range bitmap of the build side
  long long bm_min;
  unsigned long long bm_bits;
  const int32_t* direct;  // unique direct-address build: row at [key - bm_min] (no table)
  template <int ITEMS>
  __device__ __forceinline__ void eval(const int32_t (&row)[ITEMS], const bool (&valid)[ITEMS], bool (&alive)[ITEMS],
                                       int32_t (&aux)[ITEMS]) const {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) alive[i] = valid[i];
    for (int p = 0; p < np; ++p) apply_pred<ITEMS>(cols[preds[p].col], preds[p], row, alive);
    uint64_t key[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) key[i] = alive[i] ? (uint64_t)(int64_t)__ldg(k0 + row[i]) : 0;
    if (NK == 2) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i)
        key[i] = (key[i] << 32) | (uint32_t)(alive[i] ? __ldg(k1 + row[i]) : 0);
    }
    probe<ITEMS>(key, alive, aux);
  }
  // Dense path (no input selection): predicate and key columns of ITEMS consecutive rows with
  // 128-bit vector loads, all issued before the bitmap / table lookups.
  static constexpr int kDenseItems = 8;
  template <int ITEMS>
  __device__ __forceinline__ void eval_dense(int64_t r0, int64_t n, uint32_t& mask, int32_t (&aux)[ITEMS]) const {
    const bool full = r0 + ITEMS <= n;
    mask = dense_valid<ITEMS>(r0, n);
    int64_t k[ITEMS];
    dense_load<ITEMS>(DCol{k0, sizeof(KT) == 4 ? SX_I32 : SX_I64, 0}, r0, n, full, k);
    for (int p = 0; p < np; ++p) dense_pred<ITEMS>(cols[preds[p].col], preds[p], r0, n, full, mask);
    uint64_t key[ITEMS];
    bool alive[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      alive[i] = (mask >> i) & 1u;
      key[i] = (uint64_t)k[i];
    }
    if (NK == 2) {
      int64_t k2[ITEMS];
      dense_load<ITEMS>(DCol{k1, SX_I32, 0}, r0, n, full, k2);
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) key[i] = (key[i] << 32) | (uint32_t)k2[i];
    }
    probe<ITEMS>(key, alive, aux);
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) m |= (alive[i] ? 1u : 0u) << i;
    mask = m;
  }
  template <int ITEMS>
  __device__ __forceinline__ void probe(uint64_t (&key)[ITEMS], bool (&alive)[ITEMS], int32_t (&aux)[ITEMS]) const {
    if (direct) {  // bitmap word + one 4-byte read (candidates from a bitmap pass skip the bitmap)
      bool hit[ITEMS];
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const unsigned long long off = (unsigned long long)((long long)key[i] - bm_min);
        hit[i] = alive[i] && off < bm_bits;
        if (bm) {
          const uint32_t w = hit[i] ? __ldg(bm + (off >> 5)) : 0u;
          hit[i] = hit[i] && ((w >> (off & 31)) & 1u);
        }
        if (hit[i] && !member_only) aux[i] = __ldg(direct + off);
      }
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) alive[i] = alive[i] && (anti ? !hit[i] : hit[i]);
      return;
    }
    uint32_t h[ITEMS];
    bool pend[ITEMS], found[ITEMS];
    uint32_t cnt[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) cnt[i] = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      h[i] = (uint32_t)(KB == 4 ? hash32((uint32_t)key[i]) : hash64(key[i])) & mask;
      pend[i] = alive[i];
      found[i] = false;
    }
    if (bm) {  // exact pre-filter: keys absent from the build never touch the table
      uint32_t w[ITEMS];
      unsigned long long off[ITEMS];
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        off[i] = (unsigned long long)((long long)key[i] - bm_min);
        pend[i] = pend[i] && off[i] < bm_bits;
        w[i] = pend[i] ? __ldg(bm + (off[i] >> 5)) : 0u;
      }
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) pend[i] = pend[i] && ((w[i] >> (off[i] & 31)) & 1u);
      if (member_only) {  // semi / anti: the exact bitmap is the answer, the table is not needed
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) alive[i] = alive[i] && (anti ? !pend[i] : pend[i]);
        return;
      }
    }
    bool any = true;
    if (KB == 4) {
      // two 8-byte slots per 16-byte load: the aligned pair holding h, then h+2, ...  In the first
      // pair of an odd h the even slot precedes the home slot: it can never hold this key (equal
      // keys share the home slot and lie at or after it) and its emptiness must not stop the scan.
      bool first[ITEMS];
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        first[i] = (h[i] & 1u) != 0;
        h[i] &= ~1u;
      }
      while (any) {
        any = false;
        ulonglong2 s[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i)
          s[i] = pend[i] ? __ldg((const ulonglong2*)slots + (h[i] >> 1)) : make_ulonglong2(~0ull, ~0ull);
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          if (!pend[i]) continue;
          uint32_t r0 = (uint32_t)(s[i].x >> 32), r1 = (uint32_t)(s[i].y >> 32);
          bool e0 = r0 == 0xffffffffu && !first[i], e1 = r1 == 0xffffffffu;
          bool m0 = r0 != 0xffffffffu && !first[i] && (uint32_t)s[i].x == (uint32_t)key[i];
          bool m1 = !e0 && r1 != 0xffffffffu && (uint32_t)s[i].y == (uint32_t)key[i];
          if constexpr (CNT) {  // every match up to the first EMPTY slot
            cnt[i] += (m0 ? 1 : 0) + (m1 ? 1 : 0);
            pend[i] = !(e0 || e1);
          } else {
            bool h1 = m1 && !m0;
            found[i] |= m0 || h1;
            if (m0) aux[i] = (int32_t)r0;
            if (h1) aux[i] = (int32_t)r1;
            pend[i] = !(e0 || m0 || e1 || h1);
          }
          first[i] = false;
          h[i] = (h[i] + 2) & mask;
          any |= pend[i];
        }
      }
    }
    while (any) {
      any = false;
      if (KB == 4) {
      } else {
        longlong2 s[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) s[i] = pend[i] ? __ldg((const longlong2*)slots + h[i]) : make_longlong2(0, -1);
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          if (!pend[i]) continue;
          uint32_t rw = (uint32_t)(unsigned long long)s[i].y;
          bool empty = rw == 0xffffffffu, hit = !empty && (uint64_t)s[i].x == key[i];
          if constexpr (CNT) {
            cnt[i] += hit ? 1 : 0;
            pend[i] = !empty;
          } else {
            found[i] |= hit;
            if (hit) aux[i] = (int32_t)rw;
            pend[i] = !empty && !hit;
          }
          h[i] = (h[i] + 1) & mask;
          any |= pend[i];
        }
      }
    }
    if constexpr (CNT) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        alive[i] = alive[i] && cnt[i] > 0;
        aux[i] = (int32_t)cnt[i];
      }
      return;
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) alive[i] = alive[i] && (anti ? !found[i] : found[i]);
  }
};

}  // namespace sx
