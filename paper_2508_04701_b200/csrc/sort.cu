// sort.cu — H9: sx_sort_topk (K13 LSD radix sort, K14 radix-select top-k), CUB-free.
//
// PAPER.md P:191 (sorting via libcudf; here our kernels), P:422 (order-by inputs are small).
// Keys are encoded into order-preserving unsigned 32-bit words, most significant first
// (sign bit flipped; descending = bitwise NOT), followed by the input position, which makes
// every composite key unique and the result stable.  Digits (8 bits) on which
// all rows agree are skipped, so a sort costs passes only over bits that vary.
//   n <= 2048          : one CTA bitonic sort in shared memory
//   k <= 1024 (< n)    : radix select of the k-th key (one pass per varying digit, MSB first),
//                        ordered compaction of the k winners, bitonic sort of those
//   otherwise          : LSD radix sort (per pass: tile histograms, per-digit scan, stable scatter)
#include "compact.cuh"
#include <cstring>
#include <type_traits>

using namespace sx;

namespace {

constexpr int kMaxWords = 9;  // <= 8 key words + position
constexpr int kBitonicMax = 2048;

struct EncArgs {
  DCol cols[4];
  int types[4];
  int desc[4];
  int nkeys;
  int nwords;  // including the position word
  const int32_t* sel;
  int64_t n;
  uint32_t* words[kMaxWords];  // SoA
  unsigned* diff;              // [nwords]
};

__device__ __forceinline__ int encode_row(const EncArgs& a, int64_t r, int64_t pos, uint32_t* w) {
  int k = 0;
  for (int c = 0; c < a.nkeys; ++c) {
    uint32_t m = a.desc[c] ? 0xffffffffu : 0u;
    switch (a.types[c]) {
      case SX_U8: w[k++] = ((uint32_t)((const uint8_t*)a.cols[c].p)[r]) ^ m; break;
      case SX_I32:
      case SX_DATE32: w[k++] = ((uint32_t)((const int32_t*)a.cols[c].p)[r] ^ 0x80000000u) ^ m; break;
      case SX_I128: {
        const long long* p = (const long long*)a.cols[c].p + 2 * r;
        uint64_t lo = (uint64_t)p[0], hi = (uint64_t)p[1] ^ 0x8000000000000000ull;
        w[k++] = (uint32_t)(hi >> 32) ^ m;
        w[k++] = (uint32_t)hi ^ m;
        w[k++] = (uint32_t)(lo >> 32) ^ m;
        w[k++] = (uint32_t)lo ^ m;
        break;
      }
      default: {
        uint64_t u = (uint64_t)((const long long*)a.cols[c].p)[r] ^ 0x8000000000000000ull;
        w[k++] = (uint32_t)(u >> 32) ^ m;
        w[k++] = (uint32_t)u ^ m;
        break;
      }
    }
  }
  w[k++] = (uint32_t)pos;
  return k;
}

__global__ void k_encode(const __grid_constant__ EncArgs a) {
  uint32_t w0[kMaxWords], w[kMaxWords];
  int64_t r0 = a.sel ? (int64_t)a.sel[0] : 0;
  encode_row(a, r0, 0, w0);
  unsigned acc[kMaxWords];
  for (int j = 0; j < kMaxWords; ++j) acc[j] = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = a.sel ? (int64_t)a.sel[i] : i;
    encode_row(a, r, i, w);
    for (int j = 0; j < a.nwords; ++j) {
      a.words[j][i] = w[j];
      acc[j] |= w[j] ^ w0[j];
    }
  }
  for (int j = 0; j < a.nwords; ++j) {
    unsigned v = acc[j];
    for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(kFull, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicOr(a.diff + j, v);
  }
}

struct Words {
  uint32_t* w[kMaxWords];
  int nwords;
};

__device__ __forceinline__ bool key_less(const uint32_t* a, const uint32_t* b, int nw) {
  for (int j = 0; j < nw; ++j)
    if (a[j] != b[j]) return a[j] < b[j];
  return false;
}

// Bitonic sort of m <= 2048 rows (given by positions `pos`, or 0..m-1) in one CTA; writes
// out_perm[0..min(k,m)) = original row ids.
__global__ void __launch_bounds__(1024) k_bitonic(const __grid_constant__ Words W, const int32_t* pos, int64_t m,
                                                  int64_t k, const int32_t* sel, int32_t* out_perm) {
  extern __shared__ uint32_t sm[];  // [N][nwords]
  int nw = W.nwords;
  int N = 1;
  while (N < m) N <<= 1;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    for (int j = 0; j < nw; ++j) {
      uint32_t v = 0xffffffffu;
      if (i < m) {
        int64_t p = pos ? pos[i] : i;
        v = W.w[j][p];
      }
      sm[i * nw + j] = v;
    }
  }
  __syncthreads();
  uint32_t ta[kMaxWords], tb[kMaxWords];
  for (int size = 2; size <= N; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool up = ((lo & size) == 0);
        for (int j = 0; j < nw; ++j) { ta[j] = sm[lo * nw + j]; tb[j] = sm[hi * nw + j]; }
        bool sw = up ? key_less(tb, ta, nw) : key_less(ta, tb, nw);
        if (sw)
          for (int j = 0; j < nw; ++j) { sm[lo * nw + j] = tb[j]; sm[hi * nw + j] = ta[j]; }
      }
      __syncthreads();
    }
  }
  int64_t outn = k < m ? k : m;
  for (int i = threadIdx.x; i < outn; i += blockDim.x) {
    int64_t p = sm[i * nw + (nw - 1)];  // position word
    out_perm[i] = sel ? sel[p] : (int32_t)p;
  }
}

// Top-k tournament round: CTA c sorts rows [2048c, 2048c + 2048) of `pos` (or of 0..m-1) in
// shared memory and keeps its first min(k, len) positions at pos_out[k c ..].  The union of the
// chunks' top-k holds the global top-k (keys are unique: the position word breaks ties), so
// rounds shrink m by >= 2x (k <= 1024) until one k_bitonic finishes; no host synchronisation.
__global__ void __launch_bounds__(1024) k_topk_round(const __grid_constant__ Words W, const int32_t* pos, int64_t m,
                                                     int64_t k, int32_t* pos_out) {
  extern __shared__ uint32_t sm[];  // [N][nwords]
  const int nw = W.nwords;
  const int64_t c0 = (int64_t)blockIdx.x * kBitonicMax;
  const int len = (int)min((int64_t)kBitonicMax, m - c0);
  int N = 1;
  while (N < len) N <<= 1;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const int64_t p = i < len ? (pos ? (int64_t)pos[c0 + i] : c0 + i) : -1;
    for (int j = 0; j < nw; ++j) sm[i * nw + j] = p >= 0 ? W.w[j][p] : 0xffffffffu;
  }
  __syncthreads();
  uint32_t ta[kMaxWords], tb[kMaxWords];
  for (int size = 2; size <= N; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        for (int j = 0; j < nw; ++j) { ta[j] = sm[lo * nw + j]; tb[j] = sm[hi * nw + j]; }
        const bool sw = up ? key_less(tb, ta, nw) : key_less(ta, tb, nw);
        if (sw)
          for (int j = 0; j < nw; ++j) { sm[lo * nw + j] = tb[j]; sm[hi * nw + j] = ta[j]; }
      }
      __syncthreads();
    }
  }
  const int keep = (int)min(k, (int64_t)len);
  for (int i = threadIdx.x; i < keep; i += blockDim.x) pos_out[blockIdx.x * k + i] = (int32_t)sm[i * nw + (nw - 1)];
}

// ---- warp top-k (K14w, k <= 32) --------------------------------------------------------
// Each warp scans a contiguous block of >= k rows keeping its k best composite keys sorted across
// its lanes (lane i: the i-th best, all words in registers).  A row enters only if it beats the
// current k-th best (rare after the first rows: ~k ln(rows/k) insertions per warp), by a
// warp-wide shift.  The warps' lists (warps x k positions) then go through the tournament rounds.
// One pass over the encoded words instead of one radix-select pass per varying digit (Q3's top-10
// of 1.13e6 rows x 7 words: 14 digits, ~30 launches).
__global__ void __launch_bounds__(256) k_topk_warp(const __grid_constant__ Words W, int64_t n, int k, int64_t per,
                                                   int32_t* __restrict__ out_pos) {
  const int lane = threadIdx.x & 31;
  const int nw = W.nwords;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t lo = gw * per, hi = min(n, lo + per);
  if (lo >= n) return;  // (warp-uniform)
  uint32_t mine[kMaxWords];  // my list entry (lane < cnt)
#pragma unroll
  for (int j = 0; j < kMaxWords; ++j) mine[j] = 0xffffffffu;
  int cnt = 0;  // warp-uniform list length
  for (int64_t b = lo; b < hi; b += 32) {
    const int64_t r = b + lane;
    uint32_t w[kMaxWords];
    const bool in = r < hi;
#pragma unroll
    for (int j = 0; j < kMaxWords; ++j) w[j] = (in && j < nw) ? __ldg(W.w[j] + r) : 0xffffffffu;
    // the current k-th best (lane k-1) when the list is full
    bool cand = in;
    if (cnt == k) {
      bool less = false, decided = false;
#pragma unroll
      for (int j = 0; j < kMaxWords; ++j) {
        const uint32_t kj = __shfl_sync(kFull, mine[j], k - 1);
        if (j < nw && !decided && w[j] != kj) {
          less = w[j] < kj;
          decided = true;
        }
      }
      cand = in && less;
    }
    unsigned cb = __ballot_sync(kFull, cand);
    while (cb) {
      const int src = __ffs(cb) - 1;
      cb &= cb - 1;
      uint32_t nwv[kMaxWords];
#pragma unroll
      for (int j = 0; j < kMaxWords; ++j) nwv[j] = __shfl_sync(kFull, w[j], src);
      // does it still beat the k-th best?  (position among the list: entries less than it)
      bool my_less = false, decided = false;  // is my entry < new?
#pragma unroll
      for (int j = 0; j < kMaxWords; ++j) {
        if (j < nw && !decided && mine[j] != nwv[j]) {
          my_less = mine[j] < nwv[j];
          decided = true;
        }
      }
      const unsigned lb = __ballot_sync(kFull, lane < cnt && my_less);
      const int pos = __popc(lb);  // list entries before the new one (they are a prefix)
      if (pos >= k) continue;  // not better than the k-th best any more
#pragma unroll
      for (int j = 0; j < kMaxWords; ++j) {
        const uint32_t up = __shfl_up_sync(kFull, mine[j], 1);
        if (lane > pos) mine[j] = up;
        else if (lane == pos) mine[j] = nwv[j];
      }
      cnt = min(cnt + 1, k);
    }
  }
  uint32_t mpos = 0;  // my entry's position word (the last word; selects, no dynamic index)
#pragma unroll
  for (int j = 0; j < kMaxWords; ++j) mpos = j == nw - 1 ? mine[j] : mpos;
  if (lane < k) out_pos[gw * k + lane] = lane < cnt ? (int32_t)mpos : -1;
}

// compact the warp lists' positions (drop -1 entries of short lists), keep order irrelevant
__global__ void k_topk_compact(const int32_t* __restrict__ in, int64_t m, int32_t* __restrict__ out,
                               unsigned long long* count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = in[i];
    if (v >= 0) out[atomicAdd(count, 1ull)] = v;
  }
}

// ---- radix select -------------------------------------------------------------------
struct SelState {
  unsigned long long k_rem;
  int chosen;  // digit chosen in the previous pass (-1: none / reject all)
  int pad;
};

__global__ void k_sel_hist(const __grid_constant__ Words W, int64_t n, uint8_t* state_flags, int pword, int pshift,
                           int cword, int cshift, const SelState* st, unsigned* hist, int first) {
  __shared__ unsigned h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  int chosen = st->chosen;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint8_t f = first ? 1 : state_flags[i];  // 1 active, 2 accepted, 0 rejected
    if (!first && f == 1) {
      int d = (W.w[pword][i] >> pshift) & 0xff;
      f = d < chosen ? 2 : (d == chosen ? 1 : 0);
      state_flags[i] = f;
    } else if (first) {
      state_flags[i] = 1;
    }
    if (f == 1 && cword >= 0) atomicAdd(&h[(W.w[cword][i] >> cshift) & 0xff], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

__global__ void __launch_bounds__(256) k_sel_choose(unsigned* hist, SelState* st) {
  // 256 threads, one per digit: the smallest digit whose inclusive count reaches k_rem (a
  // shared-memory scan; the serial walk over the histogram took 5-17 us per pass)
  __shared__ unsigned long long s[256];
  const int t = threadIdx.x;
  const unsigned long long krem = st->k_rem;
  const unsigned long long v = hist[t];
  s[t] = v;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const unsigned long long x = t >= o ? s[t - o] : 0ull;
    __syncthreads();
    s[t] += x;
    __syncthreads();
  }
  const unsigned long long incl = s[t], excl = incl - v;
  if (krem > 0 && incl >= krem && excl < krem) {
    st->chosen = t;
    st->k_rem = krem - excl;
  } else if (t == 255 && (krem == 0 || incl < krem)) {
    st->chosen = -1;
    st->k_rem = krem > incl ? krem - incl : 0;
  }
  hist[t] = 0;
}

struct AcceptedFn {
  const uint8_t* flags;
  template <int ITEMS>
  __device__ __forceinline__ void eval(const int32_t (&row)[ITEMS], const bool (&valid)[ITEMS], bool (&alive)[ITEMS],
                                       int32_t (&aux)[ITEMS]) const {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) alive[i] = valid[i] && flags[row[i]] != 0;
  }
};

// Lanes of the warp holding the same 8-bit digit as this lane (d in [0, 256) for valid lanes):
// eight ballots (bit slices) instead of __match_any_sync, which the join partition measured at
// 2.5x the cost of plain shared atomics on B200.
__device__ __forceinline__ unsigned digit_peers(int d, bool v) {
  unsigned peers = __ballot_sync(kFull, v);
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const bool bit = (d >> b) & 1;
    const unsigned bb = __ballot_sync(kFull, bit);
    peers &= bit ? bb : ~bb;
  }
  return peers;
}

template <int J, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (J < N) {
    f(std::integral_constant<int, J>{});
    static_for<J + 1, N>(f);
  }
}

// ---- LSD radix sort -----------------------------------------------------------------
// Per varying 8-bit digit (least significant first): K13a per-tile digit counts, a multi-block
// exclusive scan of the digit-major count matrix, K13b stable scatter.  A tile is kLsdThreads x
// ITEMS elements; warp w owns the contiguous sub-tile [w*32*ITEMS, (w+1)*32*ITEMS) in (item,
// lane) order, so a per-warp running digit counter (match_any leaders) gives every element its
// stable rank; the tile is then reordered in shared memory and written digit run by digit run
// (coalesced).  Sorting is stable, so the position word is carried, never sorted on.
constexpr int kLsdThreads = 256;
constexpr int kLsdWarps = kLsdThreads / 32;

template <int ITEMS>
__global__ void __launch_bounds__(kLsdThreads) k_lsd_count(const uint32_t* __restrict__ dw, int shift, int64_t n,
                                                           int32_t* counts /* [256][ntiles] */, int64_t ntiles) {
  __shared__ int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = blockIdx.x * (int64_t)(kLsdThreads * ITEMS);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t e = base + (int64_t)i * kLsdThreads + threadIdx.x;
    if (e < n) atomicAdd(&h[(__ldg(dw + e) >> shift) & 0xff], 1);
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

template <int ITEMS>
__global__ void __launch_bounds__(kLsdThreads) k_lsd_scatter(const __grid_constant__ Words src,
                                                             const __grid_constant__ Words dst, int dword, int shift,
                                                             int64_t n, const int64_t* __restrict__ offs,
                                                             int64_t ntiles) {
  constexpr int T = kLsdThreads * ITEMS;
  extern __shared__ uint32_t stage[];  // [nwords][T]
  __shared__ int wcnt[kLsdWarps][256];
  __shared__ int dstart[256];
  __shared__ int64_t s_off[256];  // this tile's global offset of each digit run
  __shared__ int s_warp[kLsdWarps];
  __shared__ uint8_t sdig[T];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = src.nwords;
  const int64_t base = blockIdx.x * (int64_t)T;
  for (int j = threadIdx.x; j < kLsdWarps * 256; j += kLsdThreads) (&wcnt[0][0])[j] = 0;
  __syncthreads();
  int dig[ITEMS], rank[ITEMS];
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t e = base + (int64_t)w * 32 * ITEMS + i * 32 + lane;
    const bool v = e < n;
    const int d = v ? (int)((__ldg(src.w[dword] + e) >> shift) & 0xff) : 0;
    const unsigned peers = digit_peers(d, v);
    const int leader = __ffs(peers) - 1;
    int r = 0;
    if (v) r = wcnt[w][d] + __popc(peers & lt);
    __syncwarp();
    if (v && lane == leader) wcnt[w][d] += __popc(peers);
    __syncwarp();
    dig[i] = v ? d : -1;
    rank[i] = r;
  }
  __syncthreads();
  // per digit: exclusive prefix over warps (in place), tile total -> tile-local digit starts
  {
    const int d = threadIdx.x;  // kLsdThreads == 256 digits
    int run = 0;
#pragma unroll
    for (int q = 0; q < kLsdWarps; ++q) {
      const int c = wcnt[q][d];
      wcnt[q][d] = run;
      run += c;
    }
    int x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    int wo = 0;
    for (int q = 0; q < w; ++q) wo += s_warp[q];
    dstart[d] = wo + x - run;
    s_off[d] = offs[(int64_t)d * ntiles + blockIdx.x];
  }
  __syncthreads();
  // reorder the tile in shared memory (all words), then write digit runs to their offsets
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (dig[i] < 0) continue;
    const int64_t e = base + (int64_t)w * 32 * ITEMS + i * 32 + lane;
    const int pos = dstart[dig[i]] + wcnt[w][dig[i]] + rank[i];
    sdig[pos] = (uint8_t)dig[i];
    for (int j = 0; j < nw; ++j) stage[j * T + pos] = __ldg(src.w[j] + e);
  }
  __syncthreads();
  const int tcount = (int)min((int64_t)T, n - base);
  for (int p = threadIdx.x; p < tcount; p += kLsdThreads) {
    const int d = sdig[p];
    const int64_t g = s_off[d] + (p - dstart[d]);
    for (int j = 0; j < nw; ++j) dst.w[j][g] = stage[j * T + p];
  }
}

// ---- onesweep LSD radix sort (K13o) ---------------------------------------------------
// One histogram pass over every varying digit up front (K13h), a 256-way exclusive scan per
// digit, then ONE kernel per digit pass (K13s): a CTA claims the next tile (atomic ticket, so
// every predecessor is already resident), ranks its rows exactly as k_lsd_scatter does, publishes
// its per-digit counts and resolves its per-digit global offsets by decoupled look-back over the
// predecessors' published counts (Merrill & Garland's chained scan, per digit), then scatters.
// No count pass and no separate scan per digit pass: each pass reads the words once and writes
// them once.  Status words are [63:32] tag | [31:0] count, tag = 2q+1 (aggregate) / 2q+2
// (inclusive prefix) for pass q, so one zero-fill serves every pass of a sort.
constexpr int kOsMaxDigits = 32;
struct OsHist {
  const uint32_t* w[kOsMaxDigits];
  int shift[kOsMaxDigits];
  int ndig;
  int64_t n;
  unsigned* hist;  // [ndig][256]
};

__global__ void __launch_bounds__(kLsdThreads) k_os_hist(const __grid_constant__ OsHist a) {
  extern __shared__ unsigned h[];  // [ndig][256]
  for (int i = threadIdx.x; i < a.ndig * 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t* pw = nullptr;
    uint32_t v = 0;
    for (int d = 0; d < a.ndig; ++d) {
      if (a.w[d] != pw) {
        pw = a.w[d];
        v = __ldcs(pw + i);
      }
      atomicAdd(&h[d * 256 + ((v >> a.shift[d]) & 0xff)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < a.ndig * 256; i += blockDim.x)
    if (h[i]) atomicAdd(&a.hist[i], h[i]);
}

// exclusive scan of each digit's 256 counts (one CTA per digit)
__global__ void __launch_bounds__(256) k_os_scan(unsigned* hist) {
  __shared__ unsigned s[256];
  unsigned* hd = hist + blockIdx.x * 256;
  const int t = threadIdx.x;
  const unsigned v = hd[t];
  s[t] = v;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const unsigned x = t >= o ? s[t - o] : 0u;
    __syncthreads();
    s[t] += x;
    __syncthreads();
  }
  hd[t] = s[t] - v;
}

// NW (words per row, the position word last) and ITEMS are compile-time: every word of every row
// is loaded into registers at the start of the tile (one round trip; ncu on the first version,
// which re-read the words from global memory after ranking: 52% long-scoreboard stalls, 1.4 TB/s),
// then each word is staged through shared memory in sorted order and written out.
template <int ITEMS, int NW, bool MATCH>
__global__ void __launch_bounds__(kLsdThreads, ITEMS * NW > 40 ? 2 : 3) k_onesweep(const __grid_constant__ Words src,
                                                          const __grid_constant__ Words dst, int dword, int shift,
                                                          int64_t n, const unsigned* __restrict__ dbase,
                                                          unsigned long long* status, unsigned* ticket, unsigned pass,
                                                          int pos_only) {
  constexpr int T = kLsdThreads * ITEMS;
  extern __shared__ uint32_t stage[];  // [T + 1] staged words (T: dump slot), then [T] destinations
  uint32_t* sdst = stage + T + 1;
  __shared__ int wcnt[kLsdWarps][256];
  __shared__ int hcnt[256];
  __shared__ int dstart[256];
  __shared__ int64_t s_off[256];
  __shared__ int s_warp[kLsdWarps];
  __shared__ unsigned s_tile;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  for (int j = threadIdx.x; j < kLsdWarps * 256; j += kLsdThreads) (&wcnt[0][0])[j] = 0;
  hcnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * (int64_t)T;
  const unsigned long long agg_tag = (unsigned long long)(2u * pass + 1u) << 32;
  const unsigned long long inc_tag = (unsigned long long)(2u * pass + 2u) << 32;
  // 1. every word of the tile's rows (the last pass needs only the digit and position words)
  // dr[i] = digit << 16 | rank (rank: within the warp, then within the tile); -1 past the end.
  // The digit word is picked with masks, not a select on `dword`, which the compiler turns into a
  // dynamic index of val[] and moves val[] to local memory.
  uint32_t val[NW][ITEMS];
  int dr[ITEMS];
  uint32_t dmask[NW];
#pragma unroll
  for (int j = 0; j < NW; ++j) dmask[j] = 0u - (uint32_t)(j == dword);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t e = base + (int64_t)w * 32 * ITEMS + i * 32 + lane;
    const bool in = e < n;
    uint32_t dw = 0;
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      val[j][i] = (in && (!pos_only || dmask[j] || j == NW - 1)) ? __ldcs(src.w[j] + e) : 0u;
      dw |= val[j][i] & dmask[j];
    }
    dr[i] = in ? (int)((dw >> shift) & 0xff) << 16 : -1;
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i)
    if (dr[i] >= 0) atomicAdd(&hcnt[dr[i] >> 16], 1);
  __syncthreads();
  // the tile's digit counts, published before the (longer) stable ranking
  const int tcnt = hcnt[threadIdx.x];
  st_relaxed(status + tile * 256 + threadIdx.x, (tile == 0 ? inc_tag : agg_tag) | (unsigned)tcnt);
  // 2. stable ranks: per-warp running digit counters over (item, lane) order
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const bool v = dr[i] >= 0;
    const int d = v ? dr[i] >> 16 : 0;
    const unsigned peers = MATCH ? (__match_any_sync(kFull, v ? d : 256 + lane)) : digit_peers(d, v);
    const int leader = __ffs(peers) - 1;
    int r = 0;
    if (v) r = wcnt[w][d] + __popc(peers & lt);
    __syncwarp();
    if (v && lane == leader) wcnt[w][d] += __popc(peers);
    __syncwarp();
    if (v) dr[i] |= r;
  }
  __syncthreads();
  {
    const int d = threadIdx.x;  // kLsdThreads == 256 digits
    int run = 0;
#pragma unroll
    for (int q = 0; q < kLsdWarps; ++q) {
      const int c = wcnt[q][d];
      wcnt[q][d] = run;
      run += c;
    }
    int x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    int wo = 0;
    for (int q = 0; q < w; ++q) wo += s_warp[q];
    dstart[d] = wo + x - run;
    // 3. look-back over the predecessors' counts of digit d (4 predecessors per round trip)
    int64_t excl = 0;
    if (tile > 0) {
      int64_t j = tile - 1;
      bool done = false;
      while (!done) {
        unsigned long long sw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) sw[q] = j - q >= 0 ? ld_relaxed(status + (j - q) * 256 + d) : inc_tag;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (!done) {
            while ((sw[q] >> 32) < (2u * pass + 1u)) sw[q] = ld_relaxed(status + (j - q) * 256 + d);
            if (j - q >= 0) excl += (uint32_t)sw[q];
            if ((sw[q] >> 32) == (2u * pass + 2u)) done = true;
          }
        }
        j -= 4;
      }
      st_relaxed(status + tile * 256 + d, inc_tag | (unsigned)(excl + run));
    }
    s_off[d] = (int64_t)dbase[d] + excl;
  }
  __syncthreads();
  // 4. sorted positions; then each word through shared memory to its digit run
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (dr[i] < 0) continue;
    const int d = dr[i] >> 16;
    dr[i] = (d << 16) | ((dr[i] & 0xffff) + dstart[d] + wcnt[w][d]);
  }
  const int tcount = (int)min((int64_t)T, n - base);
  // destination index of every sorted position, once (n <= INT32_MAX: 32 bits); sp[i]: the item's
  // shared slot, or the dump slot T past the end (no predicate in the per-word staging below)
  int sp[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    sp[i] = dr[i] >= 0 ? (dr[i] & 0xffff) : T;
    if (dr[i] < 0) continue;
    const int d = dr[i] >> 16, p = dr[i] & 0xffff;
    sdst[p] = (uint32_t)(s_off[d] + (p - dstart[d]));
  }
  static_for<0, NW>([&](auto jc) {  // compile-time word index: val stays in registers
    constexpr int j = decltype(jc)::value;
    if (pos_only && j != NW - 1) return;
    __syncthreads();  // (first word: sdst complete; later words: the previous word's reads done)
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) stage[sp[i]] = val[j][i];
    __syncthreads();
    uint32_t* out = dst.w[j];
    if (tcount == T) {
#pragma unroll 4
      for (int p = threadIdx.x; p < T; p += kLsdThreads) __stcs(out + sdst[p], stage[p]);
    } else {
      for (int p = threadIdx.x; p < tcount; p += kLsdThreads) __stcs(out + sdst[p], stage[p]);
    }
  });
}

template <int ITEMS, int NW>
sx_status onesweep_sort(sx_ctx* ctx, Scratch& scr, Words*& a, Words*& b, int nwords, int64_t n,
                        const std::vector<std::pair<int, int>>& digits) {
  // stable ranks from bit-sliced ballots (default; 30.4 vs 31.8 ms for the 2^28-key µbench with
  // __match_any_sync, SX_SORT_RANK=match)
  const bool ballot = !(getenv("SX_SORT_RANK") && std::strcmp(getenv("SX_SORT_RANK"), "match") == 0);
  if (nwords != NW) return set_err(ctx, SX_EINVAL, "onesweep: %d words", nwords);
  constexpr int T = kLsdThreads * ITEMS;
  const int64_t ntiles = (n + T - 1) / T;
  // sort digits, least significant first (the position word is carried, never sorted on)
  std::vector<std::pair<int, int>> pass;
  for (int p = (int)digits.size() - 1; p >= 0; --p)
    if (digits[p].first != nwords - 1) pass.push_back(digits[p]);
  const int np = (int)pass.size();
  if (np == 0) return SX_OK;
  if (np > kOsMaxDigits) return set_err(ctx, SX_EINVAL, "sort key has %d digits", np);
  unsigned* hist;
  unsigned long long* status;
  unsigned* tickets;
  SX_TRY(scr.get(&hist, (size_t)np * 256));
  SX_TRY(scr.get(&status, (size_t)ntiles * 256));
  SX_TRY(scr.get(&tickets, (size_t)np));
  SX_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned) * np * 256, ctx->stream));
  SX_CUDA(cudaMemsetAsync(status, 0, sizeof(unsigned long long) * ntiles * 256, ctx->stream));
  SX_CUDA(cudaMemsetAsync(tickets, 0, sizeof(unsigned) * np, ctx->stream));
  OsHist h{};
  for (int q = 0; q < np; ++q) {
    h.w[q] = a->w[pass[q].first];
    h.shift[q] = pass[q].second;
  }
  h.ndig = np;
  h.n = n;
  h.hist = hist;
  const size_t hsm = (size_t)np * 256 * sizeof(unsigned);
  k_os_hist<<<persistent_grid(ctx, 4, (n + kLsdThreads - 1) / kLsdThreads), kLsdThreads, hsm, SX_STREAM(ctx)>>>(h);
  SX_CHECK_LAUNCH();
  k_os_scan<<<np, 256, 0, SX_STREAM(ctx)>>>(hist);
  SX_CHECK_LAUNCH();
  const size_t smem = (size_t)(2 * T + 1) * sizeof(uint32_t);
  SX_CUDA(cudaFuncSetAttribute(k_onesweep<ITEMS, NW, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SX_CUDA(cudaFuncSetAttribute(k_onesweep<ITEMS, NW, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int q = 0; q < np; ++q) {
    const int pos_only = q == np - 1;  // the last pass only needs the positions in order
    if (ballot)
      k_onesweep<ITEMS, NW, false><<<(unsigned)ntiles, kLsdThreads, smem, SX_STREAM(ctx)>>>(
          *a, *b, pass[q].first, pass[q].second, n, hist + q * 256, status, tickets + q, (unsigned)q, pos_only);
    else
      k_onesweep<ITEMS, NW, true><<<(unsigned)ntiles, kLsdThreads, smem, SX_STREAM(ctx)>>>(
          *a, *b, pass[q].first, pass[q].second, n, hist + q * 256, status, tickets + q, (unsigned)q, pos_only);
    SX_CHECK_LAUNCH();
    std::swap(a, b);
  }
  return SX_OK;
}

template <int ITEMS>
sx_status lsd_sort(sx_ctx* ctx, Scratch& scr, Words*& a, Words*& b, int nwords, int64_t n,
                   const std::vector<std::pair<int, int>>& digits) {
  constexpr int T = kLsdThreads * ITEMS;
  const int64_t ntiles = (n + T - 1) / T;
  int32_t* counts;
  int64_t* offs;
  SX_TRY(scr.get(&counts, (size_t)(256 * ntiles)));
  SX_TRY(scr.get(&offs, (size_t)(256 * ntiles) + 1));
  const size_t smem = (size_t)nwords * T * sizeof(uint32_t);
  SX_CUDA(cudaFuncSetAttribute(k_lsd_scatter<ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int p = (int)digits.size() - 1; p >= 0; --p) {
    if (digits[p].first == nwords - 1) continue;  // position word: carried, not sorted on (stability)
    int64_t total = 0;
    k_lsd_count<ITEMS><<<(unsigned)ntiles, kLsdThreads, 0, SX_STREAM(ctx)>>>(a->w[digits[p].first], digits[p].second,
                                                                              n, counts, ntiles);
    SX_CHECK_LAUNCH();
    SX_TRY(scan_counts(ctx, counts, 256 * ntiles, offs, &total));
    k_lsd_scatter<ITEMS><<<(unsigned)ntiles, kLsdThreads, smem, SX_STREAM(ctx)>>>(*a, *b, digits[p].first,
                                                                                 digits[p].second, n, offs, ntiles);
    SX_CHECK_LAUNCH();
    std::swap(a, b);
  }
  return SX_OK;
}

}  // namespace

SX_EXPORT sx_status sx_sort_topk(sx_ctx* ctx, const sx_col* cols, int ncols, const sx_sortkey* keys, int nkeys,
                                 const sx_sel* in_sel, int64_t k, sx_sel* out_perm) {
  if (!ctx || !out_perm || (nkeys > 0 && !keys)) return SX_EINVAL;
  *out_perm = sx_sel{0, nullptr};
  ProfScope ps(ctx, "sort_topk");
  if (nkeys < 1 || nkeys > 4) return set_err(ctx, SX_EINVAL, "nkeys %d (1..4)", nkeys);
  EncArgs ea{};
  int nwords = 1;
  int64_t n = -1;
  for (int c = 0; c < nkeys; ++c) {
    int col = keys[c].col;
    if (col < 0 || col >= ncols) return set_err(ctx, SX_EINVAL, "sort key column out of range");
    const sx_col& sc = cols[col];
    if (sc.validity) return set_err(ctx, SX_EUNSUPPORTED, "validity bitmaps unsupported");
    int t = sc.type;
    int w = (t == SX_U8 || t == SX_I32 || t == SX_DATE32) ? 1 : (t == SX_I64 || t == SX_DEC64) ? 2 : t == SX_I128 ? 4 : 0;
    if (!w) return set_err(ctx, SX_ETYPE, "sort key type %d unsupported", t);
    nwords += w;
    ea.cols[c] = DCol{sc.data, t, 0};
    ea.types[c] = t;
    ea.desc[c] = keys[c].desc != 0;
    if (n < 0) n = sc.len;
  }
  if (nwords > kMaxWords) return set_err(ctx, SX_EINVAL, "sort key too wide (%d words)", nwords);
  if (in_sel) n = in_sel->len;
  if (n > INT32_MAX) return set_err(ctx, SX_EINDEX, "sort input exceeds INT32_MAX rows");
  int64_t outn = (k < 0 || k > n) ? n : k;
  if (ps.on()) {  // key columns (+ selection) read once, permutation written once
    double kw = 0;
    for (int c = 0; c < nkeys; ++c) kw += type_width(cols[keys[c].col].type);
    ps.set_bytes((kw + (in_sel ? 4.0 : 0.0)) * n + 4.0 * outn);
  }
  Scratch scr(ctx);
  int32_t* perm;
  SX_TRY(scr.get(&perm, (size_t)(outn > 0 ? outn : 1)));
  if (outn == 0) {
    out_perm->idx = perm;
    scr.release(perm);
    return SX_OK;
  }
  ea.nkeys = nkeys;
  ea.nwords = nwords;
  ea.sel = in_sel ? in_sel->idx : nullptr;
  ea.n = n;
  Words W{};
  W.nwords = nwords;
  for (int j = 0; j < nwords; ++j) {
    SX_TRY(scr.get(&ea.words[j], (size_t)n));
    W.w[j] = ea.words[j];
  }
  unsigned* diff;
  SX_TRY(scr.get(&diff, kMaxWords));
  SX_CUDA(cudaMemsetAsync(diff, 0, kMaxWords * sizeof(unsigned), ctx->stream));
  ea.diff = diff;
  k_encode<<<persistent_grid(ctx, 8, (n + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(ea);
  SX_CHECK_LAUNCH();
  const int32_t* sel = in_sel ? in_sel->idx : nullptr;
  // one-CTA bitonic sort for small inputs (measured: 8192 rows x 5 words in one CTA, 0.48 ms, loses
  // to the radix select's 0.27 ms at Q18's top-100)
  if (n <= kBitonicMax) {
    size_t smem = (size_t)kBitonicMax * nwords * sizeof(uint32_t);
    SX_CUDA(cudaFuncSetAttribute(k_bitonic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_bitonic<<<1, 1024, smem, SX_STREAM(ctx)>>>(W, nullptr, n, outn, sel, perm);
    SX_CHECK_LAUNCH();
    out_perm->len = outn;
    out_perm->idx = perm;
    scr.release(perm);
    return SX_OK;
  }
  // top-k (k <= 1024) of up to 32 chunks by tournament rounds of per-chunk shared-memory sorts
  // (Q18: 0.18 vs 0.27 ms); larger inputs take the radix select below, whose passes stream the
  // key words (Q3's 1.1e6 rows x 7 words: 0.35 ms vs 2.0 ms for 552 chunk sorts).
  // SX_TOPK=select / =tournament force either path.
  const char* topk_env = getenv("SX_TOPK");
  // K14w for k <= 32 (opt-in, SX_TOPK=warp): measured slower than the radix select on Q3's
  // top-10 of 1.13e6 rows (0.40 / 0.37 vs 0.28 ms: the serial per-warp insertions and the rounds)
  const bool topk_warp = outn <= 32 && outn < n && topk_env && std::strcmp(topk_env, "warp") == 0;
  const int32_t* warp_pos = nullptr;
  int64_t warp_m = 0;
  if (topk_warp) {
    // ~4096 rows per warp (>= k, so the lists fill): few enough warps that their k-lists fit one
    // or two tournament rounds (3.5e3 warps of 320 rows for Q3 left 35e3 candidates: 0.37 ms)
    int64_t warps = std::min<int64_t>((int64_t)ctx->num_sms * 8, std::max<int64_t>(1, n / 4096));
    if (n / warps < 32 * outn) warps = std::max<int64_t>(1, n / (32 * outn));
    const int64_t per = (n + warps - 1) / warps;
    warps = (n + per - 1) / per;
    int32_t *lists, *cpos;
    SX_TRY(scr.get(&lists, (size_t)(warps * outn)));
    SX_TRY(scr.get(&cpos, (size_t)(warps * outn)));
    k_topk_warp<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, SX_STREAM(ctx)>>>(W, n, (int)outn, per, lists);
    SX_CHECK_LAUNCH();
    unsigned long long* cntp = (unsigned long long*)ctx->d_counters;
    SX_CUDA(cudaMemsetAsync(cntp, 0, 8, ctx->stream));
    k_topk_compact<<<persistent_grid(ctx, 4, (warps * outn + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
        lists, warps * outn, cpos, cntp);
    SX_CHECK_LAUNCH();
    SX_TRY(read_i64(ctx, cntp, &warp_m));
    warp_pos = cpos;
  }
  const bool topk_tour = topk_warp || (topk_env ? std::strcmp(topk_env, "tournament") == 0 : n <= 32 * (int64_t)kBitonicMax);
  if (topk_tour && outn <= 1024 && outn < n) {
    const size_t smem = (size_t)kBitonicMax * nwords * sizeof(uint32_t);
    SX_CUDA(cudaFuncSetAttribute(k_topk_round, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SX_CUDA(cudaFuncSetAttribute(k_bitonic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int32_t *pa = nullptr, *pb = nullptr;
    const int64_t c1 = (n + kBitonicMax - 1) / kBitonicMax;
    SX_TRY(scr.get(&pa, (size_t)(c1 * outn)));
    SX_TRY(scr.get(&pb, (size_t)(c1 * outn)));
    const int32_t* cur = warp_pos;  // nullptr: rows 0..m-1 (K14w: its candidate positions)
    int64_t m = warp_pos ? warp_m : n;
    int32_t* dst = pa;
    while (m > kBitonicMax) {
      const int64_t chunks = (m + kBitonicMax - 1) / kBitonicMax;
      k_topk_round<<<(unsigned)chunks, 1024, smem, SX_STREAM(ctx)>>>(W, cur, m, outn, dst);
      SX_CHECK_LAUNCH();
      const int64_t last = m - (chunks - 1) * kBitonicMax;
      m = (chunks - 1) * outn + std::min<int64_t>(outn, last);
      cur = dst;
      dst = dst == pa ? pb : pa;
    }
    k_bitonic<<<1, 1024, smem, SX_STREAM(ctx)>>>(W, cur, m, outn, sel, perm);
    SX_CHECK_LAUNCH();
    out_perm->len = outn;
    out_perm->idx = perm;
    scr.release(perm);
    return SX_OK;
  }
  unsigned hdiff[kMaxWords];
  SX_CUDA(cudaMemcpyAsync(hdiff, diff, sizeof(unsigned) * kMaxWords, cudaMemcpyDeviceToHost, ctx->stream));
  SX_CUDA(cudaStreamSynchronize(ctx->stream));
  // varying digits, most significant first: (word, shift)
  std::vector<std::pair<int, int>> digits;
  for (int j = 0; j < nwords; ++j)
    for (int s = 24; s >= 0; s -= 8)
      if ((hdiff[j] >> s) & 0xff) digits.push_back({j, s});
  if (outn <= 1024 && outn < n) {
    // radix select of the outn-th smallest composite key
    uint8_t* flags;
    unsigned* hist;
    SelState* st;
    SX_TRY(scr.get(&flags, (size_t)n));
    SX_TRY(scr.get(&hist, 256));
    SX_TRY(scr.get(&st, 1));
    SelState h0{(unsigned long long)outn, -1, 0};
    SX_CUDA(cudaMemcpyAsync(st, &h0, sizeof(h0), cudaMemcpyHostToDevice, ctx->stream));
    SX_CUDA(cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned), ctx->stream));
    unsigned grid = persistent_grid(ctx, 8, (n + kBlock - 1) / kBlock);
    int pw = -1, psh = 0;
    for (size_t p = 0; p <= digits.size(); ++p) {
      int cw = p < digits.size() ? digits[p].first : -1;
      int csh = p < digits.size() ? digits[p].second : 0;
      k_sel_hist<<<grid, kBlock, 0, SX_STREAM(ctx)>>>(W, n, flags, pw, psh, cw, csh, st, hist, p == 0);
      SX_CHECK_LAUNCH();
      if (cw >= 0) {
        k_sel_choose<<<1, 256, 0, SX_STREAM(ctx)>>>(hist, st);
        SX_CHECK_LAUNCH();
      }
      pw = cw;
      psh = csh;
    }
    // all digits decided: the remaining active rows equal the k-th key exactly (unique keys) -> accepted
    int32_t* winners = nullptr;
    AcceptedFn af{flags};
    GatherSpec none;
    none.n = 0;
    int64_t m = 0;
    SX_TRY(run_compact(ctx, af, n, nullptr, &winners, nullptr, none, &m));
    scr.ptrs.push_back(winners);
    if (m != outn) return set_err(ctx, SX_ECUDA, "radix select produced %lld of %lld rows", (long long)m, (long long)outn);
    size_t smem = (size_t)kBitonicMax * nwords * sizeof(uint32_t);
    SX_CUDA(cudaFuncSetAttribute(k_bitonic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_bitonic<<<1, 1024, smem, SX_STREAM(ctx)>>>(W, winners, m, outn, sel, perm);
    SX_CHECK_LAUNCH();
  } else {
    // LSD radix sort over the varying key digits, least significant first
    Words W2{};
    W2.nwords = nwords;
    for (int j = 0; j < nwords; ++j) SX_TRY(scr.get(&W2.w[j], (size_t)n));
    Words* a = &W;
    Words* b = &W2;
    // onesweep (default) or the count + scan + scatter LSD passes (SX_SORT=lsd, kept for A/B)
    const bool lsd = getenv("SX_SORT") && std::strcmp(getenv("SX_SORT"), "lsd") == 0;
    if (lsd) {
      if (nwords <= 3) SX_TRY(lsd_sort<16>(ctx, scr, a, b, nwords, n, digits));
      else if (nwords <= 6) SX_TRY(lsd_sort<8>(ctx, scr, a, b, nwords, n, digits));
      else SX_TRY(lsd_sort<4>(ctx, scr, a, b, nwords, n, digits));
    } else {
      switch (nwords) {  // registers: ITEMS x NW words per thread
        case 2: SX_TRY((onesweep_sort<16, 2>(ctx, scr, a, b, nwords, n, digits))); break;
        case 3: SX_TRY((onesweep_sort<16, 3>(ctx, scr, a, b, nwords, n, digits))); break;
        case 4: SX_TRY((onesweep_sort<12, 4>(ctx, scr, a, b, nwords, n, digits))); break;
        case 5: SX_TRY((onesweep_sort<8, 5>(ctx, scr, a, b, nwords, n, digits))); break;
        case 6: SX_TRY((onesweep_sort<8, 6>(ctx, scr, a, b, nwords, n, digits))); break;
        case 7: SX_TRY((onesweep_sort<6, 7>(ctx, scr, a, b, nwords, n, digits))); break;
        case 8: SX_TRY((onesweep_sort<6, 8>(ctx, scr, a, b, nwords, n, digits))); break;
        default: SX_TRY((onesweep_sort<5, 9>(ctx, scr, a, b, nwords, n, digits))); break;
      }
    }
    // positions (last word) of the first outn sorted rows -> row ids
    GatherSpec none;
    none.n = 0;
    (void)none;
    sx_sel possel{outn, (int32_t*)a->w[nwords - 1]};
    if (sel) {
      sx_col selcol{SX_I32, 0, n, sel, nullptr, nullptr};
      sx_col g;
      SX_TRY(sx_gather(ctx, &selcol, &possel, &g));
      SX_CUDA(cudaMemcpyAsync(perm, g.data, outn * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
      dfree(ctx, (void*)g.data);
    } else {
      SX_CUDA(cudaMemcpyAsync(perm, a->w[nwords - 1], outn * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    }
  }
  out_perm->len = outn;
  out_perm->idx = perm;
  scr.release(perm);
  return SX_OK;
}
