// compact.cuh — ordered stream compaction skeleton (K2) + dense materialization (K3).
//
// Three barrier-light phases (a single-pass decoupled look-back serialised small tiles on the
// look-back chain: ncu showed 60%+ of warp stalls at the tile barrier waiting for it):
//   1. k_compact_local: every CTA takes tiles of kBlock*ITEMS input positions (grid-stride),
//      evaluates the row functor for all of a thread's rows at once, ranks the survivors with
//      warp ballots + popc and a per-tile scan of (item, warp) cells, and writes them compacted
//      into a per-tile scratch region (row id, aux) plus the tile's count;
//   2. scan of the tile counts (3 tiny kernels);
//   3. k_compact_scatter: copies each tile's survivors to its final offset (coalesced), giving
//      ascending row ids; payload columns are then gathered densely (k_gather_multi).
// Inputs are read once; scratch traffic is 8 bytes per survivor each way.
//
// Functor interface:
//   template <int ITEMS> __device__ void eval(const int32_t (&row)[ITEMS], const bool (&valid)[ITEMS],
//                                            bool (&alive)[ITEMS], int32_t (&aux)[ITEMS]) const;
#pragma once
#include "common.cuh"

namespace sx {

template <class F, bool HAS_SEL, int ITEMS>
__global__ void __launch_bounds__(kBlock, 4) k_compact_local(const __grid_constant__ F f, int64_t n,
                                                          const int32_t* __restrict__ in_sel,
                                                          int32_t* __restrict__ s_row, int32_t* __restrict__ s_aux,
                                                          int32_t* __restrict__ tile_cnt, int64_t ntiles) {
  constexpr int W = kBlock / 32;
  constexpr int NE = ITEMS * W;  // (item, warp) cells, scanned in that order
  static_assert(NE <= 64, "scan assumes <= 2 cells per lane");
  __shared__ int s_cnt[NE];
  __shared__ int s_total;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * (int64_t)(kBlock * ITEMS);
    int32_t row[ITEMS];
    bool valid[ITEMS], alive[ITEMS];
    int32_t aux[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      int64_t idx = base + (int64_t)i * kBlock + threadIdx.x;
      valid[i] = idx < n;
      row[i] = (int32_t)idx;
      aux[i] = -1;
    }
    if (HAS_SEL) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) row[i] = valid[i] ? __ldg(in_sel + row[i]) : 0;
    }
    f.template eval<ITEMS>(row, valid, alive, aux);
    unsigned ball[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      ball[i] = __ballot_sync(kFull, valid[i] && alive[i]);
      if (lane == 0) s_cnt[i * W + w] = __popc(ball[i]);
    }
    __syncthreads();
    if (w == 0) {
      // cells c = item*W + warp in scan order; lane holds cells lane and lane+32
      int a = lane < NE ? s_cnt[lane] : 0;
      int b = lane + 32 < NE ? s_cnt[lane + 32] : 0;
      int pa = a, pb = b;
      for (int o = 1; o < 32; o <<= 1) {
        int ya = __shfl_up_sync(kFull, pa, o);
        int yb = __shfl_up_sync(kFull, pb, o);
        if (lane >= o) { pa += ya; pb += yb; }
      }
      int half = __shfl_sync(kFull, pa, 31);
      if (lane < NE) s_cnt[lane] = pa - a;
      if (lane + 32 < NE) s_cnt[lane + 32] = half + pb - b;
      if (lane == 31) s_total = half + pb;
    }
    __syncthreads();
    const unsigned lt = lanemask_lt();
    int32_t* tr = s_row + base;
    int32_t* ta = s_aux ? s_aux + base : nullptr;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if ((ball[i] >> lane) & 1u) {
        int pos = s_cnt[i * W + w] + __popc(ball[i] & lt);
        tr[pos] = row[i];
        if (ta) ta[pos] = aux[i];
      }
    }
    if (threadIdx.x == 0) tile_cnt[tile] = s_total;
    __syncthreads();
  }
}

// Dense variant of phase 1 (no input selection; functors with eval_dense): thread t of a tile owns
// ITEMS consecutive rows, which the functor reads with 128-bit vector loads and returns as a bit
// mask; survivors are ranked by a block scan of the per-thread counts and written (ascending) to
// the tile's scratch region.  Same scratch layout and phases 2-3 as k_compact_local.
// functors whose eval_dense is warp-cooperative: called by every lane, also past the end
template <class F, class = void>
struct warp_coop { static constexpr bool value = false; };
template <class F>
struct warp_coop<F, std::void_t<decltype(F::kWarpCoop)>> { static constexpr bool value = F::kWarpCoop; };

template <class F, class = void>
struct dense_blocks { static constexpr int value = 3; };
template <class F>
struct dense_blocks<F, std::void_t<decltype(F::kMinBlocks)>> { static constexpr int value = F::kMinBlocks; };

template <class F, int ITEMS>
__global__ void __launch_bounds__(kBlock, dense_blocks<F>::value) k_compact_dense(const __grid_constant__ F f, int64_t n,
                                                          int32_t* __restrict__ s_row, int32_t* __restrict__ s_aux,
                                                          int32_t* __restrict__ tile_cnt, int64_t ntiles) {
  constexpr int W = kBlock / 32;
  __shared__ int s_w[W];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * (int64_t)(kBlock * ITEMS);
    const int64_t r0 = base + (int64_t)threadIdx.x * ITEMS;
    uint32_t mask = 0;
    int32_t aux[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) aux[i] = -1;
    if (warp_coop<F>::value || r0 < n) f.template eval_dense<ITEMS>(r0, n, mask, aux);
    const int c = __popc(mask);
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    int wo = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const int v = s_w[q];
      wo += q < w ? v : 0;
      tot += v;
    }
    int pos = wo + x - c;
    int32_t* tr = s_row + base;
    int32_t* ta = s_aux ? s_aux + base : nullptr;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if ((mask >> i) & 1u) {
        tr[pos] = (int32_t)(r0 + i);
        if (ta) ta[pos] = aux[i];
        ++pos;
      }
    }
    if (threadIdx.x == 0) tile_cnt[tile] = tot;
    __syncthreads();
  }
}

template <class F, class = void>
struct dense_items { static constexpr int value = 0; };
template <class F>
struct dense_items<F, std::void_t<decltype(F::kDenseItems)>> { static constexpr int value = F::kDenseItems; };

// exclusive scan of int32 tile counts into int64 offsets (offsets[ntiles] = total)
static __global__ void __launch_bounds__(1024) k_scan_counts_local(const int32_t* __restrict__ cnt, int64_t n,
                                                                   int64_t* __restrict__ off,
                                                                   int64_t* __restrict__ block_sums) {
  __shared__ int64_t wsum[32];
  int64_t i = blockIdx.x * 1024ll + threadIdx.x;
  int64_t v = i < n ? cnt[i] : 0;
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t t = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(kFull, t, o);
      if (lane >= o) t += y;
    }
    wsum[lane] = t;
  }
  __syncthreads();
  int64_t incl = x + (w ? wsum[w - 1] : 0);
  if (i < n) off[i] = incl - v;
  if (threadIdx.x == 1023) block_sums[blockIdx.x] = incl;
}

static __global__ void k_scan_counts_sums(int64_t* __restrict__ sums, int64_t nb, int64_t* __restrict__ total) {
  // one warp: sequential chunks of 32 (nb is ntiles / 1024, small)
  const int lane = threadIdx.x;
  int64_t run = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += 32) {
    int64_t v = b0 + lane < nb ? sums[b0 + lane] : 0, x = v;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (b0 + lane < nb) sums[b0 + lane] = run + x - v;
    run += __shfl_sync(kFull, x, 31);
  }
  if (lane == 0) *total = run;
}

static __global__ void k_scan_counts_add(int64_t* __restrict__ off, int64_t n, const int64_t* __restrict__ sums) {
  int64_t i = blockIdx.x * 1024ll + threadIdx.x;
  if (i < n) off[i] += sums[blockIdx.x];
}

template <int TILE>
__global__ void __launch_bounds__(kBlock) k_compact_scatter(const int32_t* __restrict__ s_row,
                                                            const int32_t* __restrict__ s_aux,
                                                            const int32_t* __restrict__ tile_cnt,
                                                            const int64_t* __restrict__ tile_off, int64_t ntiles,
                                                            int32_t* __restrict__ out_sel, int32_t* __restrict__ out_aux) {
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int c = tile_cnt[tile];
    if (c == 0) continue;
    const int64_t o = tile_off[tile], base = tile * (int64_t)TILE;
    for (int j = threadIdx.x; j < c; j += blockDim.x) {
      out_sel[o + j] = __ldg(s_row + base + j);
      if (out_aux) out_aux[o + j] = __ldg(s_aux + base + j);
    }
  }
}

// Dense materialisation: out column g [i] = src[sel[i]] (or src[aux[i]] for build-side payload).
static __global__ void __launch_bounds__(kBlock) k_gather_multi(const int32_t* __restrict__ sel,
                                                               const int32_t* __restrict__ aux, int64_t n,
                                                               const __grid_constant__ GatherSpec gs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = __ldg(sel + i), a = aux ? (int64_t)__ldg(aux + i) : 0;
    for (int g = 0; g < gs.n; ++g) gather_one(gs.g[g], i, gs.g[g].by_aux ? a : r);
  }
}

// Exclusive scan of n int32 counts into off[0..n] (off[n] = total, read back into *total).
inline sx_status scan_counts(sx_ctx* ctx, const int32_t* cnt, int64_t n, int64_t* off, int64_t* total) {
  Scratch scr(ctx);
  const int64_t nb = (n + 1023) / 1024;
  int64_t* bsum;
  SX_TRY(scr.get(&bsum, (size_t)nb + 1));
  if (n > 0) {
    k_scan_counts_local<<<(unsigned)nb, 1024, 0, SX_STREAM(ctx)>>>(cnt, n, off, bsum);
    k_scan_counts_sums<<<1, 32, 0, SX_STREAM(ctx)>>>(bsum, nb, off + n);
    k_scan_counts_add<<<(unsigned)nb, 1024, 0, SX_STREAM(ctx)>>>(off, n, bsum);
    SX_CHECK_LAUNCH();
    SX_TRY(read_i64(ctx, off + n, total));
  } else {
    *total = 0;
  }
  return SX_OK;
}

// Host driver: runs the skeleton over n positions; returns the output count (one D2H read).
// Outputs are allocated here at the exact count (known after the scan): *out_sel always,
// *out_aux when out_aux != nullptr, and every gs.g[g].dst that is nullptr (count * width bytes).
// Ownership of all of them passes to the caller (also on error paths they are freed here).
template <class F, int ITEMS, bool DENSE, class AllocFn>
sx_status run_compact_tiles(sx_ctx* ctx, const F& f, int64_t n, const int32_t* in_sel, int32_t** out_sel,
                            int32_t** out_aux, GatherSpec& gs, int64_t* out_count, const bool* owned,
                            AllocFn& alloc_outputs);

template <class F, int ITEMS = 8>
sx_status run_compact(sx_ctx* ctx, const F& f, int64_t n, const int32_t* in_sel, int32_t** out_sel,
                      int32_t** out_aux, GatherSpec& gs, int64_t* out_count) {
  *out_count = 0;
  *out_sel = nullptr;
  if (out_aux) *out_aux = nullptr;
  bool owned[kMaxGather] = {};
  for (int g = 0; g < gs.n; ++g) owned[g] = gs.g[g].dst == nullptr;
  auto alloc_outputs = [&](int64_t cnt) -> sx_status {
    size_t c = (size_t)(cnt > 0 ? cnt : 1);
    SX_TRY(alloc(ctx, out_sel, c));
    if (out_aux) {
      sx_status s = alloc(ctx, out_aux, c);
      if (s != SX_OK) { dfree(ctx, *out_sel); *out_sel = nullptr; return s; }
    }
    for (int g = 0; g < gs.n; ++g) {
      if (!owned[g]) continue;
      sx_status s = alloc(ctx, (char**)&gs.g[g].dst, c * gs.g[g].width);
      if (s != SX_OK) {
        for (int h = 0; h < g; ++h) if (owned[h]) { dfree(ctx, gs.g[h].dst); gs.g[h].dst = nullptr; }
        dfree(ctx, *out_sel); *out_sel = nullptr;
        if (out_aux) { dfree(ctx, *out_aux); *out_aux = nullptr; }
        return s;
      }
    }
    return SX_OK;
  };
  if (n == 0) return alloc_outputs(0);
  constexpr int DI = dense_items<F>::value;
  if constexpr (DI > 0) {
    if (!in_sel) return run_compact_tiles<F, DI, true>(ctx, f, n, in_sel, out_sel, out_aux, gs, out_count, owned,
                                                       alloc_outputs);
  }
  return run_compact_tiles<F, ITEMS, false>(ctx, f, n, in_sel, out_sel, out_aux, gs, out_count, owned, alloc_outputs);
}

template <class F, int ITEMS, bool DENSE, class AllocFn>
sx_status run_compact_tiles(sx_ctx* ctx, const F& f, int64_t n, const int32_t* in_sel, int32_t** out_sel,
                            int32_t** out_aux, GatherSpec& gs, int64_t* out_count, const bool* owned,
                            AllocFn& alloc_outputs) {
  constexpr int TILE = kBlock * ITEMS;
  const int64_t ntiles = (n + TILE - 1) / TILE;
  Scratch scr(ctx);
  int32_t *s_row, *s_aux = nullptr, *cnt;
  int64_t *off, *bsum;
  SX_TRY(scr.get(&s_row, (size_t)ntiles * TILE));
  if (out_aux) SX_TRY(scr.get(&s_aux, (size_t)ntiles * TILE));
  SX_TRY(scr.get(&cnt, (size_t)ntiles));
  SX_TRY(scr.get(&off, (size_t)ntiles + 1));
  const int64_t nb = (ntiles + 1023) / 1024;
  SX_TRY(scr.get(&bsum, (size_t)nb + 1));
  unsigned grid = persistent_grid(ctx, 8, ntiles);
  if constexpr (DENSE)
    k_compact_dense<F, ITEMS><<<grid, kBlock, 0, SX_STREAM(ctx)>>>(f, n, s_row, s_aux, cnt, ntiles);
  else if (in_sel)
    k_compact_local<F, true, ITEMS><<<grid, kBlock, 0, SX_STREAM(ctx)>>>(f, n, in_sel, s_row, s_aux, cnt, ntiles);
  else
    k_compact_local<F, false, ITEMS><<<grid, kBlock, 0, SX_STREAM(ctx)>>>(f, n, in_sel, s_row, s_aux, cnt, ntiles);
  SX_CHECK_LAUNCH();
  k_scan_counts_local<<<(unsigned)nb, 1024, 0, SX_STREAM(ctx)>>>(cnt, ntiles, off, bsum);
  k_scan_counts_sums<<<1, 32, 0, SX_STREAM(ctx)>>>(bsum, nb, off + ntiles);
  k_scan_counts_add<<<(unsigned)nb, 1024, 0, SX_STREAM(ctx)>>>(off, ntiles, bsum);
  SX_CHECK_LAUNCH();
  int64_t count = 0;
  SX_TRY(read_i64(ctx, off + ntiles, &count));
  SX_TRY(alloc_outputs(count));
  *out_count = count;
  if (count > 0) {
    k_compact_scatter<TILE><<<persistent_grid(ctx, 8, ntiles), kBlock, 0, SX_STREAM(ctx)>>>(
        s_row, s_aux, cnt, off, ntiles, *out_sel, out_aux ? *out_aux : nullptr);
    if (gs.n > 0)
      k_gather_multi<<<persistent_grid(ctx, 8, (count + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
          *out_sel, out_aux ? *out_aux : nullptr, count, gs);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      dfree(ctx, *out_sel);
      *out_sel = nullptr;
      if (out_aux) { dfree(ctx, *out_aux); *out_aux = nullptr; }
      for (int g = 0; g < gs.n; ++g) if (owned[g]) { dfree(ctx, gs.g[g].dst); gs.g[g].dst = nullptr; }
      return set_err(ctx, SX_ECUDA, "compaction scatter: %s", cudaGetErrorString(e));
    }
  }
  return SX_OK;
}

}  // namespace sx
