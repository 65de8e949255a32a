// compact.cuh — ordered stream compaction skeleton (K2) with fused materialization (K3).
//
// One persistent pass: each CTA takes tiles of kBlock*ITEMS input positions
// (virtual tile ids from an atomic counter => forward progress for the
// look-back), evaluates a row functor for every position, ranks the survivors
// with warp ballots + popc and a per-tile scan, obtains the tile's global
// offset by decoupled look-back, and writes ascending row ids (+ an aux id and
// gathered payload columns) at their final positions.  Inputs are read once;
// outputs are written once.
//
// Functor interface:
//   template <int ITEMS> __device__ void eval(const int32_t (&row)[ITEMS], const bool (&valid)[ITEMS],
//                                            bool (&alive)[ITEMS], int32_t (&aux)[ITEMS]) const;
// The functor sees all of a thread's rows at once so it can issue their loads
// back to back (memory-level parallelism), then evaluate.
#pragma once
#include "common.cuh"

namespace sx {

template <class F, bool HAS_SEL, int ITEMS>
__global__ void __launch_bounds__(kBlock) k_compact(const __grid_constant__ F f, int64_t n, const int32_t* __restrict__ in_sel,
                                                    int32_t* __restrict__ out_sel, int32_t* __restrict__ out_aux,
                                                    const __grid_constant__ GatherSpec gs, unsigned long long* status,
                                                    unsigned int* tile_ctr, int64_t ntiles) {
  constexpr int W = kBlock / 32;
  constexpr int NE = ITEMS * W;  // (item, warp) cells, scanned in that order
  static_assert(NE <= 64, "scan assumes <= 2 cells per lane");
  __shared__ int64_t s_tile;
  __shared__ int64_t s_excl;
  __shared__ int s_cnt[NE];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  while (true) {
    if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= ntiles) break;
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
      int total = half + __shfl_sync(kFull, pb, 31);
      if (lane < NE) s_cnt[lane] = pa - a;
      if (lane + 32 < NE) s_cnt[lane + 32] = half + pb - b;
      int64_t excl = lookback_exclusive(status, tile, total);
      if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    const int64_t excl = s_excl;
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if ((ball[i] >> lane) & 1u) {
        int64_t pos = excl + s_cnt[i * W + w] + __popc(ball[i] & lt);
        out_sel[pos] = (int32_t)row[i];
        if (out_aux) out_aux[pos] = aux[i];
        for (int g = 0; g < gs.n; ++g) gather_one(gs.g[g], pos, gs.g[g].by_aux ? (int64_t)aux[i] : row[i]);
      }
    }
    __syncthreads();
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

// Host driver: runs the skeleton over n positions; returns the output count (one D2H read).
// out_sel / out_aux / gather destinations must have capacity >= n.
template <class F, int ITEMS = 8>
sx_status run_compact(sx_ctx* ctx, const F& f, int64_t n, const int32_t* in_sel, int32_t* out_sel, int32_t* out_aux,
                      const GatherSpec& gs, int64_t* out_count) {
  *out_count = 0;
  if (n == 0) return SX_OK;
  const int64_t tile_rows = (int64_t)kBlock * ITEMS;
  const int64_t ntiles = (n + tile_rows - 1) / tile_rows;
  Scratch scr(ctx);
  unsigned long long* status;
  SX_TRY(scr.get(&status, (size_t)ntiles));
  SX_CUDA(cudaMemsetAsync(status, 0, sizeof(unsigned long long) * ntiles, ctx->stream));
  unsigned int* ctr = ctx->d_counters;
  SX_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned int), ctx->stream));
  unsigned grid = persistent_grid(ctx, 8, ntiles);
  // Payload columns are gathered in a dense post-pass (one thread per output row) rather than
  // inside the scan, where only the (few) surviving lanes of each warp would be active.
  GatherSpec none;
  none.n = 0;
  if (in_sel)
    k_compact<F, true, ITEMS><<<grid, kBlock, 0, SX_STREAM(ctx)>>>(f, n, in_sel, out_sel, out_aux, none, status, ctr, ntiles);
  else
    k_compact<F, false, ITEMS><<<grid, kBlock, 0, SX_STREAM(ctx)>>>(f, n, in_sel, out_sel, out_aux, none, status, ctr, ntiles);
  SX_CHECK_LAUNCH();
  int64_t last;
  SX_TRY(read_i64(ctx, status + (ntiles - 1), &last));
  *out_count = (int64_t)((unsigned long long)last & ((1ull << 62) - 1));
  if (gs.n > 0 && *out_count > 0) {
    k_gather_multi<<<persistent_grid(ctx, 8, (*out_count + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
        out_sel, out_aux, *out_count, gs);
    SX_CHECK_LAUNCH();
  }
  return SX_OK;
}

}  // namespace sx
