// ring.cuh — K9r: warp-specialised streaming aggregation over a shared-memory tile ring.
//
// One producer warp moves whole tiles of every referenced column into a kStages-deep ring in
// shared memory with cp.async.bulk (the TMA engine's 1-D bulk copies, SASS UBLKCP); completion
// is signalled on a per-stage "full" mbarrier (expect_tx byte count).  kConsumers warps compute
// from shared memory and release a stage on its "empty" mbarrier (one arrival per consumer
// warp).  The bytes in flight per SM are bounded by the ring, not by the register file, so a
// register-heavy consumer (Q1's exact decimal accumulators) no longer limits the memory-level
// parallelism — the reason K9d stalled at 0.80 of the HBM peak (round 1: 124 registers, 2
// CTAs/SM, 24% warps active, the hottest stall the first use of each loaded byte).
//
// Each CTA streams a contiguous chunk of whole tiles (one CTA per SM); the rows after the last
// whole tile go through the program's global-load tail path in the last CTA.  Program interface
// (see Q1Prog in tpch.cu):
//   kRingCols, kRingTile (rows per stage), kRingStages, kRingConsumers, ring_width(c), ring_col(c)
//   kRingExtraBytes (dynamic shared memory after the ring, e.g. lane-private accumulators)
//   struct RingAcc (per-thread registers), struct RingShared (per-CTA merge state)
//   ring_shared_init(sh, x, tid, nthreads)          before the first barrier (x = extra smem)
//   ring_consume(b[], row0, cw, lane, acc, sh, x)   one stage: cw-th slice of the tile
//   ring_tail(r0, n, cw, lane, acc, sh, x)          rows [r0, n) (< one tile), global loads
//   ring_flush(acc, cw, lane, sh, x)                warp-collective: per-thread -> CTA state
//   ring_finish(sh, tid, nthreads, L, t)            after the last barrier: CTA state -> table
#pragma once
#include "groupby.cuh"

namespace sx {

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <class P>
__host__ __device__ constexpr size_t ring_smem_bytes();
template <class P>
__host__ __device__ constexpr size_t ring_stage_bytes() {
  size_t b = 0;
  for (int c = 0; c < P::kRingCols; ++c) b += (size_t)P::kRingTile * P::ring_width(c);
  return b;
}

template <class P>
__host__ __device__ constexpr size_t ring_smem_bytes() {
  return (size_t)P::kRingStages * ring_stage_bytes<P>() + P::kRingExtraBytes;
}

template <class P, class = void>
struct has_ring : std::false_type {};
template <class P>
struct has_ring<P, std::void_t<decltype(P::kRingCols)>> : std::true_type {};

template <class P>
__device__ __forceinline__ void ring_init_bars(uint64_t* full, uint64_t* empty) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < P::kRingStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], P::kRingConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

// The pipeline after ring_init_bars + a __syncthreads: warp kRingConsumers produces, the others
// call consume(b[], row0, cw, lane) once per tile of this CTA's chunk [t0, t1) of n / kRingTile
// whole tiles.  Returns true on consumer threads.
template <class P, class F>
__device__ __forceinline__ bool ring_pipeline(const P& prog, int64_t n, uint8_t* ring, uint64_t* full, uint64_t* empty,
                                              F&& consume) {
  constexpr int C = P::kRingCols, S = P::kRingStages, T = P::kRingTile, NC = P::kRingConsumers;
  constexpr size_t SB = ring_stage_bytes<P>();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = n / T;
  const int64_t t0 = ntiles * blockIdx.x / gridDim.x, t1 = ntiles * (blockIdx.x + 1) / gridDim.x;
  if (warp == NC) {  // producer: one elected lane issues every bulk copy
    if (lane == 0) {
      int64_t k = 0;
      for (int64_t tile = t0; tile < t1; ++tile, ++k) {
        const int s = (int)(k % S);
        if (k >= S) mbar_wait(&empty[s], (uint32_t)(((k / S) - 1) & 1));
        mbar_expect_tx(&full[s], (uint32_t)SB);
        size_t off = 0;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const int w = P::ring_width(c);
          bulk_g2s(ring + s * SB + off, (const uint8_t*)prog.ring_col(c) + tile * (int64_t)T * w, (uint32_t)(T * w),
                   &full[s]);
          off += (size_t)T * w;
        }
      }
    }
    return false;
  }
  int64_t k = 0;
  for (int64_t tile = t0; tile < t1; ++tile, ++k) {
    const int s = (int)(k % S);
    mbar_wait(&full[s], (uint32_t)((k / S) & 1));
    const uint8_t* b[C];
    size_t off = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      b[c] = ring + s * SB + off;
      off += (size_t)T * P::ring_width(c);
    }
    consume(b, tile * (int64_t)T, warp, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  return true;
}

template <class P>
__global__ void __launch_bounds__((P::kRingConsumers + 1) * 32, 1)
    k_gb_ring(const __grid_constant__ P prog, int64_t n, const __grid_constant__ Layout L, Table t) {
  constexpr int S = P::kRingStages, T = P::kRingTile;
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ __align__(8) uint64_t empty[S];
  __shared__ typename P::RingShared sh;
  ring_init_bars<P>(full, empty);
  uint8_t* const xs = ring + (size_t)S * ring_stage_bytes<P>();  // the program's extra shared memory
  prog.ring_shared_init(sh, xs, threadIdx.x, blockDim.x);
  __syncthreads();
  typename P::RingAcc acc;
  prog.ring_init(acc);
  const bool consumer = ring_pipeline(prog, n, ring, full, empty, [&](const uint8_t* const* b, int64_t row0, int cw, int lane) {
    prog.ring_consume(b, row0, cw, lane, acc, sh, xs);
  });
  if (consumer) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntiles = n / T;
    if (blockIdx.x == gridDim.x - 1 && ntiles * T < n) prog.ring_tail(ntiles * T, n, warp, lane, acc, sh, xs);
    prog.ring_flush(acc, warp, lane, sh, xs);
  }
  __syncthreads();
  prog.ring_finish(sh, threadIdx.x, blockDim.x, L, t);
}

}  // namespace sx
