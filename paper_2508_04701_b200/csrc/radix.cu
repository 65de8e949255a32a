// radix.cu — H5: hash-bit radix partitioning (K7) and the radix-partitioned hash join.
//
// "hash-bit partitioning of both join sides when build > L2"; north_star:
// "radix-partitioned joins when the build side exceeds L2".  PAPER.md P:351 lists GPU join
// algorithms (gpu-join-eth) among the techniques Sirius can adopt; P:418 — joins dominate the
// join-heavy queries.  The paper gives no kernel design; this is ours, for sm_100a:
//
//   sx_radix_partition  one pass, fan-out 2^bits (<= 2^10): partition(key) = (hash64(key) >> 48)
//                       & (2^bits - 1) — hash bits 48..57, disjoint from the table-slot bits (low)
//                       and from the shard-rank bits (top, sx_dest_rank; reading R14).
//     K7a k_part_hist     per-CTA histogram of a contiguous chunk (shared-memory atomics)
//         scan            partition-major exclusive scan -> every (partition, CTA) output cursor
//     K7b k_part_scatter  per 2048-row tile: shared-memory counting sort by partition, then the
//                         tile is written partition run by partition run (coalesced runs)
//   sx_hash_join        build + probe in one call.  Flat (sx_hash_build + sx_hash_probe) while the
//                       table fits half the L2; above that (unique build, INNER), both sides are
//                       radix-partitioned carrying their payload columns, and the partitions are
//                       joined in waves whose tables together stay L2-resident: probes hit L2
//                       instead of random HBM sectors, payloads are never gathered at random.
#include <algorithm>
#include <cstring>
#include <vector>

#include "compact.cuh"
#include "join.cuh"
#include "radix.cuh"

using namespace sx;

namespace {

constexpr int kPartThreads = 256;
constexpr int kPartItems = 8;  // (16: 4096-row tiles measured slower, 65.5 vs 59 ms join µbench)
constexpr int kPartTile = kPartThreads * kPartItems;  // rows per staged tile
constexpr int kMaxPartBits = 10;
constexpr int kPartShift = 48;
constexpr int kMaxCarry = 12;

struct PartSpec {
  DCol k0, k1;
  int nkeys;
  int bits;
  int ncarry;
  DCol carry[kMaxCarry];
  int width[kMaxCarry];
  void* out[kMaxCarry];
  int32_t* out_rowid;  // optional: original row id of every output row
  const int32_t* sel;
  int64_t n;
  int64_t chunk;  // rows per CTA (multiple of kPartTile)
};

__device__ __forceinline__ uint64_t part_key(const DCol& k0, const DCol& k1, int nkeys, int64_t r) {
  uint64_t k = (uint64_t)ldv(k0, r);
  if (nkeys == 2) k = (k << 32) | (uint32_t)ldv(k1, r);
  return k;
}

__host__ __device__ __forceinline__ uint32_t part_of(uint64_t key, int bits) {
  return (uint32_t)(hash64(key) >> kPartShift) & ((1u << bits) - 1u);
}

// 8 rows per thread per step, their key loads issued together (one row per step left the kernel
// latency-bound at ~2.3 TB/s), counted into per-warp shared histograms (fewer same-address
// conflicts), summed at the end.
constexpr int kHistItems = 8;
__global__ void __launch_bounds__(kPartThreads) k_part_hist(const __grid_constant__ PartSpec s, int32_t* hist) {
  __shared__ int h[kPartThreads / 32][1 << kMaxPartBits];
  const int P = 1 << s.bits;
  const int w = threadIdx.x >> 5;
  for (int j = threadIdx.x; j < (kPartThreads / 32) * P; j += blockDim.x) h[j / P][j % P] = 0;
  __syncthreads();
  const int64_t lo = blockIdx.x * s.chunk, hi = min(s.n, lo + s.chunk);
  for (int64_t b = lo; b < hi; b += (int64_t)kHistItems * blockDim.x) {
    uint64_t k[kHistItems];
    bool in[kHistItems];
#pragma unroll
    for (int u = 0; u < kHistItems; ++u) {
      const int64_t i = b + (int64_t)u * blockDim.x + threadIdx.x;
      in[u] = i < hi;
      const int64_t r = in[u] ? (s.sel ? (int64_t)__ldg(s.sel + i) : i) : 0;
      k[u] = in[u] ? part_key(s.k0, s.k1, s.nkeys, r) : 0;
    }
#pragma unroll
    for (int u = 0; u < kHistItems; ++u)
      if (in[u]) atomicAdd(&h[w][part_of(k[u], s.bits)], 1);
  }
  __syncthreads();
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    int c = 0;
#pragma unroll
    for (int q = 0; q < kPartThreads / 32; ++q) c += h[q][p];
    hist[(int64_t)p * gridDim.x + blockIdx.x] = c;
  }
}

__device__ __forceinline__ void copy_val(const DCol& src, int w, void* dst, int64_t d, int64_t r) {
  switch (w) {
    case 1: ((uint8_t*)dst)[d] = __ldg((const uint8_t*)src.p + r); break;
    case 4: ((int32_t*)dst)[d] = __ldg((const int32_t*)src.p + r); break;
    case 8: ((long long*)dst)[d] = __ldg((const long long*)src.p + r); break;
    default: ((longlong2*)dst)[d] = __ldg((const longlong2*)src.p + r); break;
  }
}

__global__ void __launch_bounds__(kPartThreads) k_part_scatter(const __grid_constant__ PartSpec s,
                                                               const int64_t* __restrict__ offs) {
  __shared__ int64_t cursor[1 << kMaxPartBits];
  __shared__ int cnt[1 << kMaxPartBits];
  __shared__ int start[1 << kMaxPartBits];
  __shared__ uint16_t s_part[kPartTile];
  __shared__ int32_t s_row[kPartTile];
  __shared__ int s_warp[kPartThreads / 32];
  const int P = 1 << s.bits;
  const int tid = threadIdx.x;
  for (int p = tid; p < P; p += kPartThreads) cursor[p] = offs[(int64_t)p * gridDim.x + blockIdx.x];
  const int64_t lo = blockIdx.x * s.chunk, hi = min(s.n, lo + s.chunk);
  for (int64_t base = lo; base < hi; base += kPartTile) {
    for (int p = tid; p < P; p += kPartThreads) cnt[p] = 0;
    __syncthreads();
    int32_t row[kPartItems];
    int part[kPartItems], rank[kPartItems];
#pragma unroll
    for (int i = 0; i < kPartItems; ++i) {
      const int64_t idx = base + (int64_t)i * kPartThreads + tid;
      part[i] = -1;
      if (idx < hi) {
        row[i] = s.sel ? __ldg(s.sel + idx) : (int32_t)idx;
        part[i] = (int)part_of(part_key(s.k0, s.k1, s.nkeys, row[i]), s.bits);
        rank[i] = atomicAdd(&cnt[part[i]], 1);
      }
    }
    __syncthreads();
    // exclusive scan of cnt[0..P) -> start[] (each thread scans a contiguous slice)
    {
      constexpr int kPer = (1 << kMaxPartBits) / kPartThreads;
      int loc[kPer], sum = 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int p = tid * kPer + j;
        loc[j] = p < P ? cnt[p] : 0;
        sum += loc[j];
      }
      int x = sum;
      const int lane = tid & 31, w = tid >> 5;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_warp[w] = x;
      __syncthreads();
      int wo = 0;
      for (int k = 0; k < w; ++k) wo += s_warp[k];
      int run = wo + x - sum;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int p = tid * kPer + j;
        if (p < P) start[p] = run;
        run += loc[j];
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kPartItems; ++i) {
      if (part[i] < 0) continue;
      const int pos = start[part[i]] + rank[i];
      s_part[pos] = (uint16_t)part[i];
      s_row[pos] = row[i];
    }
    __syncthreads();
    const int tcount = (int)min((int64_t)kPartTile, hi - base);
    for (int j = tid; j < tcount; j += kPartThreads) {
      const int p = s_part[j];
      const int64_t d = cursor[p] + (j - start[p]);
      const int32_t r = s_row[j];
      for (int c = 0; c < s.ncarry; ++c) copy_val(s.carry[c], s.width[c], s.out[c], d, r);
      if (s.out_rowid) s.out_rowid[d] = r;
    }
    __syncthreads();
    for (int p = tid; p < P; p += kPartThreads) cursor[p] += cnt[p];
    __syncthreads();
  }
}

// K7b' (default): 4096-row tiles; ranks within a partition from shared atomics, and every
// carried column is staged in shared memory in partition order — loaded
// coalesced at the tile's own rows, written as partition runs (~32 rows of each column per
// partition per tile at fan-out 128) — instead of re-gathering each value by row id at write
// time.  One column at a time, so the staging buffer is 16 B x 4096 at most.
constexpr int kVsItems = 16;
constexpr int kVsTile = kPartThreads * kVsItems;

__device__ __forceinline__ void stage_val(const DCol& src, int w, uint8_t* sb, int pos, int64_t r) {
  switch (w) {
    case 1: sb[pos] = __ldcs((const uint8_t*)src.p + r); break;
    case 4: ((int32_t*)sb)[pos] = __ldcs((const int32_t*)src.p + r); break;
    case 8: ((long long*)sb)[pos] = __ldcs((const long long*)src.p + r); break;
    default: ((longlong2*)sb)[pos] = __ldcs((const longlong2*)src.p + r); break;
  }
}
__device__ __forceinline__ void emit_val(int w, const uint8_t* sb, int j, void* dst, int64_t d) {
  switch (w) {
    case 1: ((uint8_t*)dst)[d] = sb[j]; break;
    case 4: ((int32_t*)dst)[d] = ((const int32_t*)sb)[j]; break;
    case 8: ((long long*)dst)[d] = ((const long long*)sb)[j]; break;
    default: ((longlong2*)dst)[d] = ((const longlong2*)sb)[j]; break;
  }
}

__global__ void __launch_bounds__(kPartThreads, 3) k_part_scatter_v(const __grid_constant__ PartSpec s,
                                                                 const int64_t* __restrict__ offs, int max_w) {
  extern __shared__ __align__(16) uint8_t sbuf[];  // kVsTile * max_w
  __shared__ int64_t cursor[1 << kMaxPartBits];
  __shared__ int cnt[1 << kMaxPartBits];
  __shared__ int start[1 << kMaxPartBits];
  __shared__ uint16_t s_part[kVsTile];
  __shared__ int s_warp[kPartThreads / 32];
  const int P = 1 << s.bits;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int p = tid; p < P; p += kPartThreads) cursor[p] = offs[(int64_t)p * gridDim.x + blockIdx.x];
  const int64_t lo = blockIdx.x * s.chunk, hi = min(s.n, lo + s.chunk);
  for (int64_t base = lo; base < hi; base += kVsTile) {
    for (int p = tid; p < P; p += kPartThreads) cnt[p] = 0;
    __syncthreads();
    // pr[i] = partition << 16 | rank within the partition (tile-local position after the scan);
    // -1 past the end.  Row ids are recomputed (or re-read from the selection) when staging.
    int pr[kVsItems];
#pragma unroll
    for (int i = 0; i < kVsItems; ++i) {
      const int64_t idx = base + (int64_t)i * kPartThreads + tid;
      pr[i] = -1;
      if (idx < hi) {
        const int32_t row = s.sel ? __ldg(s.sel + idx) : (int32_t)idx;
        const int p = (int)part_of(part_key(s.k0, s.k1, s.nkeys, row), s.bits);
        pr[i] = (p << 16) | atomicAdd(&cnt[p], 1);  // order within a partition is free (R12)
      }
    }
    __syncthreads();
    {
      constexpr int kPer = (1 << kMaxPartBits) / kPartThreads;
      int loc[kPer], sum = 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int p = tid * kPer + j;
        loc[j] = p < P ? cnt[p] : 0;
        sum += loc[j];
      }
      int x = sum;
      const int w = tid >> 5;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_warp[w] = x;
      __syncthreads();
      int wo = 0;
      for (int k = 0; k < w; ++k) wo += s_warp[k];
      int run = wo + x - sum;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int p = tid * kPer + j;
        if (p < P) start[p] = run;
        run += loc[j];
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kVsItems; ++i) {
      if (pr[i] < 0) continue;
      const int p = pr[i] >> 16;
      pr[i] = start[p] + (pr[i] & 0xffff);  // now the tile-local position
      s_part[pr[i]] = (uint16_t)p;
    }
    const int tcount = (int)min((int64_t)kVsTile, hi - base);
    const int ncols = s.ncarry + (s.out_rowid ? 1 : 0);
    for (int c = 0; c < ncols; ++c) {
      const bool rid = c == s.ncarry;
      const int w = rid ? 4 : s.width[c];
#pragma unroll
      for (int i = 0; i < kVsItems; ++i) {
        if (pr[i] < 0) continue;
        const int64_t idx = base + (int64_t)i * kPartThreads + tid;
        const int32_t row = s.sel ? __ldg(s.sel + idx) : (int32_t)idx;
        if (rid) ((int32_t*)sbuf)[pr[i]] = row;
        else stage_val(s.carry[c], w, sbuf, pr[i], row);
      }
      __syncthreads();
      void* dst = rid ? (void*)s.out_rowid : s.out[c];
      for (int j = tid; j < tcount; j += kPartThreads) {
        const int p = s_part[j];
        emit_val(w, sbuf, j, dst, cursor[p] + (j - start[p]));
      }
      __syncthreads();
    }
    for (int p = tid; p < P; p += kPartThreads) cursor[p] += cnt[p];
    __syncthreads();
  }
}

// K7r: the common case — <= 3 carried columns of 4 or 8 bytes whose first nkeys ARE the key
// columns, no selection, no row ids.  Every carried value of the tile is loaded into registers
// when the tile starts (one memory round trip per tile; the staged variant above loads each
// column after the ranking, one round trip per column: ncu long-scoreboard bound at ~1.4 TB/s),
// the partition is computed from the loaded key, ranks come from shared atomics, and each column
// then goes through shared memory to its partition runs.  512 threads x 8 rows = 4096-row tiles.
constexpr int kRsThreads = 512;
constexpr int kRsItems = 8;
constexpr int kRsTile = kRsThreads * kRsItems;

template <int NC>
__global__ void __launch_bounds__(kRsThreads, 2) k_part_scatter_r(const __grid_constant__ PartSpec s,
                                                                  const int64_t* __restrict__ offs) {
  extern __shared__ __align__(16) unsigned char rs_dyn[];
  unsigned long long* sbuf = (unsigned long long*)rs_dyn;  // [kRsTile]
  __shared__ int64_t cursor[1 << kMaxPartBits];
  __shared__ int cnt[1 << kMaxPartBits];
  __shared__ int start[1 << kMaxPartBits];
  __shared__ uint16_t s_part[kRsTile];
  __shared__ int s_warp[kRsThreads / 32];
  const int P = 1 << s.bits;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int p = tid; p < P; p += kRsThreads) cursor[p] = offs[(int64_t)p * gridDim.x + blockIdx.x];
  const int64_t lo = blockIdx.x * s.chunk, hi = min(s.n, lo + s.chunk);
  for (int64_t base = lo; base < hi; base += kRsTile) {
    for (int p = tid; p < P; p += kRsThreads) cnt[p] = 0;
    // every carried value of my rows (as 64-bit; 4-byte columns sign-extended like ldv)
    unsigned long long v[NC][kRsItems];
#pragma unroll
    for (int i = 0; i < kRsItems; ++i) {
      const int64_t idx = base + (int64_t)i * kRsThreads + tid;
      const bool in = idx < hi;
#pragma unroll
      for (int c = 0; c < NC; ++c)
        v[c][i] = !in ? 0ull
                  : s.width[c] == 8 ? (unsigned long long)__ldcs((const long long*)s.carry[c].p + idx)
                                    : (unsigned long long)(long long)__ldcs((const int32_t*)s.carry[c].p + idx);
    }
    __syncthreads();  // cnt[] cleared
    int pr[kRsItems];  // partition << 16 | rank
#pragma unroll
    for (int i = 0; i < kRsItems; ++i) {
      const int64_t idx = base + (int64_t)i * kRsThreads + tid;
      pr[i] = -1;
      if (idx < hi) {
        uint64_t k = v[0][i];
        if (NC >= 2 && s.nkeys == 2) k = (k << 32) | (uint32_t)v[NC >= 2 ? 1 : 0][i];
        const int p = (int)part_of(k, s.bits);
        pr[i] = (p << 16) | atomicAdd(&cnt[p], 1);  // order within a partition is free (R12)
      }
    }
    __syncthreads();
    {
      constexpr int kPer = (1 << kMaxPartBits) / kRsThreads;
      int loc[kPer], sum = 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int p = tid * kPer + j;
        loc[j] = p < P ? cnt[p] : 0;
        sum += loc[j];
      }
      int x = sum;
      const int w = tid >> 5;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_warp[w] = x;
      __syncthreads();
      int wo = 0;
      for (int k = 0; k < w; ++k) wo += s_warp[k];
      int run = wo + x - sum;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int p = tid * kPer + j;
        if (p < P) start[p] = run;
        run += loc[j];
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kRsItems; ++i) {
      if (pr[i] < 0) continue;
      const int p = pr[i] >> 16;
      pr[i] = start[p] + (pr[i] & 0xffff);
      s_part[pr[i]] = (uint16_t)p;
    }
    const int tcount = (int)min((int64_t)kRsTile, hi - base);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      __syncthreads();  // s_part complete / the previous column's reads done
#pragma unroll
      for (int i = 0; i < kRsItems; ++i)
        if (pr[i] >= 0) sbuf[pr[i]] = v[c][i];
      __syncthreads();
      if (s.width[c] == 8) {
        long long* dst = (long long*)s.out[c];
        for (int j = tid; j < tcount; j += kRsThreads) {
          const int p = s_part[j];
          __stcs(dst + cursor[p] + (j - start[p]), (long long)sbuf[j]);
        }
      } else {
        int32_t* dst = (int32_t*)s.out[c];
        for (int j = tid; j < tcount; j += kRsThreads) {
          const int p = s_part[j];
          __stcs(dst + cursor[p] + (j - start[p]), (int32_t)sbuf[j]);
        }
      }
    }
    __syncthreads();
    for (int p = tid; p < P; p += kRsThreads) cursor[p] += cnt[p];
    __syncthreads();
  }
}

// Partition rows (n, through sel) by hash bits; carried columns land partition-contiguous.
// offsets_h (host, P+1) receives the partition boundaries.
sx_status radix_partition(sx_ctx* ctx, PartSpec& s, int64_t* offsets_h) {
  const int P = 1 << s.bits;
  // SX_PART_SCATTER=rowid: the round-1 scatter (row ids staged, values re-gathered at write time)
  const char* mode = getenv("SX_PART_SCATTER");
  const bool v2 = !(mode && std::strcmp(mode, "rowid") == 0);
  // K7r when every carried column is 4 or 8 bytes wide, the keys are carried first, <= 3 columns
  bool reg = v2 && !(mode && std::strcmp(mode, "staged") == 0) && !s.sel && !s.out_rowid && s.ncarry >= s.nkeys &&
             s.ncarry <= 3;
  for (int c = 0; reg && c < s.ncarry; ++c) reg = s.width[c] == 4 || s.width[c] == 8;
  reg = reg && s.carry[0].p == s.k0.p && (s.nkeys == 1 || s.carry[1].p == s.k1.p);
  reg = reg && (s.nkeys == 1 ? (s.width[0] == 8 || s.k0.type == SX_I32 || s.k0.type == SX_DATE32)
                             : (s.width[0] == 4 && s.width[1] == 4));
  const int tile_rows = reg ? kRsTile : v2 ? kVsTile : kPartTile;
  int max_w = 4;
  for (int c = 0; c < s.ncarry; ++c) max_w = std::max(max_w, s.width[c]);
  const size_t vsmem = (size_t)kVsTile * max_w;
  int64_t tiles = (s.n + tile_rows - 1) / tile_rows;
  unsigned grid = persistent_grid(ctx, 4, tiles > 0 ? tiles : 1);
  int64_t tiles_per = (tiles + grid - 1) / grid;
  s.chunk = std::max<int64_t>(1, tiles_per) * tile_rows;
  grid = (unsigned)std::max<int64_t>(1, (s.n + s.chunk - 1) / s.chunk);
  Scratch scr(ctx);
  int32_t* hist;
  int64_t* offs;
  const int64_t m = (int64_t)P * grid;
  SX_TRY(scr.get(&hist, (size_t)m));
  SX_TRY(scr.get(&offs, (size_t)m + 1));
  int64_t total = 0;
  if (s.n > 0) {
    k_part_hist<<<grid, kPartThreads, 0, SX_STREAM(ctx)>>>(s, hist);
    SX_CHECK_LAUNCH();
    SX_TRY(scan_counts(ctx, hist, m, offs, &total));
    if (reg) {
      const size_t rsm = (size_t)kRsTile * sizeof(unsigned long long);
      switch (s.ncarry) {
        case 1:
          SX_CUDA(cudaFuncSetAttribute(k_part_scatter_r<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));
          k_part_scatter_r<1><<<grid, kRsThreads, rsm, SX_STREAM(ctx)>>>(s, offs);
          break;
        case 2:
          SX_CUDA(cudaFuncSetAttribute(k_part_scatter_r<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));
          k_part_scatter_r<2><<<grid, kRsThreads, rsm, SX_STREAM(ctx)>>>(s, offs);
          break;
        default:
          SX_CUDA(cudaFuncSetAttribute(k_part_scatter_r<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));
          k_part_scatter_r<3><<<grid, kRsThreads, rsm, SX_STREAM(ctx)>>>(s, offs);
          break;
      }
    } else if (v2) {
      SX_CUDA(cudaFuncSetAttribute(k_part_scatter_v, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vsmem));
      k_part_scatter_v<<<grid, kPartThreads, vsmem, SX_STREAM(ctx)>>>(s, offs, max_w);
    } else {
      k_part_scatter<<<grid, kPartThreads, 0, SX_STREAM(ctx)>>>(s, offs);
    }
    SX_CHECK_LAUNCH();
    std::vector<int64_t> all((size_t)m + 1);
    SX_CUDA(cudaMemcpyAsync(all.data(), offs, sizeof(int64_t) * (m + 1), cudaMemcpyDeviceToHost, ctx->stream));
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int p = 0; p < P; ++p) offsets_h[p] = all[(size_t)p * grid];
    offsets_h[P] = total;
  } else {
    for (int p = 0; p <= P; ++p) offsets_h[p] = 0;
  }
  return SX_OK;
}

sx_status check_keys(sx_ctx* ctx, const sx_col* cols, int ncols, const int32_t* key_cols, int nkeys, int* kb) {
  if (nkeys < 1 || nkeys > 2 || !key_cols) return set_err(ctx, SX_EINVAL, "nkeys %d (1 or 2)", nkeys);
  for (int k = 0; k < nkeys; ++k) {
    if (key_cols[k] < 0 || key_cols[k] >= ncols) return set_err(ctx, SX_EINVAL, "key column out of range");
    int t = cols[key_cols[k]].type;
    if (!(t == SX_I32 || t == SX_DATE32 || t == SX_I64) || (nkeys == 2 && t == SX_I64))
      return set_err(ctx, SX_ETYPE, "join key type %d", t);
  }
  *kb = (nkeys == 1 && cols[key_cols[0]].type != SX_I64) ? 4 : 8;
  return SX_OK;
}

// ------------------------------------------------------------------ partitioned join (waves)
struct PJoin {
  // partitioned build side
  const void* bkey;  // uint32 (kb 4) or uint64 packed keys
  const int32_t* brow;
  // partitioned probe side
  const void* pkey;
  const int32_t* prow;
  int kb;
  int bits;
  int p0;                 // first partition of the wave
  uint64_t cap;           // slots per partition table (power of two)
  HtSlot8* slots;         // wave tables: partition (p - p0) at slots + (p - p0) * cap
  int64_t b_lo, b_hi;     // build tuple range of the wave
  int64_t p_lo, p_hi;     // probe tuple range of the wave
  // outputs
  unsigned long long* cursor;
  int32_t* out_probe;     // optional
  int32_t* out_build;     // optional
  int npay;
  DCol pay_src[kMaxCarry];  // partitioned payload columns (build ones indexed by jb, probe ones by jp)
  int pay_build[kMaxCarry];
  int pay_w[kMaxCarry];
  void* pay_dst[kMaxCarry];
};

// Partitioned sides are streamed once per wave: evict-first loads (ld.global.cs) and stores
// (st.global.cs) keep the wave's tables resident in L2.
__device__ __forceinline__ uint64_t pj_key(const void* k, int kb, int64_t j) {
  return kb == 4 ? (uint64_t)__ldcs((const uint32_t*)k + j) : (uint64_t)__ldcs((const unsigned long long*)k + j);
}

__device__ __forceinline__ void copy_val_cs(const DCol& src, int w, void* dst, int64_t d, int64_t r) {
  switch (w) {
    case 1: ((uint8_t*)dst)[d] = __ldcs((const uint8_t*)src.p + r); break;
    case 4: __stcs((int32_t*)dst + d, __ldcs((const int32_t*)src.p + r)); break;
    case 8: __stcs((long long*)dst + d, __ldcs((const long long*)src.p + r)); break;
    default: __stcs((longlong2*)dst + d, __ldcs((const longlong2*)src.p + r)); break;
  }
}

__global__ void __launch_bounds__(kBlock) k_pj_build(const __grid_constant__ PJoin a) {
  for (int64_t j = a.b_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < a.b_hi;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = pj_key(a.bkey, a.kb, j);
    const uint64_t h = hash64(key);
    HtSlot8* t = a.slots + (uint64_t)(((uint32_t)(h >> kPartShift) & ((1u << a.bits) - 1u)) - a.p0) * a.cap;
    uint64_t s = h & (a.cap - 1);
    while (atomicCAS(&t[s].row, 0xffffffffu, (unsigned)(j - a.b_lo)) != 0xffffffffu) s = (s + 1) & (a.cap - 1);
    t[s].key = key;
  }
}

constexpr int kPjItems = 4;
__global__ void __launch_bounds__(kBlock, 4) k_pj_probe(const __grid_constant__ PJoin a) {
  __shared__ int s_warp[kBlock / 32];
  __shared__ unsigned long long s_base;
  const int64_t tile = (int64_t)kBlock * kPjItems;
  for (int64_t base = a.p_lo + blockIdx.x * tile; base < a.p_hi; base += (int64_t)gridDim.x * tile) {
    int64_t jb[kPjItems];
    uint64_t key[kPjItems], s[kPjItems];
    const HtSlot8* t[kPjItems];
    bool pend[kPjItems];
#pragma unroll
    for (int i = 0; i < kPjItems; ++i) {
      const int64_t j = base + (int64_t)i * kBlock + threadIdx.x;
      pend[i] = j < a.p_hi;
      key[i] = pend[i] ? pj_key(a.pkey, a.kb, j) : 0;
      const uint64_t h = hash64(key[i]);
      t[i] = a.slots + (uint64_t)(((uint32_t)(h >> kPartShift) & ((1u << a.bits) - 1u)) - a.p0) * a.cap;
      if (!pend[i]) t[i] = a.slots;
      s[i] = h & (a.cap - 1);
      jb[i] = -1;
    }
    bool any = true;
    while (any) {
      any = false;
      longlong2 v[kPjItems];
#pragma unroll
      for (int i = 0; i < kPjItems; ++i) v[i] = pend[i] ? __ldg((const longlong2*)(t[i] + s[i])) : make_longlong2(0, -1);
#pragma unroll
      for (int i = 0; i < kPjItems; ++i) {
        if (!pend[i]) continue;
        const uint32_t rw = (uint32_t)(unsigned long long)v[i].y;
        if (rw == 0xffffffffu) {
          pend[i] = false;
        } else if ((uint64_t)v[i].x == key[i]) {
          jb[i] = a.b_lo + rw;
          pend[i] = false;
        } else {
          s[i] = (s[i] + 1) & (a.cap - 1);
          any = true;
        }
      }
    }
    // tile-level output allocation: one atomic per CTA tile
    int c = 0;
#pragma unroll
    for (int i = 0; i < kPjItems; ++i) c += jb[i] >= 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int k = 0; k < kBlock / 32; ++k) tot += s_warp[k];
      s_base = tot ? atomicAdd(a.cursor, (unsigned long long)tot) : 0ull;
    }
    __syncthreads();
    int wo = 0;
    for (int k = 0; k < w; ++k) wo += s_warp[k];
    int64_t pos = (int64_t)s_base + wo + x - c;
#pragma unroll
    for (int i = 0; i < kPjItems; ++i) {
      if (jb[i] < 0) continue;
      const int64_t jp = base + (int64_t)i * kBlock + threadIdx.x;
      if (a.out_probe) __stcs(a.out_probe + pos, __ldcs(a.prow + jp));
      if (a.out_build) __stcs(a.out_build + pos, __ldcs(a.brow + jb[i]));
      for (int g = 0; g < a.npay; ++g)
        copy_val_cs(a.pay_src[g], a.pay_w[g], a.pay_dst[g], pos, a.pay_build[g] ? jb[i] : jp);
      ++pos;
    }
    __syncthreads();
  }
}

// ---- inline-value partitioned join (K8i) ---------------------------------------------------
// When each side carries at most ONE value to the output (a payload column of width <= 8, or the
// row id), the build value lives in the slot beside its key — {key64, value} — so a probe is one
// 16-byte L2 load and the output needs no second (dependent) access into the build side.  The key
// ~0 is the EMPTY marker; a build key equal to ~0 is kept in a side cell instead.  Output:
// per-CTA tile of kPiTile probes, hits staged in shared memory in probe order and written as one
// contiguous run claimed with a single atomic per tile (join output order is unspecified, R12).
struct PJoinI {
  const void* bkey;
  const void* pkey;
  int kb;
  int bits;
  int p0;
  uint64_t cap;
  ulonglong2* slots;
  int64_t b_lo, b_hi, p_lo, p_hi;
  DCol bval;  // partitioned build value (width <= 8), or row ids
  DCol pval;  // partitioned probe value, or row ids; p == nullptr: none
  int bw, pw;  // output widths (0: not produced)
  unsigned long long* cursor;
  unsigned long long* side;  // [0] 1 when the key ~0 is in the build, [1] its value
  void* out_b;
  void* out_p;
};

__device__ __forceinline__ int64_t ld_val_cs(const DCol& c, int64_t j) {
  switch (c.type) {
    case SX_U8: return (int64_t)__ldcs((const uint8_t*)c.p + j);
    case SX_I64:
    case SX_DEC64:
      return (int64_t)__ldcs((const long long*)c.p + j);
    default: return (int64_t)__ldcs((const int32_t*)c.p + j);
  }
}
__device__ __forceinline__ void st_val(void* dst, int w, int64_t d, int64_t v) {
  switch (w) {
    case 1: ((uint8_t*)dst)[d] = (uint8_t)v; break;
    case 4: __stcs((int32_t*)dst + d, (int32_t)v); break;
    default: __stcs((long long*)dst + d, (long long)v); break;
  }
}

__global__ void __launch_bounds__(kBlock) k_pji_build(const __grid_constant__ PJoinI a) {
  for (int64_t j = a.b_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < a.b_hi;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = pj_key(a.bkey, a.kb, j);
    const int64_t val = ld_val_cs(a.bval, j);
    if (key == ~0ull) {
      a.side[1] = (unsigned long long)val;
      a.side[0] = 1ull;
      continue;
    }
    const uint64_t h = hash64(key);
    ulonglong2* t = a.slots + (uint64_t)(((uint32_t)(h >> kPartShift) & ((1u << a.bits) - 1u)) - a.p0) * a.cap;
    uint64_t s = h & (a.cap - 1);
    while (atomicCAS(&t[s].x, ~0ull, key) != ~0ull) s = (s + 1) & (a.cap - 1);
    t[s].y = (unsigned long long)val;
  }
}

constexpr int kPiItems = 4;
constexpr int kPiTile = kBlock * kPiItems;
// Per warp: 32 x kPiItems probes; the probe value is loaded with the key (not after the output is
// claimed), and each warp claims its output run with its own atomic (no CTA barrier between the
// lookups and the writes; ncu on the CTA-synchronised version: 62% long-scoreboard stalls).
__global__ void __launch_bounds__(kBlock, 3) k_pji_probe(const __grid_constant__ PJoinI a) {
  const int lane = threadIdx.x & 31;
  const bool side_on = a.side[0] != 0;
  const long long side_v = (long long)a.side[1];
  const uint64_t m = a.cap - 1;
  const int64_t wstride = (int64_t)gridDim.x * kPiTile;
  const int64_t wofs = (int64_t)(threadIdx.x >> 5) * 32 * kPiItems;
  for (int64_t base = a.p_lo + blockIdx.x * (int64_t)kPiTile + wofs; base < a.p_hi; base += wstride) {
    // idx: global slot index (region base | in-region slot; regions are cap-aligned)
    uint64_t key[kPiItems], idx[kPiItems];
    long long bv[kPiItems], pv[kPiItems];
    bool pend[kPiItems], hit[kPiItems];
#pragma unroll
    for (int i = 0; i < kPiItems; ++i) {
      const int64_t j = base + (int64_t)i * 32 + lane;
      const bool v = j < a.p_hi;
      key[i] = v ? pj_key(a.pkey, a.kb, j) : ~0ull;
      pv[i] = (v && a.pw) ? ld_val_cs(a.pval, j) : 0;
    }
#pragma unroll
    for (int i = 0; i < kPiItems; ++i) {
      const int64_t j = base + (int64_t)i * 32 + lane;
      const bool v = j < a.p_hi;
      const uint64_t h = hash64(key[i]);
      idx[i] = (uint64_t)(((uint32_t)(h >> kPartShift) & ((1u << a.bits) - 1u)) - a.p0) * a.cap + (h & m);
      hit[i] = v && key[i] == ~0ull && side_on;
      bv[i] = side_v;
      pend[i] = v && key[i] != ~0ull;
      if (!pend[i]) idx[i] = 0;
    }
    bool any = true;
    while (any) {
      any = false;
      ulonglong2 sv[kPiItems];
#pragma unroll
      for (int i = 0; i < kPiItems; ++i) sv[i] = pend[i] ? __ldg(a.slots + idx[i]) : make_ulonglong2(~0ull, 0ull);
#pragma unroll
      for (int i = 0; i < kPiItems; ++i) {
        if (!pend[i]) continue;
        if (sv[i].x == key[i]) {
          hit[i] = true;
          bv[i] = (long long)sv[i].y;
          pend[i] = false;
        } else if (sv[i].x == ~0ull) {
          pend[i] = false;
        } else {
          idx[i] = (idx[i] & ~m) | ((idx[i] + 1) & m);
          any = true;
        }
      }
    }
    // the warp's hits, item by item, land contiguously in one run claimed by one atomic
    unsigned ball[kPiItems];
    int tot = 0;
#pragma unroll
    for (int i = 0; i < kPiItems; ++i) {
      ball[i] = __ballot_sync(kFull, hit[i]);
      tot += __popc(ball[i]);
    }
    unsigned long long wb = 0;
    if (lane == 0 && tot) wb = atomicAdd(a.cursor, (unsigned long long)tot);
    wb = __shfl_sync(kFull, wb, 0);
    const unsigned lt = lanemask_lt();
    int64_t pos = (int64_t)wb;
#pragma unroll
    for (int i = 0; i < kPiItems; ++i) {
      if (hit[i]) {
        const int64_t o = pos + __popc(ball[i] & lt);
        if (a.bw) st_val(a.out_b, a.bw, o, bv[i]);
        if (a.pw) st_val(a.out_p, a.pw, o, pv[i]);
      }
      pos += __popc(ball[i]);
    }
  }
}

}  // namespace

SX_EXPORT uint32_t sx_radix_of(uint64_t key, int bits) {  // host mirror of the partition function
  return (bits < 1 || bits > kMaxPartBits) ? 0u : part_of(key, bits);
}

SX_EXPORT sx_status sx_radix_partition(sx_ctx* ctx, const sx_col* cols, int ncols, const int32_t* key_cols, int nkeys,
                                       const sx_sel* in_sel, int bits, sx_col* out_cols, sx_sel* out_rows,
                                       int64_t* offsets) {
  if (!ctx || !cols || !out_cols || !offsets || bits < 1 || bits > kMaxPartBits || ncols < 1 || ncols > kMaxCarry)
    return SX_EINVAL;
  for (int c = 0; c < ncols; ++c) out_cols[c] = sx_col{};
  if (out_rows) *out_rows = sx_sel{0, nullptr};
  ProfScope ps(ctx, "radix_partition");
  DCol dc[SX_MAX_COLS];
  SX_TRY(to_dcols(ctx, cols, ncols, dc));
  int kb = 4;
  SX_TRY(check_keys(ctx, cols, ncols, key_cols, nkeys, &kb));
  const int64_t n = in_sel ? in_sel->len : cols[key_cols[0]].len;
  if (n > INT32_MAX) return set_err(ctx, SX_EINDEX, "partition input exceeds INT32_MAX rows");
  Scratch scr(ctx);
  PartSpec s{};
  s.k0 = dc[key_cols[0]];
  s.k1 = dc[nkeys > 1 ? key_cols[1] : key_cols[0]];
  s.nkeys = nkeys;
  s.bits = bits;
  s.ncarry = ncols;
  s.sel = in_sel ? in_sel->idx : nullptr;
  s.n = n;
  double row_b = 0;
  for (int c = 0; c < ncols; ++c) {
    const int w = type_width(cols[c].type);
    if (!w) return set_err(ctx, SX_ETYPE, "column %d is not fixed-width", c);
    s.carry[c] = dc[c];
    s.width[c] = w;
    SX_TRY(scr.get((char**)&s.out[c], (size_t)(n > 0 ? n : 1) * w));
    row_b += 2.0 * w;
  }
  if (out_rows) SX_TRY(scr.get(&s.out_rowid, (size_t)(n > 0 ? n : 1)));
  SX_TRY(radix_partition(ctx, s, offsets));
  for (int c = 0; c < ncols; ++c) {
    out_cols[c] = cols[c];
    out_cols[c].len = n;
    out_cols[c].data = s.out[c];
    out_cols[c].offsets = nullptr;
    scr.release(s.out[c]);
  }
  if (out_rows) {
    *out_rows = sx_sel{n, s.out_rowid};
    scr.release(s.out_rowid);
  }
  ps.set_bytes((row_b + (in_sel ? 4.0 : 0.0) + (out_rows ? 4.0 : 0.0)) * n);  // every column read + written once
  return SX_OK;
}

namespace {

// Packed key column of a partitioned side (uint32 for one 32-bit key, else uint64).
__global__ void k_pack_keys(DCol k0, DCol k1, int nkeys, int kb, int64_t n, void* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = (uint64_t)ldv(k0, i);
    if (nkeys == 2) k = (k << 32) | (uint32_t)ldv(k1, i);
    if (kb == 4) ((uint32_t*)out)[i] = (uint32_t)k;
    else ((unsigned long long*)out)[i] = k;
  }
}

}  // namespace

SX_EXPORT sx_status sx_hash_join(sx_ctx* ctx, const sx_col* build_cols, int nbuild_cols, const int32_t* build_keys,
                                 const sx_sel* build_sel, int unique_hint, const sx_col* probe_cols, int nprobe_cols,
                                 const int32_t* probe_keys, const sx_sel* probe_sel, int nkeys, int join_type,
                                 const int32_t* bp, int nbp, const int32_t* pp, int npp, int strategy,
                                 sx_sel* out_probe, sx_sel* out_build, sx_col* out_payload, int* used_strategy) {
  if (!ctx || !build_cols || !probe_cols || !build_keys || !probe_keys) return SX_EINVAL;
  if (out_probe) *out_probe = sx_sel{0, nullptr};
  if (out_build) *out_build = sx_sel{0, nullptr};
  for (int i = 0; out_payload && i < nbp + npp && i < kMaxCarry; ++i) out_payload[i] = sx_col{};
  if (used_strategy) *used_strategy = 0;
  if (nbp < 0 || npp < 0 || nbp + npp > kMaxCarry || ((nbp + npp) > 0 && !out_payload))
    return set_err(ctx, SX_EINVAL, "payload columns");
  if (join_type < SX_INNER || join_type > SX_ANTI) return set_err(ctx, SX_EINVAL, "join type %d", join_type);
  int kb = 4, kbp = 4;
  SX_TRY(check_keys(ctx, build_cols, nbuild_cols, build_keys, nkeys, &kb));
  SX_TRY(check_keys(ctx, probe_cols, nprobe_cols, probe_keys, nkeys, &kbp));
  if (kb != kbp) return set_err(ctx, SX_ETYPE, "build/probe key widths differ");
  const int64_t nb = build_sel ? build_sel->len : build_cols[build_keys[0]].len;
  const int64_t np = probe_sel ? probe_sel->len : probe_cols[probe_keys[0]].len;
  if (nb > INT32_MAX || np > INT32_MAX) return set_err(ctx, SX_EINDEX, "join side exceeds INT32_MAX rows");
  // strategy: 1 flat, 2 partitioned, 3 flat inline (K8f, below), 0 auto (partitioned when the flat
  // table would exceed half the L2)
  uint64_t flat_cap = 64;
  while (flat_cap < (uint64_t)(2 * nb)) flat_cap <<= 1;
  const size_t flat_bytes = flat_cap * (size_t)(kb == 4 ? 8 : 16);
  bool part = strategy >= 2 || (strategy == 0 && flat_bytes > ctx->l2_bytes / 2);
  if (join_type != SX_INNER || !unique_hint) part = false;  // partitioned path: PK build, INNER
  if (!part) {
    if (used_strategy) *used_strategy = 1;
    sx_ht* ht = nullptr;
    SX_TRY(sx_hash_build(ctx, build_cols, nbuild_cols, build_keys, nkeys, build_sel, nullptr, 0, unique_hint, &ht));
    sx_sel op{}, ob{};
    sx_status s = sx_hash_probe(ctx, ht, probe_cols, nprobe_cols, probe_keys, nkeys, probe_sel, nullptr, 0, join_type,
                                build_cols, nbuild_cols, bp, nbp, pp, npp, &op, join_type == SX_INNER ? &ob : nullptr,
                                out_payload);
    sx_ht_destroy(ctx, ht);
    if (s != SX_OK) return s;
    if (out_probe) *out_probe = op;
    else sx_free(ctx, op.idx);
    if (out_build) *out_build = ob;
    else sx_free(ctx, ob.idx);
    return SX_OK;
  }
  // strategy 3 (flat inline, K8f): the K8i kernels over the unpartitioned columns with zero
  // partition bits — one {key, value} table of 2^ceil(log2(2 nb)) 16-byte slots (HBM-resident
  // above ~60 MB), built once, probed once; no partition passes.  Needs one key column, no
  // selections, and at most one payload column per side (no row ids).
  if (strategy == 3 && nkeys == 1 && !build_sel && !probe_sel && !out_build && !out_probe && nbp <= 1 && npp <= 1 &&
      (nbp == 0 || type_width(build_cols[bp[0]].type) <= 8) && (npp == 0 || type_width(probe_cols[pp[0]].type) <= 8)) {
    if (used_strategy) *used_strategy = 3;
    ProfScope ps(ctx, "join_flat_inline");
    Scratch scr(ctx);
    DCol bdc[SX_MAX_COLS], pdc[SX_MAX_COLS];
    SX_TRY(to_dcols(ctx, build_cols, nbuild_cols, bdc));
    SX_TRY(to_dcols(ctx, probe_cols, nprobe_cols, pdc));
    PJoinI a{};
    a.bkey = build_cols[build_keys[0]].data;
    a.pkey = probe_cols[probe_keys[0]].data;
    a.kb = kb;
    a.bits = 0;
    a.p0 = 0;
    a.cap = flat_cap;
    void* ob_out = nullptr;
    void* op_out = nullptr;
    const size_t ocap = (size_t)(np > 0 ? np : 1);
    if (nbp == 1) {
      a.bval = bdc[bp[0]];
      a.bw = type_width(build_cols[bp[0]].type);
      SX_TRY(scr.get((char**)&ob_out, ocap * a.bw));
    }
    if (npp == 1) {
      a.pval = pdc[pp[0]];
      a.pw = type_width(probe_cols[pp[0]].type);
      SX_TRY(scr.get((char**)&op_out, ocap * a.pw));
    }
    a.out_b = ob_out;
    a.out_p = op_out;
    unsigned long long* side;
    SX_TRY(scr.get(&side, 2));
    SX_CUDA(cudaMemsetAsync(side, 0, 16, ctx->stream));
    a.side = side;
    a.cursor = (unsigned long long*)ctx->d_counters;
    SX_CUDA(cudaMemsetAsync(a.cursor, 0, 8, ctx->stream));
    ulonglong2* slots;
    SX_TRY(scr.get(&slots, (size_t)flat_cap));
    SX_CUDA(cudaMemsetAsync(slots, 0xff, (size_t)flat_cap * sizeof(ulonglong2), ctx->stream));
    a.slots = slots;
    a.b_lo = 0;
    a.b_hi = nb;
    a.p_lo = 0;
    a.p_hi = np;
    if (nb > 0 && np > 0) {
      k_pji_build<<<persistent_grid(ctx, 8, (nb + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(a);
      k_pji_probe<<<persistent_grid(ctx, 3, (np + kPiTile - 1) / kPiTile), kBlock, 0, SX_STREAM(ctx)>>>(a);
      SX_CHECK_LAUNCH();
    }
    int64_t count = 0;
    SX_TRY(read_i64(ctx, a.cursor, &count));
    if (nbp == 1) {
      out_payload[0] = build_cols[bp[0]];
      out_payload[0].len = count;
      out_payload[0].data = ob_out;
      out_payload[0].offsets = nullptr;
      scr.release(ob_out);
    }
    if (npp == 1) {
      out_payload[nbp] = probe_cols[pp[0]];
      out_payload[nbp].len = count;
      out_payload[nbp].data = op_out;
      out_payload[nbp].offsets = nullptr;
      scr.release(op_out);
    }
    const double kbytes = type_width(build_cols[build_keys[0]].type);
    ps.set_bytes(kbytes * (nb + np) + 2.0 * (a.bw + a.pw) * count);
    return SX_OK;
  }
  if (used_strategy) *used_strategy = 2;
  ProfScope ps(ctx, "join_partitioned");
  Scratch scr(ctx);
  DCol bdc[SX_MAX_COLS], pdc[SX_MAX_COLS];
  SX_TRY(to_dcols(ctx, build_cols, nbuild_cols, bdc));
  SX_TRY(to_dcols(ctx, probe_cols, nprobe_cols, pdc));
  // fan-out: per-partition tables of <= SX_PJ_PART_MB (default 32) MB (join µbench: 52.8 ms at
  // 32 MB, 59.0 at 16, 57.7 at 64, 70.8 at 8: fewer partitions give longer runs per partition in
  // each scatter tile, so fewer partial-sector writes)
  const int part_mb = getenv("SX_PJ_PART_MB") ? std::max(1, atoi(getenv("SX_PJ_PART_MB"))) : 32;
  int bits = 1;
  while (bits < kMaxPartBits && (flat_bytes >> bits) > ((uint64_t)part_mb << 20)) ++bits;
  const int P = 1 << bits;
  // partition both sides: carried = key columns, then payloads; + row ids if requested
  auto part_side = [&](const sx_col* cols, const DCol* dc, const int32_t* keys, const sx_sel* sel, int64_t n,
                       const int32_t* pay, int npay, bool rowid, PartSpec& s, std::vector<int64_t>& off) -> sx_status {
    s = PartSpec{};
    s.k0 = dc[keys[0]];
    s.k1 = dc[nkeys > 1 ? keys[1] : keys[0]];
    s.nkeys = nkeys;
    s.bits = bits;
    s.sel = sel ? sel->idx : nullptr;
    s.n = n;
    int c = 0;
    for (int k = 0; k < nkeys; ++k, ++c) {
      s.carry[c] = dc[keys[k]];
      s.width[c] = type_width(cols[keys[k]].type);
    }
    for (int g = 0; g < npay; ++g, ++c) {
      const int w = type_width(cols[pay[g]].type);
      if (!w) return set_err(ctx, SX_ETYPE, "payload must be fixed-width");
      s.carry[c] = dc[pay[g]];
      s.width[c] = w;
    }
    s.ncarry = c;
    for (int k = 0; k < c; ++k) SX_TRY(scr.get((char**)&s.out[k], (size_t)(n > 0 ? n : 1) * s.width[k]));
    if (rowid) SX_TRY(scr.get(&s.out_rowid, (size_t)(n > 0 ? n : 1)));
    off.assign((size_t)P + 1, 0);
    return radix_partition(ctx, s, off.data());
  };
  for (int g = 0; g < nbp; ++g)
    if (bp[g] < 0 || bp[g] >= nbuild_cols) return set_err(ctx, SX_EINVAL, "build payload column out of range");
  for (int g = 0; g < npp; ++g)
    if (pp[g] < 0 || pp[g] >= nprobe_cols) return set_err(ctx, SX_EINVAL, "probe payload column out of range");
  PartSpec bs, psp;
  std::vector<int64_t> boff, poff;
  SX_TRY(part_side(build_cols, bdc, build_keys, build_sel, nb, bp, nbp, out_build != nullptr, bs, boff));
  SX_TRY(part_side(probe_cols, pdc, probe_keys, probe_sel, np, pp, npp, out_probe != nullptr, psp, poff));
  // packed keys of both partitioned sides (a single key column already is one: 4-byte keys are
  // read as uint32, int64 keys as uint64)
  const void *bkey = bs.out[0], *pkey = psp.out[0];
  if (nkeys == 2) {
    void *bk2, *pk2;
    SX_TRY(scr.get((char**)&bk2, (size_t)(nb > 0 ? nb : 1) * kb));
    SX_TRY(scr.get((char**)&pk2, (size_t)(np > 0 ? np : 1) * kb));
    bkey = bk2;
    pkey = pk2;
    DCol b0{bs.out[0], build_cols[build_keys[0]].type, 0}, b1{bs.out[nkeys - 1], SX_I32, 0};
    DCol p0{psp.out[0], probe_cols[probe_keys[0]].type, 0}, p1{psp.out[nkeys - 1], SX_I32, 0};
    if (nb > 0) k_pack_keys<<<persistent_grid(ctx, 8, (nb + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(b0, b1, nkeys, kb, nb, bk2);
    if (np > 0) k_pack_keys<<<persistent_grid(ctx, 8, (np + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(p0, p1, nkeys, kb, np, pk2);
    SX_CHECK_LAUNCH();
  }
  // outputs (unique build: at most one match per probe row)
  const size_t ocap = (size_t)(np > 0 ? np : 1);
  // inline-value path (K8i): each side carries at most one value of width <= 8 (a payload column
  // or its row ids); SX_PJ_INLINE=0 forces the row-id path below
  auto carry_ok = [&](int npay, const sx_col* cols, const int32_t* pay, bool rows) {
    if (npay == 0) return true;
    return npay == 1 && !rows && type_width(cols[pay[0]].type) <= 8;
  };
  const bool inline_off = getenv("SX_PJ_INLINE") && getenv("SX_PJ_INLINE")[0] == '0';
  if (!inline_off && carry_ok(nbp, build_cols, bp, out_build != nullptr) &&
      carry_ok(npp, probe_cols, pp, out_probe != nullptr)) {
    PJoinI a{};
    a.bkey = bkey;
    a.pkey = pkey;
    a.kb = kb;
    a.bits = bits;
    void* ob_out = nullptr;
    void* op_out = nullptr;
    if (nbp == 1) {
      a.bval = DCol{bs.out[nkeys], build_cols[bp[0]].type, 0};
      a.bw = bs.width[nkeys];
    } else if (out_build) {
      a.bval = DCol{bs.out_rowid, SX_I32, 0};
      a.bw = 4;
    }
    if (npp == 1) {
      a.pval = DCol{psp.out[nkeys], probe_cols[pp[0]].type, 0};
      a.pw = psp.width[nkeys];
    } else if (out_probe) {
      a.pval = DCol{psp.out_rowid, SX_I32, 0};
      a.pw = 4;
    }
    if (a.bw) SX_TRY(scr.get((char**)&ob_out, ocap * a.bw));
    if (a.pw) SX_TRY(scr.get((char**)&op_out, ocap * a.pw));
    a.out_b = ob_out;
    a.out_p = op_out;
    unsigned long long* side;
    SX_TRY(scr.get(&side, 2));
    SX_CUDA(cudaMemsetAsync(side, 0, 16, ctx->stream));
    a.side = side;
    a.cursor = (unsigned long long*)ctx->d_counters;
    SX_CUDA(cudaMemsetAsync(a.cursor, 0, 8, ctx->stream));
    int64_t maxb = 1;
    for (int p = 0; p < P; ++p) maxb = std::max<int64_t>(maxb, boff[p + 1] - boff[p]);
    uint64_t cap = 64;
    while (cap < (uint64_t)(2 * maxb)) cap <<= 1;
    const size_t part_bytes = cap * sizeof(ulonglong2);
    const int l2div = getenv("SX_PJ_L2DIV") ? std::max(1, atoi(getenv("SX_PJ_L2DIV"))) : 3;
    int W = (int)std::max<size_t>(1, (ctx->l2_bytes / l2div) / part_bytes);
    W = std::min(W, P);
    ulonglong2* slots;
    SX_TRY(scr.get(&slots, (size_t)W * cap));
    a.slots = slots;
    a.cap = cap;
    for (int p0 = 0; p0 < P; p0 += W) {
      const int p1 = std::min(P, p0 + W);
      a.p0 = p0;
      a.b_lo = boff[p0];
      a.b_hi = boff[p1];
      a.p_lo = poff[p0];
      a.p_hi = poff[p1];
      if (a.b_hi == a.b_lo || a.p_hi == a.p_lo) continue;
      SX_CUDA(cudaMemsetAsync(slots, 0xff, (size_t)(p1 - p0) * cap * sizeof(ulonglong2), ctx->stream));
      const int64_t nbw = a.b_hi - a.b_lo, npw = a.p_hi - a.p_lo;
      k_pji_build<<<persistent_grid(ctx, 8, (nbw + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(a);
      k_pji_probe<<<persistent_grid(ctx, 3, (npw + kPiTile - 1) / kPiTile), kBlock, 0, SX_STREAM(ctx)>>>(a);
      SX_CHECK_LAUNCH();
      SX_CUDA(cudaMemsetAsync(side, 0, 16, ctx->stream));  // the side cell belongs to one wave
    }
    int64_t count = 0;
    SX_TRY(read_i64(ctx, a.cursor, &count));
    if (nbp == 1) {
      out_payload[0] = build_cols[bp[0]];
      out_payload[0].len = count;
      out_payload[0].data = ob_out;
      out_payload[0].offsets = nullptr;
      scr.release(ob_out);
    } else if (out_build) {
      *out_build = sx_sel{count, (int32_t*)ob_out};
      scr.release(ob_out);
    }
    if (npp == 1) {
      out_payload[nbp] = probe_cols[pp[0]];
      out_payload[nbp].len = count;
      out_payload[nbp].data = op_out;
      out_payload[nbp].offsets = nullptr;
      scr.release(op_out);
    } else if (out_probe) {
      *out_probe = sx_sel{count, (int32_t*)op_out};
      scr.release(op_out);
    }
    double kbytes = 0;
    for (int k = 0; k < nkeys; ++k) kbytes += type_width(build_cols[build_keys[k]].type);
    double b = (kbytes + (build_sel ? 4.0 : 0.0)) * nb + (kbytes + (probe_sel ? 4.0 : 0.0)) * np;
    b += 2.0 * (nbp ? a.bw : 0) * count + 2.0 * (npp ? a.pw : 0) * count;
    b += ((out_probe ? 4.0 : 0.0) + (out_build ? 4.0 : 0.0)) * count;
    ps.set_bytes(b);
    return SX_OK;
  }
  int32_t *op = nullptr, *ob = nullptr;
  if (out_probe) SX_TRY(scr.get(&op, ocap));
  if (out_build) SX_TRY(scr.get(&ob, ocap));
  PJoin a{};
  a.bkey = bkey;
  a.pkey = pkey;
  a.brow = bs.out_rowid;
  a.prow = psp.out_rowid;
  a.kb = kb;
  a.bits = bits;
  a.out_probe = op;
  a.out_build = ob;
  a.npay = nbp + npp;
  for (int g = 0; g < nbp; ++g) {
    a.pay_src[g] = DCol{bs.out[nkeys + g], build_cols[bp[g]].type, 0};
    a.pay_build[g] = 1;
    a.pay_w[g] = bs.width[nkeys + g];
  }
  for (int g = 0; g < npp; ++g) {
    a.pay_src[nbp + g] = DCol{psp.out[nkeys + g], probe_cols[pp[g]].type, 0};
    a.pay_build[nbp + g] = 0;
    a.pay_w[nbp + g] = psp.width[nkeys + g];
  }
  for (int g = 0; g < a.npay; ++g) SX_TRY(scr.get((char**)&a.pay_dst[g], ocap * a.pay_w[g]));
  a.cursor = (unsigned long long*)ctx->d_counters;
  SX_CUDA(cudaMemsetAsync(a.cursor, 0, 8, ctx->stream));
  // per-partition table size from the largest build partition; waves of partitions whose tables
  // together fit about half the L2
  int64_t maxb = 1;
  for (int p = 0; p < P; ++p) maxb = std::max<int64_t>(maxb, boff[p + 1] - boff[p]);
  uint64_t cap = 64;
  while (cap < (uint64_t)(2 * maxb)) cap <<= 1;
  const size_t part_bytes = cap * sizeof(HtSlot8);
  const int l2div = getenv("SX_PJ_L2DIV") ? std::max(1, atoi(getenv("SX_PJ_L2DIV"))) : 3;
  int W = (int)std::max<size_t>(1, (ctx->l2_bytes / l2div) / part_bytes);
  W = std::min(W, P);
  HtSlot8* slots;
  SX_TRY(scr.get(&slots, (size_t)W * cap));
  a.slots = slots;
  a.cap = cap;
  for (int p0 = 0; p0 < P; p0 += W) {
    const int p1 = std::min(P, p0 + W);
    a.p0 = p0;
    a.b_lo = boff[p0];
    a.b_hi = boff[p1];
    a.p_lo = poff[p0];
    a.p_hi = poff[p1];
    if (a.b_hi == a.b_lo || a.p_hi == a.p_lo) continue;
    SX_CUDA(cudaMemsetAsync(slots, 0xff, (size_t)(p1 - p0) * cap * sizeof(HtSlot8), ctx->stream));
    const int64_t nbw = a.b_hi - a.b_lo, npw = a.p_hi - a.p_lo;
    k_pj_build<<<persistent_grid(ctx, 8, (nbw + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(a);
    k_pj_probe<<<persistent_grid(ctx, 8, (npw + kBlock * kPjItems - 1) / (kBlock * kPjItems)), kBlock, 0, SX_STREAM(ctx)>>>(a);
    SX_CHECK_LAUNCH();
  }
  int64_t count = 0;
  SX_TRY(read_i64(ctx, a.cursor, &count));
  if (out_probe) {
    *out_probe = sx_sel{count, op};
    scr.release(op);
  }
  if (out_build) {
    *out_build = sx_sel{count, ob};
    scr.release(ob);
  }
  for (int g = 0; g < a.npay; ++g) {
    const sx_col& src = g < nbp ? build_cols[bp[g]] : probe_cols[pp[g - nbp]];
    out_payload[g] = src;
    out_payload[g].len = count;
    out_payload[g].data = a.pay_dst[g];
    out_payload[g].offsets = nullptr;
    scr.release(a.pay_dst[g]);
  }
  // algorithmic bytes: both sides' keys (+ selections) read once, payloads read once and written
  // once per output, row-id outputs once (build + probe definitions)
  double kbytes = 0;
  for (int k = 0; k < nkeys; ++k) kbytes += type_width(build_cols[build_keys[k]].type);
  double b = (kbytes + (build_sel ? 4.0 : 0.0)) * nb + (kbytes + (probe_sel ? 4.0 : 0.0)) * np;
  for (int g = 0; g < a.npay; ++g) b += 2.0 * a.pay_w[g] * count;
  b += ((out_probe ? 4.0 : 0.0) + (out_build ? 4.0 : 0.0)) * count;
  ps.set_bytes(b);
  return SX_OK;
}

namespace sx {
sx_status radix_partition_carry(sx_ctx* ctx, DCol k0, DCol k1, int nkeys, const DCol* carry, const int* width,
                                int ncarry, const int32_t* sel, int64_t n, int bits, void* const* out,
                                int64_t* offsets_h) {
  if (ncarry > kMaxCarry || bits < 1 || bits > kMaxPartBits) return set_err(ctx, SX_EINVAL, "radix partition spec");
  PartSpec s{};
  s.k0 = k0;
  s.k1 = k1;
  s.nkeys = nkeys;
  s.bits = bits;
  s.ncarry = ncarry;
  for (int c = 0; c < ncarry; ++c) {
    s.carry[c] = carry[c];
    s.width[c] = width[c];
    s.out[c] = out[c];
  }
  s.sel = sel;
  s.n = n;
  return radix_partition(ctx, s, offsets_h);
}
}  // namespace sx
