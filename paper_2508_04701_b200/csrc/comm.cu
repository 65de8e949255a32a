// comm.cu — H10: multi-GPU exchange.  PAPER.md P:284 ("exchange is modeled as
// dedicated physical operators ... broadcast, shuffle, merge ... implemented using NCCL
// primitives"), P:458 (Q3's distributed plan shuffles orders and lineitem).
//
//   sx_partition_by_rank  destination rank = ((hash64(key) >> 32) * nranks) >> 32 (the high hash
//                         bits; table slots use the low bits — reading R14), rows regrouped by
//                         destination in ONE pass (histogram, scan, stable scatter; K15a/b below)
//   sx_shuffle            partition_by_rank + counts allgather + one group of ncclSend/ncclRecv
//   sx_allgather          counts allgather + ncclBroadcast from every rank (variable lengths)
// One process per GPU; the communicator comes from ncclCommInitRank with a unique id the caller
// distributes (bench.py uses torch.distributed for that plumbing only).
#include <nccl.h>

#include <vector>

#include "compact.cuh"

using namespace sx;

struct sx_comm {
  ncclComm_t nccl = nullptr;
  int rank = 0, nranks = 1;
};

#define SX_NCCL(call)                                                                                     \
  do {                                                                                                    \
    ncclResult_t r_ = (call);                                                                             \
    if (r_ != ncclSuccess) return ::sx::set_err(ctx, SX_ENCCL, "%s: %s", #call, ncclGetErrorString(r_));  \
  } while (0)

namespace {

__device__ __forceinline__ int dest_rank(uint64_t key, int nranks) {
  return (int)(((hash64(key) >> 32) * (uint64_t)nranks) >> 32);
}

// One-pass stable partition by destination rank (the earlier version ran one
// ordered compaction per destination, reading the input nranks times).
//   K15a k_rank_hist     per 2048-row tile: destination histogram -> hist[d * ntiles + tile]
//        scan            destination-major exclusive scan -> every (destination, tile) cursor
//   K15b k_rank_scatter  per tile: rows in index order (i, warp, lane); __match_any_sync ranks each
//                        row among its warp's rows of the same destination, a shared-memory scan
//                        over (destination, i, warp) orders the warp groups; every carried column
//                        is written straight to its destination segment (input order kept).
constexpr int kRpThreads = 256;
constexpr int kRpItems = 8;
constexpr int kRpTile = kRpThreads * kRpItems;
constexpr int kRpWarps = kRpThreads / 32;
constexpr int kMaxRanks = 64;

struct RankPartSpec {
  DCol k0, k1;
  int nkeys, nranks;
  const int32_t* sel;
  int64_t n, ntiles;
  int ncols;
  DCol src[kMaxGather];
  int width[kMaxGather];
  void* dst[kMaxGather];
};

__device__ __forceinline__ int row_dest(const RankPartSpec& s, int64_t r) {
  uint64_t key = (uint64_t)ldv(s.k0, r);
  if (s.nkeys == 2) key = (key << 32) | (uint32_t)ldv(s.k1, r);
  return dest_rank(key, s.nranks);
}

__global__ void __launch_bounds__(kRpThreads) k_rank_hist(const __grid_constant__ RankPartSpec s, int32_t* hist) {
  __shared__ int h[kMaxRanks];
  for (int64_t tile = blockIdx.x; tile < s.ntiles; tile += gridDim.x) {
    for (int d = threadIdx.x; d < s.nranks; d += kRpThreads) h[d] = 0;
    __syncthreads();
    const int64_t base = tile * kRpTile;
#pragma unroll
    for (int i = 0; i < kRpItems; ++i) {
      const int64_t idx = base + i * kRpThreads + threadIdx.x;
      if (idx < s.n) atomicAdd(&h[row_dest(s, s.sel ? (int64_t)__ldg(s.sel + idx) : idx)], 1);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < s.nranks; d += kRpThreads) hist[(int64_t)d * s.ntiles + tile] = h[d];
    __syncthreads();
  }
}

__device__ __forceinline__ void put_val(const DCol& src, int w, void* dst, int64_t d, int64_t r) {
  switch (w) {
    case 1: ((uint8_t*)dst)[d] = __ldg((const uint8_t*)src.p + r); break;
    case 4: ((int32_t*)dst)[d] = __ldg((const int32_t*)src.p + r); break;
    case 8: ((long long*)dst)[d] = __ldg((const long long*)src.p + r); break;
    default: ((longlong2*)dst)[d] = __ldg((const longlong2*)src.p + r); break;
  }
}

__global__ void __launch_bounds__(kRpThreads) k_rank_scatter(const __grid_constant__ RankPartSpec s,
                                                             const int64_t* __restrict__ offs) {
  // wc[(d * kRpItems + i) * kRpWarps + w]: rows of warp w, item i bound for d (then its scan)
  __shared__ int wc[kMaxRanks * kRpItems * kRpWarps];
  __shared__ int wsum[kRpWarps];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int m = s.nranks * kRpItems * kRpWarps;  // <= 4096
  constexpr int kPer = kMaxRanks * kRpItems * kRpWarps / kRpThreads;
  for (int64_t tile = blockIdx.x; tile < s.ntiles; tile += gridDim.x) {
    for (int j = tid; j < m; j += kRpThreads) wc[j] = 0;
    __syncthreads();
    const int64_t base = tile * kRpTile;
    int32_t row[kRpItems];
    int dst[kRpItems], rnk[kRpItems];
#pragma unroll
    for (int i = 0; i < kRpItems; ++i) {
      const int64_t idx = base + i * kRpThreads + tid;
      dst[i] = -1;
      if (idx < s.n) {
        row[i] = s.sel ? __ldg(s.sel + idx) : (int32_t)idx;
        dst[i] = row_dest(s, row[i]);
      }
      const unsigned peers = __match_any_sync(kFull, dst[i]);
      rnk[i] = __popc(peers & lanemask_lt());
      if (dst[i] >= 0 && rnk[i] == 0) wc[(dst[i] * kRpItems + i) * kRpWarps + w] = __popc(peers);
    }
    __syncthreads();
    // exclusive scan of wc[0..m) (destination-major): each thread a contiguous slice of kPer
    {
      int loc[kPer], sum = 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int k = tid * kPer + j;
        loc[j] = k < m ? wc[k] : 0;
        sum += loc[j];
      }
      int x = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[w] = x;
      __syncthreads();
      int run = x - sum;
      for (int k = 0; k < w; ++k) run += wsum[k];
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int k = tid * kPer + j;
        if (k < m) wc[k] = run;
        run += loc[j];
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kRpItems; ++i) {
      if (dst[i] < 0) continue;
      const int d = dst[i];
      // tile-local position within d's segment = scan(d, i, w) - scan(d, 0, 0) + rank
      const int64_t pos = offs[(int64_t)d * s.ntiles + tile] + (wc[(d * kRpItems + i) * kRpWarps + w] -
                                                                wc[d * kRpItems * kRpWarps]) + rnk[i];
      for (int c = 0; c < s.ncols; ++c) put_val(s.src[c], s.width[c], s.dst[c], pos, row[i]);
    }
    __syncthreads();
  }
}

__global__ void k_rank_counts(const int64_t* __restrict__ offs, int64_t ntiles, int nranks, int64_t total,
                              int64_t* __restrict__ counts) {
  const int d = threadIdx.x;
  if (d < nranks) counts[d] = (d + 1 < nranks ? offs[(int64_t)(d + 1) * ntiles] : total) - offs[(int64_t)d * ntiles];
}

}  // namespace

SX_EXPORT int sx_dest_rank(uint64_t key, int nranks) {  // host mirror of the device function (tests)
  return (int)(((hash64(key) >> 32) * (uint64_t)nranks) >> 32);
}

SX_EXPORT sx_status sx_partition_by_rank(sx_ctx* ctx, const sx_col* cols, int ncols, const int32_t* key_cols,
                                         int nkeys, const sx_sel* in_sel, int nranks, sx_col* out_cols,
                                         int64_t* counts) {
  if (!ctx || !cols || !key_cols || !out_cols || !counts || nkeys < 1 || nkeys > 2 || nranks < 1 ||
      ncols > kMaxGather)
    return SX_EINVAL;
  ProfScope ps(ctx, "partition_rank");
  DCol dc[SX_MAX_COLS];
  SX_TRY(to_dcols(ctx, cols, ncols, dc));
  for (int k = 0; k < nkeys; ++k) {
    if (key_cols[k] < 0 || key_cols[k] >= ncols) return set_err(ctx, SX_EINVAL, "key column out of range");
    int t = cols[key_cols[k]].type;
    if (!is_int_type(t) || (nkeys == 2 && key_bits(t) > 32)) return set_err(ctx, SX_ETYPE, "shuffle key type %d", t);
  }
  if (nranks > kMaxRanks) return set_err(ctx, SX_EINVAL, "nranks %d > %d", nranks, kMaxRanks);
  int64_t n = in_sel ? in_sel->len : cols[key_cols[0]].len;
  if (n > INT32_MAX) return set_err(ctx, SX_EINDEX, "%lld rows > INT32_MAX", (long long)n);
  Scratch scr(ctx);
  RankPartSpec s{};
  s.k0 = dc[key_cols[0]];
  s.k1 = dc[nkeys > 1 ? key_cols[1] : key_cols[0]];
  s.nkeys = nkeys;
  s.nranks = nranks;
  s.sel = in_sel ? in_sel->idx : nullptr;
  s.n = n;
  s.ntiles = (n + kRpTile - 1) / kRpTile;
  s.ncols = ncols;
  for (int c = 0; c < ncols; ++c) {
    int w = type_width(cols[c].type);
    if (!w) return set_err(ctx, SX_ETYPE, "column %d is not fixed-width", c);
    s.src[c] = dc[c];
    s.width[c] = w;
    SX_TRY(scr.get((char**)&s.dst[c], (size_t)(n > 0 ? n : 1) * w));
  }
  for (int d = 0; d < nranks; ++d) counts[d] = 0;
  if (n > 0) {
    const int64_t m = (int64_t)nranks * s.ntiles;
    int32_t* hist;
    int64_t *offs, *dcounts;
    SX_TRY(scr.get(&hist, (size_t)m));
    SX_TRY(scr.get(&offs, (size_t)m + 1));
    SX_TRY(scr.get(&dcounts, (size_t)nranks));
    const unsigned grid = persistent_grid(ctx, 4, s.ntiles);
    k_rank_hist<<<grid, kRpThreads, 0, SX_STREAM(ctx)>>>(s, hist);
    SX_CHECK_LAUNCH();
    int64_t total = 0;
    SX_TRY(scan_counts(ctx, hist, m, offs, &total));
    k_rank_scatter<<<grid, kRpThreads, 0, SX_STREAM(ctx)>>>(s, offs);
    SX_CHECK_LAUNCH();
    k_rank_counts<<<1, kMaxRanks, 0, SX_STREAM(ctx)>>>(offs, s.ntiles, nranks, total, dcounts);
    SX_CHECK_LAUNCH();
    SX_CUDA(cudaMemcpyAsync(counts, dcounts, sizeof(int64_t) * nranks, cudaMemcpyDeviceToHost, ctx->stream));
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  for (int c = 0; c < ncols; ++c) {
    out_cols[c] = cols[c];
    out_cols[c].len = n;
    out_cols[c].data = s.dst[c];
    out_cols[c].offsets = nullptr;
    scr.release(s.dst[c]);
  }
  if (ps.on()) {  // keys read twice is implementation cost: every carried column read + written once
    double w = 0;
    for (int c = 0; c < ncols; ++c) w += type_width(cols[c].type);
    ps.set_bytes(2.0 * w * (double)n + (in_sel ? 4.0 * n : 0.0));
  }
  return SX_OK;
}

SX_EXPORT sx_status sx_comm_unique_id(void* out) {
  if (!out) return SX_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SX_ENCCL;
  memcpy(out, &id, sizeof id);
  return SX_OK;
}

SX_EXPORT sx_status sx_comm_init(sx_ctx* ctx, const void* unique_id, int rank, int nranks, sx_comm** out) {
  if (!ctx || !unique_id || !out || nranks < 1 || rank < 0 || rank >= nranks) return SX_EINVAL;
  *out = nullptr;
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof id);
  SX_CUDA(cudaSetDevice(ctx->device));
  sx_comm* c = new sx_comm();
  c->rank = rank;
  c->nranks = nranks;
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return set_err(ctx, SX_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  *out = c;
  return SX_OK;
}

SX_EXPORT void sx_comm_destroy(sx_comm* c) {
  if (!c) return;
  if (c->nccl) ncclCommDestroy(c->nccl);
  delete c;
}

SX_EXPORT int sx_comm_rank(const sx_comm* c) { return c ? c->rank : -1; }
SX_EXPORT int sx_comm_size(const sx_comm* c) { return c ? c->nranks : -1; }

namespace {

// allgather one int64 per rank -> host array
sx_status allgather_i64(sx_ctx* ctx, sx_comm* comm, int64_t v, std::vector<int64_t>& all) {
  Scratch scr(ctx);
  int64_t* d;
  SX_TRY(scr.get(&d, (size_t)comm->nranks + 1));
  SX_CUDA(cudaMemcpyAsync(d + comm->nranks, &v, sizeof v, cudaMemcpyHostToDevice, ctx->stream));
  SX_NCCL(ncclAllGather(d + comm->nranks, d, 1, ncclInt64, comm->nccl, ctx->stream));
  all.assign(comm->nranks, 0);
  SX_CUDA(cudaMemcpyAsync(all.data(), d, sizeof(int64_t) * comm->nranks, cudaMemcpyDeviceToHost, ctx->stream));
  SX_CUDA(cudaStreamSynchronize(ctx->stream));
  return SX_OK;
}

}  // namespace

namespace {
// Issue one grouped batch of point-to-point calls; ncclGroupEnd runs on every path (an error
// inside the group must not leave NCCL's group state open).
template <class F>
sx_status nccl_group(sx_ctx* ctx, F&& body) {
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return set_err(ctx, SX_ENCCL, "ncclGroupStart: %s", ncclGetErrorString(r));
  ncclResult_t rb = body();
  ncclResult_t re = ncclGroupEnd();
  if (rb != ncclSuccess) return set_err(ctx, SX_ENCCL, "grouped send/recv: %s", ncclGetErrorString(rb));
  if (re != ncclSuccess) return set_err(ctx, SX_ENCCL, "ncclGroupEnd: %s", ncclGetErrorString(re));
  return SX_OK;
}
}  // namespace

SX_EXPORT sx_status sx_shuffle(sx_ctx* ctx, sx_comm* comm, const sx_col* cols, int ncols, const int32_t* key_cols,
                               int nkeys, const sx_sel* in_sel, sx_col* out_cols, int64_t* out_rows) {
  if (!ctx || !comm || !out_cols || !out_rows || ncols < 1 || ncols > kMaxGather) return SX_EINVAL;
  *out_rows = 0;
  for (int c = 0; c < ncols; ++c) out_cols[c] = sx_col{};
  ProfScope ps(ctx, "shuffle");
  const int g = comm->nranks;
  std::vector<int64_t> send(g), recv((size_t)g * g);
  std::vector<sx_col> part(ncols);
  SX_TRY(sx_partition_by_rank(ctx, cols, ncols, key_cols, nkeys, in_sel, g, part.data(), send.data()));
  Scratch scr(ctx);  // partitioned send buffers, and the outputs until the exchange succeeded
  for (int c = 0; c < ncols; ++c) scr.ptrs.push_back((void*)part[c].data);
  // counts matrix: every rank learns every rank's per-destination counts
  int64_t* dsend;
  int64_t* dall;
  SX_TRY(scr.get(&dsend, (size_t)g));
  SX_TRY(scr.get(&dall, (size_t)g * g));
  SX_CUDA(cudaMemcpyAsync(dsend, send.data(), sizeof(int64_t) * g, cudaMemcpyHostToDevice, ctx->stream));
  SX_NCCL(ncclAllGather(dsend, dall, g, ncclInt64, comm->nccl, ctx->stream));
  SX_CUDA(cudaMemcpyAsync(recv.data(), dall, sizeof(int64_t) * g * g, cudaMemcpyDeviceToHost, ctx->stream));
  SX_CUDA(cudaStreamSynchronize(ctx->stream));
  int64_t total = 0;
  for (int s = 0; s < g; ++s) total += recv[(size_t)s * g + comm->rank];
  std::vector<char*> out(ncols);
  for (int c = 0; c < ncols; ++c) SX_TRY(scr.get(&out[c], (size_t)(total > 0 ? total : 1) * type_width(cols[c].type)));
  // every column's sends and receives in ONE group (NCCL overlaps them across peers and columns)
  SX_TRY(nccl_group(ctx, [&]() -> ncclResult_t {
    for (int c = 0; c < ncols; ++c) {
      const int w = type_width(cols[c].type);
      int64_t soff = 0, roff = 0;
      for (int peer = 0; peer < g; ++peer) {
        const int64_t sc = send[peer], rc = recv[(size_t)peer * g + comm->rank];
        ncclResult_t r = ncclSuccess;
        if (sc) r = ncclSend((const char*)part[c].data + soff * w, (size_t)sc * w, ncclUint8, peer, comm->nccl, ctx->stream);
        if (r == ncclSuccess && rc) r = ncclRecv(out[c] + roff * w, (size_t)rc * w, ncclUint8, peer, comm->nccl, ctx->stream);
        if (r != ncclSuccess) return r;
        soff += sc;
        roff += rc;
      }
    }
    return ncclSuccess;
  }));
  for (int c = 0; c < ncols; ++c) {
    out_cols[c] = cols[c];
    out_cols[c].len = total;
    out_cols[c].data = out[c];
    out_cols[c].offsets = nullptr;
    scr.release(out[c]);
  }
  *out_rows = total;
  if (ps.on()) {  // a shuffle's bytes are the bytes leaving this GPU
    double w = 0, rows_out = 0;
    for (int c = 0; c < ncols; ++c) w += type_width(cols[c].type);
    for (int peer = 0; peer < g; ++peer)
      if (peer != comm->rank) rows_out += (double)send[peer];
    ps.set_bytes(w * rows_out);
  }
  return SX_OK;
}

SX_EXPORT sx_status sx_allgather(sx_ctx* ctx, sx_comm* comm, const sx_col* cols, int ncols, sx_col* out_cols,
                                 int64_t* out_rows) {
  if (!ctx || !comm || (ncols > 0 && (!cols || !out_cols)) || !out_rows || ncols > SX_MAX_COLS) return SX_EINVAL;
  *out_rows = 0;
  for (int c = 0; c < ncols; ++c) out_cols[c] = sx_col{};
  ProfScope ps(ctx, "allgather");
  int64_t n = ncols > 0 ? cols[0].len : 0;
  for (int c = 0; c < ncols; ++c) {
    if (cols[c].len != n) return set_err(ctx, SX_EINVAL, "allgather columns differ in length");
    if (!type_width(cols[c].type)) return set_err(ctx, SX_ETYPE, "column %d is not fixed-width", c);
  }
  std::vector<int64_t> all;
  SX_TRY(allgather_i64(ctx, comm, n, all));
  int64_t total = 0;
  for (int64_t v : all) total += v;
  Scratch scr(ctx);  // outputs until the exchange succeeded
  std::vector<char*> out(ncols);
  for (int c = 0; c < ncols; ++c) SX_TRY(scr.get(&out[c], (size_t)(total > 0 ? total : 1) * type_width(cols[c].type)));
  SX_TRY(nccl_group(ctx, [&]() -> ncclResult_t {
    for (int c = 0; c < ncols; ++c) {
      const int w = type_width(cols[c].type);
      int64_t off = 0;
      for (int r = 0; r < comm->nranks; ++r) {
        if (all[r]) {
          ncclResult_t e = ncclBroadcast(r == comm->rank ? cols[c].data : out[c] + off * w, out[c] + off * w,
                                         (size_t)all[r] * w, ncclUint8, r, comm->nccl, ctx->stream);
          if (e != ncclSuccess) return e;
        }
        off += all[r];
      }
    }
    return ncclSuccess;
  }));
  for (int c = 0; c < ncols; ++c) {
    out_cols[c] = cols[c];
    out_cols[c].len = total;
    out_cols[c].data = out[c];
    out_cols[c].offsets = nullptr;
    scr.release(out[c]);
  }
  *out_rows = total;
  if (ps.on()) {  // this rank's rows sent to every other rank
    double w = 0;
    for (int c = 0; c < ncols; ++c) w += type_width(cols[c].type);
    ps.set_bytes(w * (double)n * (comm->nranks - 1));
  }
  return SX_OK;
}
