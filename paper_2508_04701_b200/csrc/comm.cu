// comm.cu — H10: multi-GPU exchange.  PAPER.md P:284 ("exchange is modeled as
// dedicated physical operators ... broadcast, shuffle, merge ... implemented using NCCL
// primitives"), P:458 (Q3's distributed plan shuffles orders and lineitem).
//
//   sx_partition_by_rank  destination rank = ((hash64(key) >> 32) * nranks) >> 32 (the high hash
//                         bits; table slots use the low bits — reading R14), rows regrouped by
//                         destination (stable within each destination: ordered compaction per rank)
//   sx_shuffle            partition_by_rank + counts all-to-all + grouped ncclSend/ncclRecv
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

// rows whose destination is `dest` (ordered compaction functor)
struct DestFn {
  DCol k0, k1;
  int nkeys, nranks, dest;
  template <int ITEMS>
  __device__ __forceinline__ void eval(const int32_t (&row)[ITEMS], const bool (&valid)[ITEMS], bool (&alive)[ITEMS],
                                       int32_t (&aux)[ITEMS]) const {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      bool a = valid[i];
      if (a) {
        uint64_t key = (uint64_t)ldv(k0, row[i]);
        if (nkeys == 2) key = (key << 32) | (uint32_t)ldv(k1, row[i]);
        a = dest_rank(key, nranks) == dest;
      }
      alive[i] = a;
    }
  }
};

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
  int64_t n = in_sel ? in_sel->len : cols[key_cols[0]].len;
  Scratch scr(ctx);
  std::vector<void*> dst(ncols);
  for (int c = 0; c < ncols; ++c) {
    int w = type_width(cols[c].type);
    if (!w) return set_err(ctx, SX_ETYPE, "column %d is not fixed-width", c);
    SX_TRY(scr.get((char**)&dst[c], (size_t)(n > 0 ? n : 1) * w));
  }
  int64_t off = 0;
  for (int d = 0; d < nranks; ++d) {
    DestFn f{dc[key_cols[0]], dc[nkeys > 1 ? key_cols[1] : key_cols[0]], nkeys, nranks, d};
    GatherSpec gs;
    gs.n = ncols;
    for (int c = 0; c < ncols; ++c) {
      int w = type_width(cols[c].type);
      gs.g[c].src = dc[c];
      gs.g[c].dst = (char*)dst[c] + off * w;
      gs.g[c].by_aux = 0;
      gs.g[c].width = w;
    }
    int64_t cnt = 0;
    int32_t* sel = nullptr;  // destination d's row ids (temporary); payload lands at dst + off
    SX_TRY(run_compact(ctx, f, n, in_sel ? in_sel->idx : nullptr, &sel, nullptr, gs, &cnt));
    dfree(ctx, sel);
    counts[d] = cnt;
    off += cnt;
  }
  for (int c = 0; c < ncols; ++c) {
    out_cols[c] = cols[c];
    out_cols[c].len = n;
    out_cols[c].data = dst[c];
    out_cols[c].offsets = nullptr;
    scr.release(dst[c]);
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

SX_EXPORT sx_status sx_shuffle(sx_ctx* ctx, sx_comm* comm, const sx_col* cols, int ncols, const int32_t* key_cols,
                               int nkeys, const sx_sel* in_sel, sx_col* out_cols, int64_t* out_rows) {
  if (!ctx || !comm || !out_cols || !out_rows) return SX_EINVAL;
  *out_rows = 0;
  ProfScope ps(ctx, "shuffle");
  const int g = comm->nranks;
  std::vector<int64_t> send(g), recv((size_t)g * g);
  std::vector<sx_col> part(ncols);
  SX_TRY(sx_partition_by_rank(ctx, cols, ncols, key_cols, nkeys, in_sel, g, part.data(), send.data()));
  Scratch scr(ctx);
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
  for (int c = 0; c < ncols; ++c) {
    int w = type_width(cols[c].type);
    char* out;
    SX_TRY(alloc(ctx, &out, (size_t)(total > 0 ? total : 1) * w));
    SX_NCCL(ncclGroupStart());
    int64_t soff = 0, roff = 0;
    for (int peer = 0; peer < g; ++peer) {
      int64_t sc = send[peer], rc = recv[(size_t)peer * g + comm->rank];
      if (sc) SX_NCCL(ncclSend((const char*)part[c].data + soff * w, (size_t)sc * w, ncclUint8, peer, comm->nccl, ctx->stream));
      if (rc) SX_NCCL(ncclRecv(out + roff * w, (size_t)rc * w, ncclUint8, peer, comm->nccl, ctx->stream));
      soff += sc;
      roff += rc;
    }
    SX_NCCL(ncclGroupEnd());
    out_cols[c] = cols[c];
    out_cols[c].len = total;
    out_cols[c].data = out;
    out_cols[c].offsets = nullptr;
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
  if (!ctx || !comm || (ncols > 0 && (!cols || !out_cols)) || !out_rows) return SX_EINVAL;
  *out_rows = 0;
  ProfScope ps(ctx, "allgather");
  int64_t n = ncols > 0 ? cols[0].len : 0;
  std::vector<int64_t> all;
  SX_TRY(allgather_i64(ctx, comm, n, all));
  int64_t total = 0;
  for (int64_t v : all) total += v;
  for (int c = 0; c < ncols; ++c) {
    if (cols[c].len != n) return set_err(ctx, SX_EINVAL, "allgather columns differ in length");
    int w = type_width(cols[c].type);
    if (!w) return set_err(ctx, SX_ETYPE, "column %d is not fixed-width", c);
    char* out;
    SX_TRY(alloc(ctx, &out, (size_t)(total > 0 ? total : 1) * w));
    SX_NCCL(ncclGroupStart());
    int64_t off = 0;
    for (int r = 0; r < comm->nranks; ++r) {
      if (all[r]) SX_NCCL(ncclBroadcast(r == comm->rank ? cols[c].data : out + off * w, out + off * w,
                                        (size_t)all[r] * w, ncclUint8, r, comm->nccl, ctx->stream));
      off += all[r];
    }
    SX_NCCL(ncclGroupEnd());
    out_cols[c] = cols[c];
    out_cols[c].len = total;
    out_cols[c].data = out;
    out_cols[c].offsets = nullptr;
  }
  *out_rows = total;
  if (ps.on()) {  // this rank's rows sent to every other rank
    double w = 0;
    for (int c = 0; c < ncols; ++c) w += type_width(cols[c].type);
    ps.set_bytes(w * (double)n * (comm->nranks - 1));
  }
  return SX_OK;
}
