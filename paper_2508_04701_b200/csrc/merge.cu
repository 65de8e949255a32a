// merge.cu — FINAL phase of a distributed aggregation ("allgather merge of partial
// aggregates"; PAPER.md P:342 — avg must be carried as sum+count to be mergeable):
//   sx_groupby_merge: group partial rows by key and combine their states exactly
//                     (SUM: int128 add, COUNT: add, MIN/MAX: min/max);
//   sx_avg:           avg = (double)sum / (double)count / 10^scale (reading R3).
#include "gb_host.cuh"

using namespace sx;

namespace {

__global__ void k_pack_keys(DCol k0, DCol k1, int nkeys, int64_t n, unsigned long long* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = ldv(k0, i);
    out[i] = nkeys == 1 ? (unsigned long long)a
                        : (((unsigned long long)(uint32_t)a << 32) | (uint32_t)ldv(k1, i));
  }
}

__global__ void k_avg(const long long* __restrict__ sum /* I128 pairs */, const long long* __restrict__ cnt, int64_t n,
                      int scale, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double sc = 1.0;
    for (int q = 0; q < scale; ++q) sc *= 10.0;
    out[i] = i128_to_double((unsigned long long)sum[2 * i], sum[2 * i + 1]) / (double)cnt[i] / sc;
  }
}

}  // namespace

SX_EXPORT sx_status sx_groupby_merge(sx_ctx* ctx, const sx_col* keys, int nkeys, const sx_col* parts,
                                     const int32_t* ops, int nparts, const sx_having* having, int64_t groups_hint,
                                     sx_col* out_keys, sx_col* out_parts, int64_t* out_ngroups) {
  if (!ctx || !out_ngroups || nkeys < 1 || nkeys > 2 || !keys || !out_keys || nparts < 0 || nparts > SX_MAX_AGGS ||
      (nparts > 0 && (!parts || !ops || !out_parts)))
    return SX_EINVAL;
  *out_ngroups = 0;
  for (int k = 0; k < nkeys; ++k) out_keys[k] = sx_col{};
  for (int j = 0; j < nparts; ++j) out_parts[j] = sx_col{};
  ProfScope ps(ctx, "groupby_merge");
  int64_t n = keys[0].len;
  GbPlan P;
  std::memset(&P, 0, sizeof P);
  P.nkeys = nkeys;
  int kbits = 0;
  for (int k = 0; k < nkeys; ++k) {
    int t = keys[k].type;
    if (t != SX_U8 && t != SX_I32 && t != SX_DATE32 && t != SX_I64) return set_err(ctx, SX_ETYPE, "merge key type %d", t);
    if (nkeys == 2 && key_bits(t) > 32) return set_err(ctx, SX_ETYPE, "two-column keys must each be <= 32 bits");
    if (keys[k].len != n) return set_err(ctx, SX_EINVAL, "key columns differ in length");
    P.key_types[k] = P.out_key_type[k] = t;
    kbits += key_bits(t);
  }
  Layout& L = P.L;
  L.key_bytes = (nkeys == 1 && kbits <= 32) ? 4 : 8;
  L.nst = nparts;
  P.naggs = nparts;
  P.count_state = -1;
  MergeArgs m;
  std::memset(&m, 0, sizeof m);
  m.n = n;
  for (int j = 0; j < nparts; ++j) {
    if (parts[j].len != n) return set_err(ctx, SX_EINVAL, "partial columns differ in length");
    if (parts[j].validity) return set_err(ctx, SX_EUNSUPPORTED, "validity bitmaps unsupported");
    P.agg_op[j] = ops[j];
    P.agg_state[j] = j;
    switch (ops[j]) {
      case SX_SUM:
        if (parts[j].type != SX_I128) return set_err(ctx, SX_ETYPE, "SUM partials must be SX_I128");
        L.kind[j] = ST_SUM;
        m.lo[j] = (const unsigned long long*)parts[j].data;
        m.lo_stride[j] = 2;
        m.hi[j] = (const int*)((const char*)parts[j].data + 8);
        m.hi_stride[j] = 4;
        break;
      case SX_COUNT:
      case SX_MIN:
      case SX_MAX:
        if (parts[j].type != SX_I64) return set_err(ctx, SX_ETYPE, "COUNT/MIN/MAX partials must be SX_I64");
        L.kind[j] = ops[j] == SX_COUNT ? ST_COUNT : ops[j] == SX_MIN ? ST_MIN : ST_MAX;
        if (ops[j] == SX_COUNT) P.count_state = j;
        m.lo[j] = (const unsigned long long*)parts[j].data;
        m.lo_stride[j] = 1;
        break;
      default:
        return set_err(ctx, SX_EINVAL, "merge op %d (AVG: merge SUM and COUNT, then sx_avg)", ops[j]);
    }
  }
  // layout: key, 8-byte fields, 4-byte sum-hi fields
  int off = L.key_bytes == 4 ? 8 : 8;
  int first4 = -1;
  if (L.key_bytes == 4)
    for (int j = 0; j < nparts && first4 < 0; ++j)
      if (L.kind[j] == ST_SUM) { first4 = j; L.off4[j] = 4; }
  for (int j = 0; j < nparts; ++j) { L.off8[j] = off; off += 8; }
  for (int j = 0; j < nparts; ++j)
    if (L.kind[j] == ST_SUM && j != first4) { L.off4[j] = off; off += 4; }
  L.slot_bytes = (off + 7) & ~7;
  P.has_having = having != nullptr;
  if (having) {
    if (having->agg < 0 || having->agg >= nparts) return set_err(ctx, SX_EINVAL, "having index out of range");
    P.hv = *having;
  }
  Scratch scr(ctx);
  unsigned long long* packed;
  SX_TRY(scr.get(&packed, (size_t)(n > 0 ? n : 1)));
  DCol k0{keys[0].data, keys[0].type, 0}, k1{nkeys > 1 ? keys[1].data : keys[0].data, nkeys > 1 ? keys[1].type : keys[0].type, 0};
  if (n > 0) {
    k_pack_keys<<<persistent_grid(ctx, 8, (n + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(k0, k1, nkeys, n, packed);
    SX_CHECK_LAUNCH();
  }
  m.key = packed;
  uint64_t want = groups_hint > 0 ? (uint64_t)groups_hint : (uint64_t)(n > 16 ? n : 16);
  uint64_t cap = pow2_at_least(want + want / 3 + 1);
  if (cap < (uint64_t)n + (uint64_t)n / 3 + 1 && groups_hint <= 0) cap = pow2_at_least((uint64_t)n + n / 3 + 1);
  uint8_t* table;
  int* side;
  SX_TRY(scr.get(&table, (cap + 1) * L.slot_bytes));
  SX_TRY(scr.get(&side, 1));
  SX_CUDA(cudaMemsetAsync(table, 0, (cap + 1) * L.slot_bytes, ctx->stream));
  SX_CUDA(cudaMemsetAsync(side, 0, sizeof(int), ctx->stream));
  SX_CUDA(cudaMemsetAsync(ctx->d_flags, 0, 4 * sizeof(int), ctx->stream));
  Table t{table, cap - 1, side, ctx->d_flags + 1};
  if (n > 0) {
    k_gb_merge_records<<<persistent_grid(ctx, 8, (n + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(m, L, t);
    SX_CHECK_LAUNCH();
  }
  SlotFn sf;
  std::memset(&sf, 0, sizeof sf);
  sf.slots = table;
  sf.cap = cap;
  sf.slot_bytes = L.slot_bytes;
  sf.key_bytes = L.key_bytes;
  sf.side_used = side;
  sf.nsub = 1;
  sf.has_having = P.has_having;
  if (P.has_having) {
    int s = P.hv.agg;
    sf.hv_kind = L.kind[s];
    sf.hv_off8 = L.off8[s];
    sf.hv_off4 = L.off4[s];
    sf.hv_op = P.hv.op;
    sf.hv_lo = P.hv.lo;
    sf.hv_hi = P.hv.hi;
  }
  int32_t* ids;
  int64_t ng = 0;
  GatherSpec none;
  none.n = 0;
  SX_TRY(run_compact(ctx, sf, (int64_t)(cap + 1), nullptr, &ids, nullptr, none, &ng));
  scr.ptrs.push_back(ids);
  int flags[4];
  SX_CUDA(cudaMemcpy(flags, ctx->d_flags, sizeof flags, cudaMemcpyDeviceToHost));
  if (flags[1]) return set_err(ctx, SX_ENOMEM, "merge table full (groups_hint too small)");
  EmitArgs ea;
  std::memset(&ea, 0, sizeof ea);
  ea.slots = table;
  ea.ids = ids;
  ea.n = ng;
  ea.cap = cap;
  ea.L = L;
  ea.nkeys = nkeys;
  ea.naggs = nparts;
  ea.count_state = P.count_state;
  for (int k = 0; k < nkeys; ++k) {
    ea.out_key_type[k] = P.out_key_type[k];
    SX_TRY(scr.get((char**)&ea.out_key[k], (size_t)ng * type_width(P.out_key_type[k])));
  }
  for (int j = 0; j < nparts; ++j) {
    ea.agg_op[j] = ops[j];
    ea.agg_state[j] = j;
    SX_TRY(scr.get((char**)&ea.out_agg[j], (size_t)ng * type_width(agg_out_type(ops[j]))));
  }
  if (ng > 0) {
    k_gb_emit<<<persistent_grid(ctx, 8, (ng + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(ea);
    SX_CHECK_LAUNCH();
  }
  for (int k = 0; k < nkeys; ++k) {
    out_keys[k] = sx_col{P.out_key_type[k], 0, ng, ea.out_key[k], nullptr, nullptr};
    scr.release(ea.out_key[k]);
  }
  for (int j = 0; j < nparts; ++j) {
    out_parts[j] = sx_col{agg_out_type(ops[j]), 0, ng, ea.out_agg[j], nullptr, nullptr};
    scr.release(ea.out_agg[j]);
  }
  *out_ngroups = ng;
  return SX_OK;
}

SX_EXPORT sx_status sx_avg(sx_ctx* ctx, const sx_col* sum, const sx_col* count, int scale, sx_col* out) {
  if (!ctx || !sum || !count || !out) return SX_EINVAL;
  *out = sx_col{};
  if (sum->type != SX_I128 || count->type != SX_I64) return set_err(ctx, SX_ETYPE, "sx_avg needs I128 sum, I64 count");
  if (sum->len != count->len) return set_err(ctx, SX_EINVAL, "length mismatch");
  if (scale < 0 || scale > 18) return set_err(ctx, SX_EINVAL, "scale %d", scale);
  double* o;
  SX_TRY(alloc(ctx, &o, (size_t)(sum->len > 0 ? sum->len : 1)));
  if (sum->len > 0) {
    k_avg<<<persistent_grid(ctx, 8, (sum->len + kBlock - 1) / kBlock), kBlock, 0, SX_STREAM(ctx)>>>(
        (const long long*)sum->data, (const long long*)count->data, sum->len, scale, o);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      dfree(ctx, o);
      return set_err(ctx, SX_ECUDA, "sx_avg: %s", cudaGetErrorString(e));
    }
  }
  *out = sx_col{SX_F64, 0, sum->len, o, nullptr, nullptr};
  return SX_OK;
}
