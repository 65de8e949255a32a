// filter.cu — H1/H2: predicate scan (K1), string CONTAINS (K4), ordered
// compaction with fused materialization (K2/K3).  PAPER.md P:254 ("custom
// CUDA kernels ... predicate pushdown, and materialization"), P:422 (filter
// dominates Q6/Q19), P:271 (int32 kernel row ids).
#include "compact.cuh"
#include "filter.cuh"

using namespace sx;

namespace sx {

sx_status filter_internal(sx_ctx* ctx, const sx_col* cols, int ncols, const sx_pred* conj, int npred,
                          const sx_sel* in_sel, const int32_t* gather_cols, int ngather, sx_sel* out_sel,
                          sx_col* out_cols) {
  Scratch scr(ctx);
  int64_t n = 0;
  int ncontains = 0;
  for (int i = 0; i < npred; ++i) {
    if (conj[i].col < 0 || conj[i].col >= ncols) return set_err(ctx, SX_EINVAL, "predicate %d column out of range", i);
    ncontains += conj[i].op == SX_CONTAINS;
  }
  if (ncontains && npred != 1)
    return set_err(ctx, SX_EUNSUPPORTED, "SX_CONTAINS cannot be combined with other predicates in one sx_filter");
  if (ngather < 0 || ngather > kMaxGather) return set_err(ctx, SX_EINVAL, "ngather %d out of range", ngather);
  DCol dc[SX_MAX_COLS];
  // string columns are validated separately (DCol only carries fixed-width columns)
  for (int i = 0; i < ncols; ++i) {
    if (cols[i].validity) return set_err(ctx, SX_EUNSUPPORTED, "column %d has a validity bitmap (null-free v1)", i);
    if (cols[i].len > INT32_MAX) return set_err(ctx, SX_EINDEX, "column %d has more than INT32_MAX rows", i);
    SX_TRY(check_aligned(ctx, cols[i], i));
  }
  if (ncols > SX_MAX_COLS) return set_err(ctx, SX_EINVAL, "too many columns");
  for (int i = 0; i < ncols; ++i) dc[i] = DCol{cols[i].data, cols[i].type, 0};
  if (npred > 0) n = cols[conj[0].col].len;
  else if (ncols > 0) n = cols[0].len;
  if (in_sel) {
    if (in_sel->len > INT32_MAX) return set_err(ctx, SX_EINDEX, "selection longer than INT32_MAX");
    n = in_sel->len;
  }
  GatherSpec gs;
  gs.n = ngather;
  for (int g = 0; g < ngather; ++g) {
    int c = gather_cols[g];
    if (c < 0 || c >= ncols) return set_err(ctx, SX_EINVAL, "gather column %d out of range", c);
    int w = type_width(cols[c].type);
    if (w == 0) return set_err(ctx, SX_ETYPE, "gather column %d is not fixed-width", c);
    gs.g[g].src = dc[c];
    gs.g[g].by_aux = 0;
    gs.g[g].width = w;
    gs.g[g].dst = nullptr;  // allocated by run_compact at the exact output count
  }
  int32_t* sel = nullptr;
  int64_t count = 0;
  const int32_t* isel = in_sel ? in_sel->idx : nullptr;
  if (ncontains) {
    const sx_pred& p = conj[0];
    const sx_col& c = cols[p.col];
    if (c.type != SX_STR || !c.offsets) return set_err(ctx, SX_ETYPE, "SX_CONTAINS needs an SX_STR column");
    if (p.pattern_len < 0 || p.pattern_len > ContainsFn::kMaxPat || (p.pattern_len > 0 && !p.pattern))
      return set_err(ctx, SX_EINVAL, "pattern length %d (max %d)", p.pattern_len, ContainsFn::kMaxPat);
    ContainsFn f;
    f.offsets = c.offsets;
    f.chars = (const uint8_t*)c.data;
    f.plen = p.pattern_len;
    for (int i = 0; i < p.pattern_len; ++i) f.pat[i] = (uint8_t)p.pattern[i];
    SX_TRY(run_compact(ctx, f, n, isel, &sel, nullptr, gs, &count));
  } else {
    ConjFn f;
    SX_TRY(check_preds(ctx, cols, ncols, conj, npred, f.preds));
    for (int i = 0; i < ncols; ++i) f.cols[i] = dc[i];
    f.np = npred;
    SX_TRY(run_compact(ctx, f, n, isel, &sel, nullptr, gs, &count));
  }
  out_sel->len = count;
  out_sel->idx = sel;
  for (int g = 0; g < ngather; ++g) {
    out_cols[g] = cols[gather_cols[g]];
    out_cols[g].len = count;
    out_cols[g].data = gs.g[g].dst;
    out_cols[g].offsets = nullptr;
  }
  return SX_OK;
}

}  // namespace sx

SX_EXPORT sx_status sx_filter(sx_ctx* ctx, const sx_col* cols, int ncols, const sx_pred* conj, int npred,
                              const sx_sel* in_sel, const int32_t* gather_cols, int ngather, sx_sel* out_sel,
                              sx_col* out_cols) {
  if (!ctx || !out_sel || (npred > 0 && !conj) || (ngather > 0 && (!gather_cols || !out_cols))) return SX_EINVAL;
  *out_sel = sx_sel{0, nullptr};
  for (int g = 0; g < ngather && g < kMaxGather; ++g) out_cols[g] = sx_col{};
  ProfScope ps(ctx, "filter");
  sx_status st = filter_internal(ctx, cols, ncols, conj, npred, in_sel, gather_cols, ngather, out_sel, out_cols);
  if (st == SX_OK && ps.on()) {  // predicate columns + selection in + sel out (+ gathered, read and written)
    int64_t n = in_sel ? in_sel->len : (npred > 0 ? cols[conj[0].col].len : (ncols > 0 ? cols[0].len : 0));
    RefCols rc;
    double b = in_sel ? 4.0 * n : 0.0;
    for (int p = 0; p < npred; ++p) {
      rc.add(conj[p].col);
      const sx_col& c = cols[conj[p].col];
      if (c.type == SX_STR && n > 0) {  // string bytes of the scanned rows
        int64_t hi = 0;
        cudaMemcpy(&hi, c.offsets + c.len, sizeof hi, cudaMemcpyDeviceToHost);
        b += (double)hi * n / (double)(c.len > 0 ? c.len : 1);
      }
    }
    b += rc.row_bytes(cols, ncols) * n + 4.0 * out_sel->len;
    for (int g = 0; g < ngather; ++g) b += 2.0 * type_width(cols[gather_cols[g]].type) * out_sel->len;
    ps.set_bytes(b);
  }
  return st;
}
