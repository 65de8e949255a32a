// groupby.cu — H3/H7/H8: sx_groupby_agg (hash group-by with sum/count/min/max/avg over
// exact integer value expressions; keyless reduce; HAVING).
//
// PAPER.md P:96/P:191 (aggregations via libcudf; here our kernels), P:420 (group-by is
// substantial in Q1 — few groups => memory contention — and Q18 — many groups)
// (avg carried as sum+count).  Output group order is unspecified.
#include "compact.cuh"
#include "gb_host.cuh"

using namespace sx;

SX_EXPORT sx_status sx_groupby_agg(sx_ctx* ctx, const sx_col* cols, int ncols, const sx_key* keys, int nkeys,
                                   const sx_sel* in_sel, const sx_pred* where, int nwhere, const sx_agg* aggs,
                                   int naggs, const sx_having* having, int64_t groups_hint, sx_col* out_keys,
                                   sx_col* out_aggs, int64_t* out_ngroups) {
  if (!ctx || !out_ngroups || (naggs > 0 && (!aggs || !out_aggs)) || (nkeys > 0 && (!keys || !out_keys)))
    return SX_EINVAL;
  *out_ngroups = 0;
  for (int i = 0; i < nkeys && i < 2; ++i) out_keys[i] = sx_col{};
  for (int i = 0; i < naggs && i < SX_MAX_AGGS; ++i) out_aggs[i] = sx_col{};
  ProfScope ps(ctx, "groupby");
  // K18: the plain shape (one integer key, plain-column aggregates, no filter) in shared memory
  sx_status st = gb_simple(ctx, cols, ncols, keys, nkeys, in_sel, nwhere, aggs, naggs, having, groups_hint, out_keys,
                           out_aggs, out_ngroups);
  if (st != SX_EUNSUPPORTED) {
    if (st == SX_OK && ps.on()) {  // key + value columns once; the G output rows once
      RefCols rc;
      rc.add(keys[0].col);
      for (int a = 0; a < naggs; ++a)
        if (aggs[a].op != SX_COUNT) rc.add(aggs[a].value.t[0].f[0].col);
      double out_row = type_width(out_keys[0].type);
      for (int a = 0; a < naggs; ++a) out_row += type_width(out_aggs[a].type);
      ps.set_bytes(rc.row_bytes(cols, ncols) * (double)cols[keys[0].col].len + out_row * (double)*out_ngroups);
    }
    return st;
  }
  ctx->err.clear();
  GbPlan plan;
  SX_TRY(gb_plan(ctx, cols, ncols, keys, nkeys, aggs, naggs, having, &plan));
  GbArgs A;
  std::memset(&A, 0, sizeof A);
  SX_TRY(to_dcols(ctx, cols, ncols, A.cols));
  SX_TRY(check_preds(ctx, cols, ncols, where, nwhere, A.preds));
  A.np = nwhere;
  A.nkeys = nkeys;
  for (int k = 0; k < nkeys; ++k) { A.kc[k] = keys[k].col; A.kfn[k] = keys[k].fn; }
  for (int a = 0; a < plan.L.nst; ++a) A.expr[a] = plan.state_expr[a];
  A.ovf_flag = ctx->d_flags;
  int64_t n = in_sel ? in_sel->len : (ncols > 0 ? cols[0].len : 0);
  if (!in_sel && nkeys > 0) n = cols[keys[0].col].len;
  if (n > INT32_MAX) return set_err(ctx, SX_EINDEX, "group-by input exceeds INT32_MAX rows");
  InterpProg prog;
  prog.A = A;
  prog.ovf_flag = ctx->d_flags;
  st = gb_run(ctx, prog, plan, in_sel ? in_sel->idx : nullptr, n, groups_hint, out_keys, out_aggs, out_ngroups);
  if (st == SX_OK && ps.on()) {  // referenced columns + selection once; the G output rows once
    RefCols rc;
    for (int k = 0; k < nkeys; ++k) rc.add(keys[k].col);
    for (int p = 0; p < nwhere; ++p) rc.add(where[p].col);
    for (int a = 0; a < naggs; ++a)
      if (aggs[a].op != SX_COUNT)
        for (int t = 0; t < aggs[a].value.nterms && t < 2; ++t)
          for (int f = 0; f < aggs[a].value.t[t].nf && f < 3; ++f) rc.add(aggs[a].value.t[t].f[f].col);
    double out_row = 0;
    for (int k = 0; k < nkeys; ++k) out_row += type_width(out_keys[k].type);
    for (int a = 0; a < naggs; ++a) out_row += type_width(out_aggs[a].type);
    ps.set_bytes((rc.row_bytes(cols, ncols) + (in_sel ? 4.0 : 0.0)) * n + out_row * (double)*out_ngroups);
  }
  return st;
}
