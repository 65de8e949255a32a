// groupby.cu — H3/H7/H8: sx_groupby_agg (hash group-by with sum/count/min/max/avg over
// exact integer value expressions; keyless reduce; HAVING).
//
// PAPER.md P:96/P:191 (aggregations via libcudf; here our kernels), P:420 (group-by is
// substantial in Q1 — few groups => memory contention — and Q18 — many groups)
// (avg carried as sum+count).  Output group order is unspecified.
#include "compact.cuh"
#include "gb_host.cuh"

using namespace sx;

namespace sx {

struct InterpRow {
  DCol cols[SX_MAX_COLS];
  DPred preds[SX_MAX_PREDS];
  int np;
  int nkeys;
  int kc[2];
  int kfn[2];
  int nst;
  int kind[kMaxStates];
  sx_expr expr[kMaxStates];
  int* ovf_flag;
  __device__ __forceinline__ bool row(int64_t r, uint64_t& key, int64_t (&v)[kMaxStates]) const {
    if (!eval_conj(cols, preds, np, r)) return false;
    key = 0;
    if (nkeys >= 1) {
      int64_t k0 = ldv(cols[kc[0]], r);
      if (kfn[0] == SX_KEY_YEAR) k0 = civil_year((int32_t)k0);
      if (nkeys == 1) {
        key = (uint64_t)k0;
      } else {
        int64_t k1 = ldv(cols[kc[1]], r);
        if (kfn[1] == SX_KEY_YEAR) k1 = civil_year((int32_t)k1);
        key = ((uint64_t)(uint32_t)k0 << 32) | (uint32_t)k1;
      }
    }
    bool ovf = false;
    for (int a = 0; a < nst; ++a) v[a] = kind[a] == ST_COUNT ? 0 : eval_expr(expr[a], cols, r, ovf);
    if (ovf) atomicExch(ovf_flag, 1);
    return true;
  }
};

}  // namespace sx

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
  GbPlan plan;
  SX_TRY(gb_plan(ctx, cols, ncols, keys, nkeys, aggs, naggs, having, &plan));
  InterpRow fn;
  SX_TRY(to_dcols(ctx, cols, ncols, fn.cols));
  SX_TRY(check_preds(ctx, cols, ncols, where, nwhere, fn.preds));
  fn.np = nwhere;
  fn.nkeys = nkeys;
  for (int k = 0; k < nkeys; ++k) { fn.kc[k] = keys[k].col; fn.kfn[k] = keys[k].fn; }
  fn.nst = plan.L.nst;
  for (int a = 0; a < plan.L.nst; ++a) { fn.kind[a] = plan.L.kind[a]; fn.expr[a] = plan.state_expr[a]; }
  fn.ovf_flag = ctx->d_flags;
  int64_t n = in_sel ? in_sel->len : (ncols > 0 ? cols[0].len : 0);
  if (!in_sel && nkeys > 0) n = cols[keys[0].col].len;
  if (n > INT32_MAX) return set_err(ctx, SX_EINDEX, "group-by input exceeds INT32_MAX rows");
  return gb_run(ctx, fn, plan, in_sel ? in_sel->idx : nullptr, n, groups_hint, out_keys, out_aggs, out_ngroups);
}
