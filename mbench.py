"""mbench.py — operator micro-benchmarks of the sx hot path (bench.py --workload join|join-zipf|groupby|sort).

SURVEY.md §8(d):
  C5a  join: build 2^27 (int64 key mix64(i), int64 payload i) x probe 2^30 (key of a uniform or
       Zipf(1.0) rank through an affine permutation, payload j) -> 2^30 (build payload, probe payload)
       pairs; algorithmic bytes 2 + 16 + 16 GiB.  Both strategies of sx_hash_join (flat table / radix
       partitioned, H5) are timed; `value` is the automatic choice.
  C5b  group-by sweep: N = 2^30 rows (int64 key mix64(g), g ~ U[0, G); DEC64 value) for
       G = 2^2 .. 2^26; sum, count, min, max, avg; bytes N*16 + G*(8 + 16 + 8 + 8 + 8 + 8).
  sort (ours): 2^28 uniform int64 keys + int32 payload; full sx_sort_topk; bytes 2*N*12.
Inputs are generated on the device (gen/, untimed) and are >> L2 (126 MB): no flush needed.
Parity at full size: the join against the oracle's closed form over the same generated rows (CPU,
chunked); group-by and sort against properties computed with library primitives (torch).
"""
from __future__ import annotations

import json
import os
import statistics
import time

import numpy as np
import torch

import gen
import paper_2508_04701_b200 as sx
from paper_2508_04701_b200 import _abi as A


def _time(fn, steps, warmup, stream):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def _free_outputs(ctx, op, ob, pays):
    for s in (op, ob):
        if s is not None:
            ctx.free_ptr(s.idx)
    for c in pays:
        ctx.free_ptr(c.data)


def _i64_pair_hash(b: torch.Tensor, p: torch.Tensor) -> int:
    """Σ mod 2^64 of the oracle's pair hash (oracle.or_pair_mix), in torch int64 (wrapping) arithmetic."""
    m32 = 0xFFFFFFFF
    c1 = 0x9E3779B97F4A7C15 - (1 << 64)
    c2 = 0xD6E8FEB86659FD93 - (1 << 64)
    tot = 0
    for i in range(0, b.numel(), 1 << 26):
        z = (b[i:i + (1 << 26)] * c1) ^ p[i:i + (1 << 26)]
        z = (z ^ ((z >> 32) & m32)) * c2
        z = z ^ ((z >> 32) & m32)
        tot += int(z.sum().item())
    return tot % (1 << 64)


def join(args, ctx, zipf: bool):
    import oracle  # test infrastructure: the closed-form check of the full-size result

    nb, npr = 1 << args.mb_build_log2, 1 << args.mb_probe_log2
    bk, bp = gen.mb_join_build(nb, device="cuda")
    pk, pp = gen.mb_join_probe(nb, npr, zipf, seed=args.seed, device="cuda")
    bcols, pcols = [sx.col(bk), sx.col(bp)], [sx.col(pk), sx.col(pp)]
    stream = torch.cuda.current_stream()

    def step(strategy):
        op, ob, pays, used = ctx.hash_join(bcols, [0], pcols, [0], "inner", unique=True, bp=[1], pp=[1],
                                           strategy=strategy, rows=(False, False), raw=True)
        _free_outputs(ctx, op, ob, pays)
        return used

    used_auto = step(0)
    ms = {}
    for name, st in (("flat", 1), ("partitioned", 2), ("flat_inline", 3)):
        ms[name] = _time(lambda: step(st), args.steps, args.warmup, stream)
    sx.lib().sx_launch_count(ctx.h, 1)
    ms_auto = _time(lambda: step(0), args.steps, 0, stream)
    launches = sx.lib().sx_launch_count(ctx.h, 1) / args.steps
    # parity: full-size result summary vs the oracle closed form over the same rows (CPU, chunked)
    op, ob, (gb, gp), _ = ctx.hash_join(bcols, [0], pcols, [0], "inner", unique=True, bp=[1], pp=[1], strategy=0,
                                        rows=(False, False))
    got = {"count": int(gb.numel()), "sum_build": int(gb.sum().item()), "sum_probe": int(gp.sum().item()),
           "pair_hash": _i64_pair_hash(gb, gp)}
    del gb, gp
    want = {"count": 0, "sum_build": 0, "sum_probe": 0, "pair_hash": 0}
    t0 = time.time()
    chunk = 1 << 24
    for r0 in range(0, npr, chunk):
        k, p = gen.mb_join_probe(nb, npr, zipf, seed=args.seed, r0=r0, r1=min(npr, r0 + chunk))
        s = oracle.mb_join_closed(nb, k, p)
        for key in want:
            want[key] += s[key]
    want["pair_hash"] %= 1 << 64
    t_or = time.time() - t0
    parity = "closed form (oracle, all %d pairs): %s" % (want["count"], "OK" if got == want else f"MISMATCH {got} vs {want}")
    algo = (nb + npr) * 16 + want["count"] * 16
    strat = {1: "flat", 2: "partitioned", 3: "flat_inline"}[used_auto]
    return {
        "workload": f"join µbench {'Zipf(1.0)' if zipf else 'uniform'}: build 2^{args.mb_build_log2} x probe "
                    f"2^{args.mb_probe_log2} int64 (SURVEY §8(d) C5a)",
        "ms": ms_auto, "algo_bytes": algo, "launches": launches, "parity": parity,
        "extra": {"strategy_auto": strat, "ms_flat": round(ms["flat"], 3), "ms_partitioned": round(ms["partitioned"], 3),
                  "ms_flat_inline": round(ms["flat_inline"], 3),
                  "gbs_flat": round(algo / ms["flat"] / 1e6, 1), "gbs_partitioned": round(algo / ms["partitioned"] / 1e6, 1),
                  "gbs_flat_inline": round(algo / ms["flat_inline"] / 1e6, 1),
                  "oracle_check_s": round(t_or, 1), "rows_per_s": round(npr / (ms_auto / 1e3), 1)},
        "kernel": f"sx_hash_join ({strat})",
    }


def groupby(args, ctx):
    n = 1 << args.mb_gb_log2
    Gs = [1 << g for g in range(2, 27)] if not args.mb_groups else [int(x) for x in args.mb_groups.split(",")]
    stream = torch.cuda.current_stream()
    points, tot_b, tot_ms, bad = [], 0.0, 0.0, []
    launches = 0
    for G in Gs:
        k, v = gen.mb_groupby(n, G, seed=args.seed, device="cuda")
        cols = [sx.col(k), sx.col(v, A.SX_DEC64, 2)]
        val = [(1, [(1, 1, 0)])]
        aggs = [("sum", val), ("count", []), ("min", val), ("max", val), ("avg", val, 2)]

        def step():
            return ctx.groupby(cols, [(0, "id")], aggs, groups_hint=G, raw=True)

        def run_free():
            ok, oa, ng = step()
            for c in list(ok) + list(oa):
                ctx.free_ptr(c.data)

        sx.lib().sx_launch_count(ctx.h, 1)
        ms = _time(run_free, args.steps, args.warmup, stream)
        launches += sx.lib().sx_launch_count(ctx.h, 1) / (args.steps + args.warmup)
        b = n * 16 + G * 56
        points.append({"G": G, "ms": round(ms, 4), "gbs": round(b / ms / 1e6, 1)})
        tot_b += b
        tot_ms += ms
        # parity by properties (torch primitives): group count, Σcount, Σsum, sampled groups exactly
        keys, (s, c, mn, mx, av), _ = ctx.groupby(cols, [(0, "id")], aggs, groups_hint=G)
        ng = int(keys[0].numel())
        err = []
        if ng != int(torch.unique(k).numel()):
            err.append("ngroups")
        if int(c.sum().item()) != n:
            err.append("count")
        lo = s[:, 0].cpu().numpy().view(np.uint64).astype(object)
        hi = s[:, 1].cpu().numpy().astype(object)
        if int(sum(lo) + (sum(hi) << 64)) != int(v.sum().item()):
            err.append("sum")
        for gi in torch.randint(0, ng, (4,)).tolist():
            m = k == keys[0][gi]
            vv = v[m]
            s_exact = int(lo[gi]) + (int(hi[gi]) << 64)
            if (s_exact != int(vv.sum().item()) or int(c[gi]) != int(m.sum().item()) or int(mn[gi]) != int(vv.min().item())
                    or int(mx[gi]) != int(vv.max().item())):
                err.append(f"group{gi}")
        if err:
            bad.append((G, err))
        del k, v, keys, s, c, mn, mx, av
        torch.cuda.empty_cache()
    parity = "properties (torch): ngroups, Σcount, Σsum, 4 sampled groups exact per G: " + ("OK" if not bad else f"FAIL {bad}")
    return {
        "workload": f"group-by sweep µbench: N = 2^{args.mb_gb_log2} int64 keys, G = {Gs[0]}..{Gs[-1]} "
                    "(sum, count, min, max, avg; SURVEY §8(d) C5b)",
        "ms": tot_ms, "algo_bytes": tot_b, "launches": launches, "parity": parity,
        "extra": {"points": points}, "kernel": "sx_groupby_agg (sweep total)",
    }


def sort(args, ctx):
    n = 1 << args.mb_sort_log2
    k, p = gen.mb_sort(n, seed=args.seed, device="cuda")
    cols = [sx.col(k), sx.col(p)]
    stream = torch.cuda.current_stream()

    def run_free():
        perm = ctx.sort_topk(cols, [(0, False)], raw=True)
        ctx.free_ptr(perm.idx)

    sx.lib().sx_launch_count(ctx.h, 1)
    ms = _time(run_free, args.steps, args.warmup, stream)
    launches = sx.lib().sx_launch_count(ctx.h, 1) / (args.steps + args.warmup)
    perm = ctx.sort_topk(cols, [(0, False)]).long()
    ks = k[perm]
    ok = bool((ks[1:] >= ks[:-1]).all().item()) and bool((torch.sort(perm).values == torch.arange(n, device="cuda")).all().item())
    parity = "properties (torch): permutation and non-decreasing keys: " + ("OK" if ok else "FAIL")
    return {"workload": f"sort µbench: 2^{args.mb_sort_log2} uniform int64 keys + int32 payload (ours, SURVEY §8(d))",
            "ms": ms, "algo_bytes": 2 * n * 12, "launches": launches, "parity": parity,
            "extra": {"keys_per_s": round(n / (ms / 1e3), 1)}, "kernel": "sx_sort_topk (full)"}


def run(args, metric, clock_sampler, peak, peak_src):
    ctx = sx.Ctx(0)
    with clock_sampler(0) as clk:
        if args.workload in ("join", "join-zipf"):
            r = join(args, ctx, args.workload == "join-zipf")
        elif args.workload == "groupby":
            r = groupby(args, ctx)
        else:
            r = sort(args, ctx)
    ms = r["ms"]
    gbs = r["algo_bytes"] / (ms / 1e3) / 1e9
    line = {
        "metric": metric, "value": round(gbs, 2), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded generator on the device)",
        "config": {"workload": r["workload"], "seed": args.seed, "algorithmic_bytes_per_step": r["algo_bytes"],
                   "l2_note": "inputs >> 126 MB L2; no flush needed"},
        "parity": r["parity"],
        "roofline": {"bound": "hbm", "kernel": r["kernel"], "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(gbs / peak, 4), "traffic": None, "peak_source": peak_src},
        "gpu_launches": r["launches"], "clocks": clk.summary(), **r["extra"],
    }
    print(json.dumps(line))
