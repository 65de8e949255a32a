"""bench.py — TPC-H Q1+Q6+Q3+Q9+Q18 on the B200-native sx hot path (one JSON line).

A "step" is one pass of the whole hot path: the five fixed plans (filter, compaction,
hash build/probe, group-by, top-k: SURVEY.md §8(a) H1-H9) over the resident SF100 tables
(BASELINE.json configs[2], the metric's single-GPU configuration).

    python bench.py [--gpus N --steps K --warmup W] [--sf 100] [--impl sx|reference]

value     = algorithmic bytes scanned per step (every referenced column read once at its
            stored width, + mandatory state; SURVEY §8(d) / DESIGN.md) / device time, GB/s,
            whole job (sum over ranks).  Inputs (36 GB at SF100) are >> L2 (126 MB): no flush needed.
e2e       = the same metric through the public C ABI with HOST (pinned) inputs: sx_tpch_upload copies
            every column H2D inside libsx, the plans' results are written to host memory; all timed.
roofline  = the dominant operator (largest device time in the step, from sx per-call CUDA events
            on the launching stream), achieved algorithmic GB/s vs MEASURED_PEAKS.json hbm_gbs.
cpu_baseline = the CPU oracle (single thread) on a bounded sample (SF 1) on this host.
--impl reference: the oracle timed as the reference arm (rank 0 only), same metric/unit.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TPC-H query time & HBM GB/s vs peak at SF100 (1 B200) / SF1000 (1-8 GPU)"
QUERIES = ("q1", "q6", "q3", "q9", "q18")


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# ---------------------------------------------------------------------------------- bytes
def table_sizes(tables) -> dict:
    n = {}
    n["l"] = int(tables["lineitem"]["l_shipdate"].shape[0])
    n["o"] = int(tables["orders"]["o_orderkey"].shape[0])
    n["c"] = int(tables["customer"]["c_custkey"].shape[0])
    n["p"] = int(tables["part"]["p_partkey"].shape[0])
    n["p_chars"] = int(tables["part"]["p_name_chars"].shape[0])
    n["ps"] = int(tables["partsupp"]["ps_partkey"].shape[0])
    n["s"] = int(tables["supplier"]["s_suppkey"].shape[0])
    ok = tables["lineitem"]["l_orderkey"]
    n["kb"] = int(ok.element_size() if hasattr(ok, "element_size") else ok.itemsize)
    return n


def query_bytes(n: dict) -> dict:
    """Algorithmic bytes per query: referenced columns read once at stored width (+ group state
    written and read for Q18's 1.5e8-group aggregation).  SURVEY App. C 'Bytes per query'."""
    kb = n["kb"]
    return {
        "q1": n["l"] * (4 + 1 + 1 + 8 * 4),
        "q6": n["l"] * (4 + 8 * 3),
        "q3": n["l"] * (kb + 4 + 8 + 8) + n["o"] * (kb + 4 + 4 + 4) + n["c"] * (4 + 1),
        "q9": n["l"] * (4 + 4 + kb + 8 * 3) + n["p"] * (4 + 8) + n["p_chars"] + n["ps"] * 16 + n["s"] * 8
              + n["o"] * (kb + 4),
        "q18": n["l"] * (kb + 8) + n["o"] * (kb + 4 + 4 + 8) + n["c"] * 4 + 2 * n["o"] * (kb + 8),
    }


# ---------------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = os.path.join("/tmp", f"sx_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.proc or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------- oracle (CPU)
def oracle_bin():
    path = os.path.join(ROOT, "oracle", "sx_oracle")
    if not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", ROOT, "oracle"], check=True)
    return path


def oracle_bytes(sf_milli: int) -> int:
    import gen

    t = gen.cpu_tables(sf_milli, seed=42)
    return sum(query_bytes(table_sizes(t)).values())


def run_oracle(sf_milli: int, reps: int) -> list[float]:
    """Seconds per rep (sum over the five queries), generation excluded."""
    per_rep = [0.0] * reps
    for q in QUERIES:
        r = subprocess.run([oracle_bin(), "--query", q, "--sf-milli", str(sf_milli), "--reps", str(reps)],
                           check=True, capture_output=True, text=True)
        d = json.loads(r.stdout.strip().splitlines()[-1])
        for i, s in enumerate(d["seconds"]):
            per_rep[i] += s
    return per_rep


# ---------------------------------------------------------------------------------- main
def bench_config(args, world: int) -> dict:
    """The workload a bench line is quoted on; identical in the sx and the reference arm."""
    sf_total = args.sf * world
    return {"workload": f"TPC-H Q1+Q6+Q3+Q9+Q18 SF{args.sf:g} (one step = all five plans)",
            "sf": args.sf, "seed": args.seed,
            "l2_note": "inputs (>30 GB) >> 126 MB L2; no flush needed",
            "parallelism": (f"sharded x{world}: rank r holds shard r of SF{sf_total:g}; "
                            "allgather/shuffle over NCCL" if world > 1 else "single GPU")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sf", type=float, default=100.0)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--impl", default="sx", choices=["sx", "reference"])
    ap.add_argument("--cpu-sf", type=float, default=10.0, help="oracle sample scale factor (cpu_baseline)")
    ap.add_argument("--ref-sf", type=float, default=1.0, help="oracle sample scale factor per step (--impl reference)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--workload", default="tpch", choices=["tpch", "join", "join-zipf", "groupby", "sort"],
                    help="tpch (default): Q1+Q6+Q3+Q9+Q18 step; others: operator µbenchmarks (mbench.py)")
    ap.add_argument("--mb-build-log2", type=int, default=27)
    ap.add_argument("--mb-probe-log2", type=int, default=30)
    ap.add_argument("--mb-gb-log2", type=int, default=30)
    ap.add_argument("--mb-groups", default="", help="comma list of G (default 2^2..2^26)")
    ap.add_argument("--mb-sort-log2", type=int, default=28)
    args = ap.parse_args()

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    import gen

    sf_milli = gen.sf_to_milli(args.sf)
    cpu_milli = gen.sf_to_milli(args.cpu_sf)

    if args.workload != "tpch" and args.impl == "sx":
        import mbench

        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        peak = float(peaks.get("hbm_gbs", 6650.0))
        src = "of measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "of fallback (B200_PROFILING.md 6.65 TB/s)"
        mbench.run(args, METRIC, ClockSampler, peak, src)
        return

    if args.impl == "reference":
        cpu_milli = gen.sf_to_milli(args.ref_sf)
        args.cpu_sf = args.ref_sf
        if rank != 0:
            return
        reps = args.warmup + args.steps
        secs = run_oracle(cpu_milli, reps)[args.warmup:]
        b = oracle_bytes(cpu_milli)
        t = statistics.mean(secs)
        v = b / t / 1e9
        sample = (f"bounded sample of the SF{args.sf * args.gpus:g} workload: the same five plans at SF "
                  f"{args.cpu_sf:g} per step ({b / 1e9:.2f} GB algorithmic), materialised host "
                  "columns, generation excluded, single-threaded C++ oracle")
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded TPC-H-shaped generator)",
            # the same config as the sx arm's line (the workload this arm samples); the sample itself
            # is described in cpu_baseline.sample
            "config": bench_config(args, args.gpus),
            "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2508_04701_b200 as sx
    from paper_2508_04701_b200 import tpch

    ctx = sx.Ctx(local)
    if world > 1:
        # weak scaling: total SF = sf x world, rank r holds shard r of every table (orders and
        # lineitem co-partitioned on orderkey); exchanges (allgather / shuffle) run over libsx's
        # NCCL communicator; torch.distributed only distributes the NCCL unique id.
        from paper_2508_04701_b200.sharded import NcclComm, ShardedTpch

        uid = [NcclComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = NcclComm(ctx, rank, world, uid[0])
        sf_total = sf_milli * world
        tables = gen.gpu_tables(sf_total, seed=args.seed, shard=(rank, world), device=f"cuda:{local}")
        runner = ShardedTpch(ctx, comm, [tables])
        run = runner.run
    else:
        sf_total = sf_milli
        tables = gen.gpu_tables(sf_milli, seed=args.seed, device=f"cuda:{local}")
        T = tpch.Tpch(ctx, tables)
        run = T.run
    n = table_sizes(tables)
    qb = query_bytes(n)
    step_bytes = sum(qb.values())
    job_bytes = step_bytes
    if dist:
        tb = torch.tensor([step_bytes], dtype=torch.float64, device="cuda")
        dist.all_reduce(tb)
        job_bytes = float(tb.item())

    # parity at full size against the committed oracle answers (when present for this SF/seed)
    parity = "not checked (no committed answers for this SF/seed)"
    ans_path = os.path.join(ROOT, "tests", "golden", f"answers_sf{sf_total}_seed{args.seed}.json")
    results = {q: run(q) for q in QUERIES}
    if os.path.exists(ans_path):
        import oracle as _or  # test infrastructure: only the committed answer decoding is used here
        from tests.helpers import rows_equal

        ans = json.load(open(ans_path))["answers"]
        bad = []
        for q in QUERIES:
            if q not in ans:
                continue
            want = [tuple(r) for r in ans[q]]
            if q == "q9":
                want = [(_or.NATIONS[r[0]], r[1], r[2]) for r in want]
            if q == "q18":
                want = [(_or.c_name(r[0]),) + tuple(r) for r in want]
            if not rows_equal(results[q], want):
                bad.append(q)
        parity = "bit-exact vs committed CPU-oracle answers: " + ("ALL OK" if not bad else "MISMATCH " + ",".join(bad))

    for _ in range(args.warmup):
        for q in QUERIES:
            run(q)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    ctx.profile(True)
    ctx.profile_read()
    sx.lib().sx_launch_count(ctx.h, 1)
    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            for q in QUERIES:
                run(q)
        e1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    launches = sx.lib().sx_launch_count(ctx.h, 1)
    prof = ctx.profile_read(with_bytes=True)
    ctx.profile(False)
    ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = job_bytes / (ms / 1e3) / 1e9

    # per-operator breakdown (query-level entries and operator entries in call order); every sx call
    # reports its algorithmic bytes (SURVEY §8(d) definition 1) beside its CUDA-event time
    per_q = {q.upper(): [] for q in QUERIES}
    ops, op_b = {}, {}
    cur = None
    # profile records are pushed at scope entry: query scope first, then its operator calls
    for name, t, b in prof:
        if name in per_q:
            per_q[name].append(t)
            cur = name
        else:
            key = f"{cur}/{name}"
            ops.setdefault(key, []).append(t)
            op_b.setdefault(key, []).append(b)
    q_ms = {q: round(statistics.mean(v), 4) for q, v in per_q.items() if v}
    op_ms = {k: round(sum(v) / args.steps, 4) for k, v in ops.items()}
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "of measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "of fallback (B200_PROFILING.md 6.65 TB/s)"
    # per-operator achieved algorithmic GB/s and fraction of the HBM peak
    op_gbs = {k: {"ms": op_ms[k], "gb": round(sum(op_b[k]) / args.steps / 1e9, 4),
                  "gbs": round(sum(op_b[k]) / (sum(ops[k]) / 1e3) / 1e9, 1) if sum(ops[k]) > 0 else None}
              for k in ops}
    # "frac" = ALGORITHMIC bytes (every referenced column once) / time / peak.  A kernel that skips
    # sectors (Q6's lazy loads fetch discount/quantity/price only where a shipdate qualifies) can
    # read above 1.0 here; "dram_frac" (ncu DRAM bytes from profiles/traffic.json, when captured)
    # is the bandwidth the kernel actually pulled.
    traffic_all = {}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic_all = json.load(open(tp))
    for k, v in op_gbs.items():
        v["frac"] = round(v["gbs"] / peak, 4) if v["gbs"] is not None else None
        v["frac_kind"] = "algorithmic"
        calls = len(ops[k]) / args.steps
        if traffic_all.get(k) and v["ms"]:
            v["dram_frac"] = round(traffic_all[k] / (v["ms"] / max(calls, 1) / 1e3) / 1e9 / peak, 4)
    dom = max(op_ms, key=op_ms.get) if op_ms else None
    roof = None
    if dom:
        calls = len(ops[dom]) / args.steps
        dur = op_ms[dom] / max(calls, 1)
        ob = sum(op_b[dom]) / len(op_b[dom])
        traffic = traffic_all.get(dom)
        ach = ob / (dur / 1e3) / 1e9 if ob > 0 else None
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1) if ach else None, "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4) if ach else None, "traffic": traffic, "algorithmic_bytes": round(ob),
                "ms_per_launch": round(dur, 4), "peak_source": peak_src}

    # e2e: the public C ABI with HOST (pinned) inputs: sx_tpch_upload copies every column H2D inside
    # the library, the five plans run, their results land in host memory; all of it timed per step
    e2e = None
    if not args.no_e2e and world == 1:
        host = {tn: {cn: torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for cn, t in cols.items()}
                for tn, cols in tables.items()}
        for tn, cols in tables.items():
            for cn, t in cols.items():
                host[tn][cn].copy_(t)
        torch.cuda.synchronize()
        h2d = sum(t.numel() * t.element_size() for cols in host.values() for t in cols.values())
        e0.record(stream)
        for _ in range(args.e2e_steps):
            Te = tpch.Tpch.upload(ctx, host)
            for q in QUERIES:
                Te.run(q)  # results land in host memory inside the call
            Te.free()
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / args.e2e_steps
        # result bytes per step (host row structs): Q1 4x, Q6 1x, Q3 10x, Q9 175x, Q18 100x rows
        d2h = 4 * 112 + 32 + 10 * 40 + 175 * 24 + 100 * 40
        ev = job_bytes / (e_ms / 1e3) / 1e9
        e2e = {"value": round(ev, 3), "unit": "GB/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": d2h,
               "ms_per_step": round(e_ms, 3), "path": "sx_tpch_upload (host pinned -> device inside libsx) + sx_tpch_q*"}
        del host
    elif not args.no_e2e:
        # sharded: every rank's shard copied from pinned host memory, then the sharded plans
        host = {tn: {cn: torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for cn, t in cols.items()}
                for tn, cols in tables.items()}
        for tn, cols in tables.items():
            for cn, t in cols.items():
                host[tn][cn].copy_(t)
        torch.cuda.synchronize()
        h2d = sum(t.numel() * t.element_size() for cols in host.values() for t in cols.values())
        e0.record(stream)
        for _ in range(args.e2e_steps):
            for tn, cols in host.items():
                for cn, t in cols.items():
                    tables[tn][cn].copy_(t, non_blocking=True)
            for q in QUERIES:
                run(q)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.e2e_steps], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
        d2h = 4 * 112 + 32 + 10 * 40 + 175 * 24 + 100 * 40
        e2e = {"value": round(job_bytes / (e_ms / 1e3) / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": d2h, "ms_per_step": round(e_ms, 3)}
        del host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            secs = run_oracle(cpu_milli, 1)
            b = oracle_bytes(cpu_milli)
            cpu = {"value": round(b / secs[0] / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                   "sample": f"TPC-H Q1+Q6+Q3+Q9+Q18 at SF {args.cpu_sf:g} ({b / 1e9:.2f} GB algorithmic), "
                             f"single-threaded C++ oracle, materialised host columns, {secs[0]:.1f} s",
                   "host_cpus": os.cpu_count()}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (seeded TPC-H-shaped generator, generated in HBM; decimals scaled int64)",
            "config": bench_config(args, world),
            "workload_detail": {"rows_lineitem": n["l"], "algorithmic_bytes_per_step": step_bytes,
                                "query_bytes": qb, "sf_total": sf_total / 1000, "job_bytes_per_step": job_bytes},
            "query_ms": q_ms, "operator_ms": op_ms, "operator_roofline": op_gbs, "parity": parity,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if "MISMATCH" in parity:
            # a step whose results differ from the oracle has no valid throughput
            line["value"] = None
            line["invalid"] = "parity mismatch at full size: " + parity
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    if rank == 0 and "MISMATCH" in parity:
        sys.exit(1)


if __name__ == "__main__":
    main()
