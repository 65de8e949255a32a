"""Run one TPC-H query of the executor repeatedly (for ncu launch lists / per-query profiling).

    python tools/run_query.py --query q18 --sf 100 --reps 2
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file out.csv \
        python tools/run_query.py --query q18 --sf 100 --reps 1 --warm 1

Prints per-operator CUDA-event times of the last repetition.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import gen  # noqa: E402
import paper_2508_04701_b200 as sx  # noqa: E402
from paper_2508_04701_b200.tpch import Tpch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--query", default="q18")
    ap.add_argument("--sf", type=float, default=100.0)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--warm", type=int, default=0, help="unprofiled runs before --reps (with cudaProfilerStart gating)")
    a = ap.parse_args()
    ctx = sx.Ctx(0)
    tables = gen.gpu_tables(gen.sf_to_milli(a.sf), a.seed)
    t = Tpch(ctx, tables)
    for _ in range(a.warm):
        t.run(a.query)
    torch.cuda.synchronize()
    for r in range(a.reps):
        ctx.profile(True)
        t.run(a.query)
        prof = ctx.profile_read()
        ctx.profile(False)
    for name, ms in prof:
        print(f"{ms:9.3f}  {name}")


if __name__ == "__main__":
    main()
