"""Diagnose the Q18 'big quantity' case (quantities >= 2^40) strategy by strategy.

    SX_RUNS_LEAN=0 timeout 90 python tools/diag_q18big.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2508_04701_b200 as sx  # noqa: E402
from paper_2508_04701_b200 import tpch  # noqa: E402
from tests.helpers import rows_equal  # noqa: E402


def main():
    ctx = sx.Ctx(0)
    host = gen.cpu_tables(100, seed=13)
    li = {k: v.copy() for k, v in host["lineitem"].items()}
    n = len(li["l_orderkey"])
    li["l_quantity"][[5, 70_000, n - 1]] = 1 << 41
    host = dict(host)
    host["lineitem"] = li
    dev = {t: {c: torch.from_numpy(np.ascontiguousarray(a)).cuda() for c, a in cols.items()} for t, cols in host.items()}
    T = tpch.Tpch(ctx, dev)
    t0 = time.time()
    print("env:", {k: v for k, v in os.environ.items() if k.startswith("SX_")}, flush=True)
    got = T.run("q18")
    torch.cuda.synchronize()
    print("q18 done in %.2f s" % (time.time() - t0), flush=True)
    want = oracle.run_query("q18", host)
    print("parity:", rows_equal(got, want), flush=True)


if __name__ == "__main__":
    main()
