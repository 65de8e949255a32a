"""One join µbench call (2^27 x 2^30 int64) with a given strategy — for ncu captures.

    python tools/join_one.py STRATEGY
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2508_04701_b200 as sx  # noqa: E402

strategy = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = sx.Ctx(0)
nb, npr = 1 << 27, 1 << 30
bk, bp = gen.mb_join_build(nb, device="cuda")
pk, pp = gen.mb_join_probe(nb, npr, False, seed=42, device="cuda")
_, _, pays, used = ctx.hash_join([sx.col(bk), sx.col(bp)], [0], [sx.col(pk), sx.col(pp)], [0], "inner", unique=True,
                                 bp=[1], pp=[1], strategy=strategy, rows=(False, False))
print("strategy", used, "rows", int(pays[0].numel()))
