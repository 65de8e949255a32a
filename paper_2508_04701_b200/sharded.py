"""Sharded (multi-GPU) TPC-H plans over the sx C ABI — SURVEY §8(e).

Placement: rank r of g holds shard r of every table (gen.gpu_tables(shard=(r, g))): contiguous
key ranges of customer/part/partsupp/supplier and contiguous order ranges of orders together with
their lineitems, so orders and lineitem are co-partitioned on orderkey.  Each plan is a local
pipeline of sx_* operators plus exchange operators:

* broadcast (sx_allgather): small dimension sets — customer keys (Q3), green parts / partsupp /
  supplier (Q9), Q18 candidates — and the partial aggregates / local top-k rows that every rank
  merges (sx_groupby_merge, sx_sort_topk);
* shuffle (sx_shuffle, NCCL all-to-all): re-partitions orders and lineitem on hash(orderkey) when
  they are not co-partitioned (``co_located=False``: Q3 — the Doris plan of P:458 — Q9's orders
  join and Q18's group-by / orders join).

Communicators: ``NcclComm`` (one process per GPU, libsx's NCCL exchange) and ``LoopbackComm``
(g logical ranks inside one process on one GPU; the exchange is device-to-device copies) — the
latter runs the same plans on a single B200 so sharded results can be checked against the
single-GPU executor and the oracle (tests/test_gpu_sharded.py).  Plans are written over a list of
the ranks this process drives (1 for NCCL, g for loopback); every collective takes and returns
one entry per local rank.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A
from . import col as mkcol
from .tpch import NATIONS, default_params

_TORCH = None


def _t():
    global _TORCH
    if _TORCH is None:
        import torch

        _TORCH = torch
    return _TORCH


def typed(t, typ):
    return (t, typ)


def sxcol(tc):
    t, typ = tc
    return mkcol(t, typ)


# ------------------------------------------------------------------------------- communicators
class LoopbackComm:
    """g logical ranks in one process on one GPU; exchange = stream-ordered device copies."""

    def __init__(self, ctx, nranks: int):
        self.ctx, self.nranks = ctx, nranks

    def _concat(self, parts, typ):
        torch = _t()
        n = sum(p.shape[0] for p in parts)
        shape = (n, 2) if typ == A.SX_I128 else (n,)
        out = torch.empty(shape, dtype=parts[0].dtype, device=parts[0].device)
        off = 0
        for p in parts:
            self.ctx.copy_into(out, off, p, p.shape[0])
            off += p.shape[0]
        return out

    def allgather(self, per_rank):
        """per_rank[r] = list of (tensor, type) -> list (per rank) of lists of (tensor, type)."""
        ncols = len(per_rank[0])
        out = [typed(self._concat([per_rank[r][c][0] for r in range(self.nranks)], per_rank[0][c][1]),
                     per_rank[0][c][1]) for c in range(ncols)]
        return [out for _ in range(self.nranks)]

    def shuffle(self, per_rank, key_cols):
        g = self.nranks
        parts, counts = [], []
        for r in range(g):
            p, cnt = self.ctx.partition_by_rank([sxcol(c) for c in per_rank[r]], key_cols, g)
            parts.append(p)
            counts.append(cnt)
        out = []
        for d in range(g):
            cols = []
            for c in range(len(per_rank[0])):
                segs = []
                for s in range(g):
                    off = sum(counts[s][:d])
                    segs.append(parts[s][c][off:off + counts[s][d]])
                cols.append(typed(self._concat(segs, per_rank[0][c][1]), per_rank[0][c][1]))
            out.append(cols)
        return out


class NcclComm:
    """This process's rank of an NCCL communicator built by libsx (sx_comm_init)."""

    def __init__(self, ctx, rank: int, nranks: int, unique_id: bytes):
        self.ctx, self.rank, self.nranks = ctx, rank, nranks
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        ctx.check(ctx.L.sx_comm_init(ctx.h, buf, rank, nranks, C.byref(h)))
        self.h = h

    @staticmethod
    def unique_id() -> bytes:
        from . import lib

        buf = (C.c_uint8 * 128)()
        st = lib().sx_comm_unique_id(buf)
        if st != 0:
            raise RuntimeError("sx_comm_unique_id failed")
        return bytes(buf)

    def close(self):
        if getattr(self, "h", None):
            self.ctx.L.sx_comm_destroy(self.h)
            self.h = None

    def allgather(self, per_rank):
        (cols,) = per_rank
        ca = (A.Col * len(cols))(*[sxcol(c) for c in cols])
        outs = (A.Col * len(cols))()
        n = C.c_int64()
        self.ctx.check(self.ctx.L.sx_allgather(self.ctx.h, self.h, ca, len(cols), outs, C.byref(n)))
        return [[typed(self.ctx.take_col(outs[i]), cols[i][1]) for i in range(len(cols))]]

    def shuffle(self, per_rank, key_cols):
        (cols,) = per_rank
        ca = (A.Col * len(cols))(*[sxcol(c) for c in cols])
        kc = (C.c_int32 * len(key_cols))(*key_cols)
        outs = (A.Col * len(cols))()
        n = C.c_int64()
        self.ctx.check(self.ctx.L.sx_shuffle(self.ctx.h, self.h, ca, len(cols), kc, len(key_cols), None, outs,
                                             C.byref(n)))
        return [[typed(self.ctx.take_col(outs[i]), cols[i][1]) for i in range(len(cols))]]


# ------------------------------------------------------------------------------- plans
def _okt(t):
    return A.SX_I64 if t.element_size() == 8 else A.SX_I32


def _np(t):
    return t.cpu().numpy()


def _i128(a):
    return [(int(lo) & ((1 << 64) - 1)) | (int(hi) << 64) for lo, hi in a]


E_DP = [(1, [(4, 1, 0), (5, -1, 100)])]


class ShardedTpch:
    """TPC-H Q1/Q3/Q6/Q9/Q18 over the local ranks' shards with an exchange communicator."""

    def __init__(self, ctx, comm, shards: list, co_located: bool = True):
        self.ctx, self.comm, self.shards, self.co_located = ctx, comm, shards, co_located
        self.R = range(len(shards))

    # ---- Q1: local group-by -> allgather partials -> merge -> avg -> order by flags
    def q1(self, p=None):
        P = p or default_params()
        c = self.ctx
        parts = []
        for t in self.shards:
            li = t["lineitem"]
            cols = [mkcol(li["l_shipdate"], A.SX_DATE32), mkcol(li["l_returnflag"], A.SX_U8),
                    mkcol(li["l_linestatus"], A.SX_U8)] + [mkcol(li[k], A.SX_DEC64) for k in
                                                           ("l_quantity", "l_extendedprice", "l_discount", "l_tax")]
            aggs = [("sum", [(1, [(3, 1, 0)])]), ("sum", [(1, [(4, 1, 0)])]), ("sum", [(1, [(4, 1, 0), (5, -1, 100)])]),
                    ("sum", [(1, [(4, 1, 0), (5, -1, 100), (6, 1, 100)])]), ("sum", [(1, [(5, 1, 0)])]), ("count", [])]
            k, a, _ = c.groupby(cols, [(1, "id"), (2, "id")], aggs, where=[(0, "le", P.q1_shipdate_max)], groups_hint=4)
            parts.append([typed(k[0], A.SX_U8), typed(k[1], A.SX_U8)] + [typed(x, A.SX_I128) for x in a[:5]]
                         + [typed(a[5], A.SX_I64)])
        g = self.comm.allgather(parts)[0]
        k, m, n = c.groupby_merge([sxcol(g[0]), sxcol(g[1])], [sxcol(x) for x in g[2:]], ["sum"] * 5 + ["count"],
                                  groups_hint=8)
        cnt = mkcol(m[5], A.SX_I64)
        avgs = [c.avg(mkcol(m[i], A.SX_I128), cnt, 2) for i in (0, 1, 4)]
        perm = c.sort_topk([mkcol(k[0], A.SX_U8), mkcol(k[1], A.SX_U8)], [(0, 0), (1, 0)])
        pk = [_np(c.gather(mkcol(x, A.SX_U8), perm)) for x in k]
        pm = [_i128(_np(c.gather(mkcol(m[i], A.SX_I128), perm))) for i in range(4)]
        pa = [_np(c.gather(mkcol(x, A.SX_F64), perm)) for x in avgs]
        pc = _np(c.gather(cnt, perm))
        return [(chr(pk[0][i]), chr(pk[1][i]), pm[0][i], pm[1][i], pm[2][i], pm[3][i], float(pa[0][i]),
                 float(pa[1][i]), float(pa[2][i]), int(pc[i])) for i in range(n)]

    # ---- Q6: local keyless reduce -> allgather -> merge
    def q6(self, p=None):
        P = p or default_params()
        c = self.ctx
        torch = _t()
        parts = []
        for t in self.shards:
            li = t["lineitem"]
            cols = [mkcol(li["l_shipdate"], A.SX_DATE32)] + [mkcol(li[k], A.SX_DEC64) for k in
                                                               ("l_discount", "l_quantity", "l_extendedprice")]
            where = [(0, "ge", P.q6_date_lo), (0, "lt", P.q6_date_hi), (1, "between", P.q6_disc_lo, P.q6_disc_hi),
                     (2, "lt", P.q6_qty_lt)]
            _, a, _ = c.groupby(cols, [], [("sum", [(1, [(3, 1, 0), (1, 1, 0)])]), ("count", [])], where=where)
            parts.append([typed(torch.zeros(1, dtype=torch.uint8, device=a[0].device), A.SX_U8),
                          typed(a[0], A.SX_I128), typed(a[1], A.SX_I64)])
        g = self.comm.allgather(parts)[0]
        _, m, _ = c.groupby_merge([sxcol(g[0])], [sxcol(g[1]), sxcol(g[2])], ["sum", "count"], groups_hint=1)
        s, n = _i128(_np(m[0]))[0], int(_np(m[1])[0])
        return [(None if n == 0 else s,)]

    # ---- Q3: broadcast customer keys; (optionally) shuffle orders and lineitem on orderkey;
    #      local joins and group-by (complete per orderkey); local top-k -> allgather -> top-k
    def q3(self, p=None):
        P = p or default_params()
        c = self.ctx
        ck = []
        for t in self.shards:
            cu = t["customer"]
            _, g = c.filter([mkcol(cu["c_custkey"], A.SX_I32), mkcol(cu["c_mktsegment"], A.SX_U8)],
                            [(1, "eq", P.q3_segment)], gather=[0])
            ck.append([typed(g[0], A.SX_I32)])
        allc = self.comm.allgather(ck)
        ords, lis = [], []
        for r, t in zip(self.R, self.shards):
            o, li = t["orders"], t["lineitem"]
            okt = _okt(o["o_orderkey"])
            ht = c.hash_build([sxcol(allc[r][0])], [0], unique=True)
            _, _, po = c.hash_probe(ht, [mkcol(o["o_custkey"], A.SX_I32), mkcol(o["o_orderdate"], A.SX_DATE32),
                                         mkcol(o["o_orderkey"], okt), mkcol(o["o_shippriority"], A.SX_I32)],
                                    [0], "semi", where=[(1, "lt", P.q3_date)], pp=[2, 1, 3])
            ht.close()
            ords.append([typed(po[0], okt), typed(po[1], A.SX_DATE32), typed(po[2], A.SX_I32)])
            cols = [mkcol(li["l_orderkey"], okt), mkcol(li["l_shipdate"], A.SX_DATE32),
                    mkcol(li["l_extendedprice"], A.SX_DEC64), mkcol(li["l_discount"], A.SX_DEC64)]
            sel, gl = c.filter(cols, [(1, "gt", P.q3_date)], gather=[0, 2, 3])
            lis.append([typed(gl[0], okt), typed(gl[1], A.SX_DEC64), typed(gl[2], A.SX_DEC64)])
        if not self.co_located:
            ords = self.comm.shuffle(ords, [0])
            lis = self.comm.shuffle(lis, [0])
        tops = []
        for r in self.R:
            okt = ords[r][0][1]
            ht = c.hash_build([sxcol(x) for x in ords[r]], [0], unique=True)
            _, _, pay = c.hash_probe(ht, [sxcol(x) for x in lis[r]], [0], "inner",
                                     build_cols=[sxcol(x) for x in ords[r]], bp=[1, 2], pp=[0, 1, 2])
            ht.close()
            gcols = [mkcol(pay[2], okt), mkcol(pay[3], A.SX_DEC64), mkcol(pay[4], A.SX_DEC64),
                     mkcol(pay[0], A.SX_DATE32), mkcol(pay[1], A.SX_I32)]
            k, a, _ = c.groupby(gcols, [(0, "id")], [("sum", [(1, [(1, 1, 0), (2, -1, 100)])]),
                                                      ("min", [(1, [(3, 1, 0)])]), ("min", [(1, [(4, 1, 0)])])],
                                groups_hint=max(1, pay[0].shape[0] // 2))
            cols = [typed(a[0], A.SX_I128), typed(a[1], A.SX_I64), typed(k[0], okt), typed(a[2], A.SX_I64)]
            perm = c.sort_topk([sxcol(x) for x in cols[:3]], [(0, 1), (1, 0), (2, 0)], P.q3_limit)
            tops.append([typed(c.gather(sxcol(x), perm), x[1]) for x in cols])
        g = self.comm.allgather(tops)[0]
        perm = c.sort_topk([sxcol(x) for x in g[:3]], [(0, 1), (1, 0), (2, 0)], P.q3_limit)
        rev = _i128(_np(c.gather(sxcol(g[0]), perm)))
        od, ok, pr = (_np(c.gather(sxcol(g[i]), perm)) for i in (1, 2, 3))
        return [(int(ok[i]), rev[i], int(od[i]), int(pr[i])) for i in range(len(rev))]

    # ---- Q9: broadcast green parts, partsupp', supplier; orders local; partial group-by -> merge
    def q9(self, p=None):
        P = p or default_params()
        c = self.ctx
        color = P.q9_color if isinstance(P.q9_color, bytes) else bytes(P.q9_color)
        color = color.split(b"\0")[0]
        gp = []
        for t in self.shards:
            pt = t["part"]
            _, g = c.filter([mkcol(pt["p_name_chars"], A.SX_STR, offsets=pt["p_name_offsets"]),
                             mkcol(pt["p_partkey"], A.SX_I32)], [(0, "contains", color)], gather=[1])
            gp.append([typed(g[0], A.SX_I32)])
        green = self.comm.allgather(gp)
        l2s, pss = [], []
        for r, t in zip(self.R, self.shards):
            li, ps = t["lineitem"], t["partsupp"]
            okt = _okt(li["l_orderkey"])
            ht = c.hash_build([sxcol(green[r][0])], [0], unique=True)
            lcols = [mkcol(li["l_partkey"], A.SX_I32), mkcol(li["l_suppkey"], A.SX_I32), mkcol(li["l_orderkey"], okt),
                     mkcol(li["l_quantity"], A.SX_DEC64), mkcol(li["l_extendedprice"], A.SX_DEC64),
                     mkcol(li["l_discount"], A.SX_DEC64)]
            _, _, l2 = c.hash_probe(ht, lcols, [0], "semi", pp=[0, 1, 2, 3, 4, 5])
            l2s.append([typed(l2[0], A.SX_I32), typed(l2[1], A.SX_I32), typed(l2[2], okt)]
                       + [typed(x, A.SX_DEC64) for x in l2[3:]])
            pcols = [mkcol(ps["ps_partkey"], A.SX_I32), mkcol(ps["ps_suppkey"], A.SX_I32),
                     mkcol(ps["ps_supplycost"], A.SX_DEC64)]
            _, _, pp = c.hash_probe(ht, pcols, [0], "semi", pp=[0, 1, 2])
            ht.close()
            pss.append([typed(pp[0], A.SX_I32), typed(pp[1], A.SX_I32), typed(pp[2], A.SX_DEC64)])
        psall = self.comm.allgather(pss)
        supp = self.comm.allgather([[typed(t["supplier"]["s_suppkey"], A.SX_I32),
                                     typed(t["supplier"]["s_nationkey"], A.SX_I32)] for t in self.shards])
        l4s = []
        for r, t in zip(self.R, self.shards):
            okt = l2s[r][2][1]
            ps_cols = [sxcol(x) for x in psall[r]]
            ht = c.hash_build(ps_cols, [0, 1], unique=True)
            _, _, l3 = c.hash_probe(ht, [sxcol(x) for x in l2s[r]], [0, 1], "inner", build_cols=ps_cols, bp=[2],
                                    pp=[1, 2, 3, 4, 5])
            ht.close()
            s_cols = [sxcol(x) for x in supp[r]]
            ht = c.hash_build(s_cols, [0], unique=True)
            l3c = [mkcol(l3[0], A.SX_DEC64), mkcol(l3[1], A.SX_I32), mkcol(l3[2], okt), mkcol(l3[3], A.SX_DEC64),
                   mkcol(l3[4], A.SX_DEC64), mkcol(l3[5], A.SX_DEC64)]
            _, _, l4 = c.hash_probe(ht, l3c, [1], "inner", build_cols=s_cols, bp=[1], pp=[0, 2, 3, 4, 5])
            ht.close()
            l4s.append([typed(l4[0], A.SX_I32), typed(l4[1], A.SX_DEC64), typed(l4[2], okt), typed(l4[3], A.SX_DEC64),
                        typed(l4[4], A.SX_DEC64), typed(l4[5], A.SX_DEC64)])
        ords = [[typed(t["orders"]["o_orderkey"], _okt(t["orders"]["o_orderkey"])),
                 typed(t["orders"]["o_orderdate"], A.SX_DATE32)] for t in self.shards]
        if not self.co_located:  # the orders join needs both sides on the owner rank of orderkey
            l4s = self.comm.shuffle(l4s, [2])
            ords = self.comm.shuffle(ords, [0])
        parts = []
        for r in self.R:
            l4c = [sxcol(x) for x in l4s[r]]
            ht = c.hash_build(l4c, [2])
            _, _, l5 = c.hash_probe(ht, [sxcol(x) for x in ords[r]], [0], "inner", build_cols=l4c,
                                    bp=[0, 1, 3, 4, 5], pp=[1])
            ht.close()
            gcols = [mkcol(l5[0], A.SX_I32), mkcol(l5[1], A.SX_DEC64), mkcol(l5[2], A.SX_DEC64),
                     mkcol(l5[3], A.SX_DEC64), mkcol(l5[4], A.SX_DEC64), mkcol(l5[5], A.SX_DATE32)]
            k, a, _ = c.groupby(gcols, [(0, "id"), (5, "year")],
                                [("sum", [(1, [(3, 1, 0), (4, -1, 100)]), (-1, [(1, 1, 0), (2, 1, 0)])])], groups_hint=256)
            parts.append([typed(k[0], A.SX_I32), typed(k[1], A.SX_I32), typed(a[0], A.SX_I128)])
        g = self.comm.allgather(parts)[0]
        k, m, n = c.groupby_merge([sxcol(g[0]), sxcol(g[1])], [sxcol(g[2])], ["sum"], groups_hint=256)
        torch = _t()
        order = sorted(range(25), key=lambda i: NATIONS[i])
        rank_of = np.empty(25, np.int32)
        rank_of[order] = np.arange(25, dtype=np.int32)
        rk = c.gather(mkcol(torch.from_numpy(rank_of).to(k[0].device), A.SX_I32), k[0])
        perm = c.sort_topk([mkcol(rk, A.SX_I32), mkcol(k[1], A.SX_I32)], [(0, 0), (1, 1)])
        nk = _np(c.gather(mkcol(k[0], A.SX_I32), perm))
        yr = _np(c.gather(mkcol(k[1], A.SX_I32), perm))
        sm = _i128(_np(c.gather(mkcol(m[0], A.SX_I128), perm)))
        return [(NATIONS[int(nk[i])], int(yr[i]), sm[i]) for i in range(n)]

    # ---- Q18: local group-by on orderkey (co-partitioned) + HAVING; orders local; customer join by
    #      broadcasting the (tiny) candidates; local top-k -> allgather -> top-k
    def q18(self, p=None):
        P = p or default_params()
        c = self.ctx
        lis, ords = [], []
        for t in self.shards:
            li, o = t["lineitem"], t["orders"]
            okt = _okt(o["o_orderkey"])
            lis.append([typed(li["l_orderkey"], okt), typed(li["l_quantity"], A.SX_DEC64)])
            ords.append([typed(o["o_orderkey"], okt), typed(o["o_custkey"], A.SX_I32),
                         typed(o["o_orderdate"], A.SX_DATE32), typed(o["o_totalprice"], A.SX_DEC64)])
        if not self.co_located:  # the group-by and the orders join are complete per orderkey owner
            lis = self.comm.shuffle(lis, [0])
            ords = self.comm.shuffle(ords, [0])
        cands = []
        for r in self.R:
            okt = ords[r][0][1]
            k, a, _ = c.groupby([sxcol(x) for x in lis[r]], [(0, "id")],
                                [("sum", [(1, [(1, 1, 0)])])], having=(0, "gt", P.q18_qty_gt),
                                groups_hint=max(1, ords[r][0][0].shape[0]))
            bcols = [mkcol(k[0], okt), mkcol(a[0], A.SX_I128)]
            ht = c.hash_build(bcols, [0], unique=True)
            _, _, cc = c.hash_probe(ht, [sxcol(x) for x in ords[r]], [0], "inner", build_cols=bcols, bp=[1],
                                    pp=[0, 1, 2, 3])
            ht.close()
            cands.append([typed(cc[0], A.SX_I128), typed(cc[1], okt), typed(cc[2], A.SX_I32),
                          typed(cc[3], A.SX_DATE32), typed(cc[4], A.SX_DEC64)])
        allc = self.comm.allgather(cands)
        joined = []
        for r, t in zip(self.R, self.shards):
            cols = [sxcol(x) for x in allc[r]]
            ht = c.hash_build(cols, [2])
            _, _, rr = c.hash_probe(ht, [mkcol(t["customer"]["c_custkey"], A.SX_I32)], [0], "inner", build_cols=cols,
                                    bp=[0, 1, 2, 3, 4])
            ht.close()
            joined.append([typed(x, allc[r][i][1]) for i, x in enumerate(rr)])
        R = self.comm.allgather(joined)[0]
        perm = c.sort_topk([sxcol(R[4]), sxcol(R[3]), sxcol(R[1])], [(0, 1), (1, 0), (2, 0)], P.q18_limit)
        sq = _i128(_np(c.gather(sxcol(R[0]), perm)))
        ok, ck, od, tp = (_np(c.gather(sxcol(R[i]), perm)) for i in (1, 2, 3, 4))
        return [("Customer#%09d" % int(ck[i]), int(ck[i]), int(ok[i]), int(od[i]), int(tp[i]), sq[i])
                for i in range(len(sq))]

    def run(self, q: str, p=None):
        return getattr(self, q)(p)
