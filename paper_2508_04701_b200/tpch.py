"""Fixed-plan TPC-H executor binding: Q1/Q3/Q6/Q9/Q18 via sx_tpch_q* (include/sx.h).

Tables are dicts of torch CUDA tensors in the gen/ layout.  Results come back in
the canonical row form shared with the oracle's decoder (see oracle/__init__.py),
so tests compare them directly.
"""
from __future__ import annotations

import ctypes as C

from . import _abi as A

QUERIES = ("q1", "q6", "q3", "q9", "q18")

NATIONS = [
    "ALGERIA", "ARGENTINA", "BRAZIL", "CANADA", "EGYPT", "ETHIOPIA", "FRANCE", "GERMANY",
    "INDIA", "INDONESIA", "IRAN", "IRAQ", "JAPAN", "JORDAN", "KENYA", "MOROCCO",
    "MOZAMBIQUE", "PERU", "CHINA", "ROMANIA", "SAUDI ARABIA", "VIETNAM", "RUSSIA",
    "UNITED KINGDOM", "UNITED STATES",
]

# column -> (table, sx type, scale)
_SCHEMA = {
    "l_orderkey": ("lineitem", None, 0), "l_partkey": ("lineitem", A.SX_I32, 0), "l_suppkey": ("lineitem", A.SX_I32, 0),
    "l_quantity": ("lineitem", A.SX_DEC64, 2), "l_extendedprice": ("lineitem", A.SX_DEC64, 2),
    "l_discount": ("lineitem", A.SX_DEC64, 2), "l_tax": ("lineitem", A.SX_DEC64, 2),
    "l_returnflag": ("lineitem", A.SX_U8, 0), "l_linestatus": ("lineitem", A.SX_U8, 0),
    "l_shipdate": ("lineitem", A.SX_DATE32, 0),
    "o_orderkey": ("orders", None, 0), "o_custkey": ("orders", A.SX_I32, 0), "o_orderdate": ("orders", A.SX_DATE32, 0),
    "o_shippriority": ("orders", A.SX_I32, 0), "o_totalprice": ("orders", A.SX_DEC64, 2),
    "c_custkey": ("customer", A.SX_I32, 0), "c_mktsegment": ("customer", A.SX_U8, 0),
    "p_partkey": ("part", A.SX_I32, 0), "p_name": ("part", A.SX_STR, 0),
    "ps_partkey": ("partsupp", A.SX_I32, 0), "ps_suppkey": ("partsupp", A.SX_I32, 0),
    "ps_supplycost": ("partsupp", A.SX_DEC64, 2),
    "s_suppkey": ("supplier", A.SX_I32, 0), "s_nationkey": ("supplier", A.SX_I32, 0),
}


def _i128(v) -> int:
    return (int(v.hi) << 64) | int(v.lo)


def default_params(**over) -> A.TpchParams:
    from . import lib

    p = A.TpchParams()
    lib().sx_tpch_default_params(C.byref(p))
    for k, v in over.items():
        if k == "q9_color":
            v = v.encode() if isinstance(v, str) else v
        setattr(p, k, v)
    return p


class Tpch:
    """Device-resident TPC-H tables bound to an sx context."""

    def __init__(self, ctx, tables: dict):
        self.ctx = ctx
        self.tables = tables
        T = A.TpchTables()
        for name, (tname, typ, scale) in _SCHEMA.items():
            t = tables.get(tname)
            if t is None:
                continue
            if name == "p_name":
                chars, offs = t["p_name_chars"], t["p_name_offsets"]
                setattr(T, name, A.Col(A.SX_STR, 0, offs.shape[0] - 1, chars.data_ptr() if chars.numel() else None,
                                       offs.data_ptr(), None))
                continue
            if name not in t:
                continue
            x = t[name]
            if typ is None:  # orderkey: I32 or I64 by width
                typ = A.SX_I64 if x.element_size() == 8 else A.SX_I32
            setattr(T, name, A.Col(typ, scale, x.shape[0], x.data_ptr() if x.numel() else None, None, None))
        self.T = T

    @classmethod
    def upload(cls, ctx, host_tables: dict) -> "Tpch":
        """Tables in host memory (CPU torch tensors, pinned for full PCIe speed) -> device copies made
        by the library (sx_tpch_upload: stream-ordered H2D inside the C ABI).  free() releases them."""
        h = cls(ctx, host_tables)
        dev = A.TpchTables()
        ctx.check(ctx.L.sx_tpch_upload(ctx.h, C.byref(h.T), C.byref(dev)))
        obj = cls.__new__(cls)
        obj.ctx, obj.tables, obj.T, obj._owned = ctx, host_tables, dev, True
        return obj

    def free(self):
        if getattr(self, "_owned", False):
            self.ctx.L.sx_tpch_tables_free(self.ctx.h, C.byref(self.T))
            self._owned = False

    def run(self, q: str, params: A.TpchParams | None = None) -> list:
        c = self.ctx
        P = params or default_params()
        n = C.c_int64()
        if q == "q1":
            out = (A.Q1Row * 64)()
            c.check(c.L.sx_tpch_q1(c.h, C.byref(self.T), C.byref(P), out, 64, C.byref(n)))
            return [(chr(r.returnflag), chr(r.linestatus), _i128(r.sum_qty), _i128(r.sum_base_price),
                     _i128(r.sum_disc_price), _i128(r.sum_charge), r.avg_qty, r.avg_price, r.avg_disc,
                     r.count_order) for r in out[:n.value]]
        if q == "q6":
            out = A.Q6Row()
            c.check(c.L.sx_tpch_q6(c.h, C.byref(self.T), C.byref(P), C.byref(out), C.byref(n)))
            return [(None if out.is_null else _i128(out.revenue),)]
        if q == "q3":
            cap = max(int(P.q3_limit), 1) if P.q3_limit >= 0 else max(self.T.o_orderkey.len, 1)
            out = (A.Q3Row * cap)()
            c.check(c.L.sx_tpch_q3(c.h, C.byref(self.T), C.byref(P), out, cap, C.byref(n)))
            return [(r.l_orderkey, _i128(r.revenue), r.o_orderdate, r.o_shippriority) for r in out[:n.value]]
        if q == "q9":
            out = (A.Q9Row * 4096)()
            c.check(c.L.sx_tpch_q9(c.h, C.byref(self.T), C.byref(P), out, 4096, C.byref(n)))
            return [(NATIONS[r.nationkey], r.o_year, _i128(r.sum_profit)) for r in out[:n.value]]
        if q == "q18":
            cap = max(int(P.q18_limit), 1) if P.q18_limit >= 0 else max(self.T.o_orderkey.len, 1)
            out = (A.Q18Row * cap)()
            c.check(c.L.sx_tpch_q18(c.h, C.byref(self.T), C.byref(P), out, cap, C.byref(n)))
            return [("Customer#%09d" % r.c_custkey, r.c_custkey, r.o_orderkey, r.o_orderdate, r.o_totalprice,
                     _i128(r.sum_qty)) for r in out[:n.value]]
        raise ValueError(q)
